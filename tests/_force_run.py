"""Child process for test_gpu_path.test_forced_gemm_configs: runs one whole-path case with the GEMM
configuration pinned through PCPP_GEMM_FORCE (read once per process) and saves the latents."""
import sys

import numpy as np

from tests.test_gpu_path import lib_run

if __name__ == "__main__":
    out = sys.argv[1]
    xs, info = lib_run("sdxl", 32, 1, 0.0, 0, 50, "bf16", "pcpp", 2)
    np.save(out, np.stack(xs))
