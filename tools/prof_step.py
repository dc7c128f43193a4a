"""Steps of one loopback plan at a given workload (for ncu launch lists / captures).

usage: python tools/prof_step.py [n] [res] [model] [steps]   (defaults 1 128 sdxl 3)
The plan is built (GEMM table from profiles/gemm_tune_b200.txt), then `steps` steps run after
the synchronous warm-up; an ncu range of the last step's kernels is the per-step launch list."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_02962_b200 import inputs, pcpp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
res = int(sys.argv[2]) if len(sys.argv) > 2 else 128
model = sys.argv[3] if len(sys.argv) > 3 else "sdxl"
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
p = {1: 0.0, 2: 0.3, 4: 0.8, 8: 0.8}[n]
w = 4 if n > 1 else 0
os.environ.setdefault("PCPP_TUNE_FILE", os.path.join(ROOT, "profiles", "gemm_tune_b200.txt"))
blob = inputs.make_weight_blob(inputs.init_specs(pcpp.manifest(model)))
cfg = pcpp.make_config(model=model, num_steps=50, precision="bf16", scheme="pcpp", backend="loopback")
pl = pcpp.Plan(res, res, 4, n, p, w, cfg, blob)
del blob
pl.pcpp_set_cond(inputs.make_cond(1280 if model.startswith("sdxl") else 512))
if model.endswith("_xf"):
    pl.pcpp_set_context(inputs.make_context(77, 2048 if model.startswith("sdxl") else 256))
lat = torch.from_numpy(np.ascontiguousarray(inputs.make_latent(res, res))).cuda()
# PROF_RANGE=1: only the last step inside cudaProfilerStart/Stop (ncu --profile-from-start off)
rng = os.environ.get("PROF_RANGE") == "1"
for k in range(w + steps):
    if rng and k == w + steps - 1:
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
    pl.pcpp_step(lat, k)
torch.cuda.synchronize()
if rng:
    torch.cuda.cudart().cudaProfilerStop()
print("launches/step", pl.pcpp_query()["n_kernels_per_step"])
pl.close()
