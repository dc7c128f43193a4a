"""PEER backend, executed for real: n processes (torchrun, one rank each) exchange bands by one-sided
stores into each other's device memory and synchronise with device flag barriers (App. A P:238;
§3.2).  The box of the GPU tests has one GPU, so the ranks share cuda:0 (separate CUDA contexts;
the stores go through the CUDA IPC mappings exactly as they would over NVLink).  The trajectory of
every step and the gathered x_0 of pcpp_sample must equal the LOOPBACK backend's bitwise."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [
    # model, H, n, p, w, S, steps, precision, scheme
    ("tiny", 32, 2, 0.25, 1, 4, 4, "bf16", "pcpp"),          # config T
    ("tiny", 32, 4, 0.5, 2, 4, 4, "fp32", "fullmap"),
    ("tiny", 32, 2, 1.0, 1, 4, 3, "bf16", "sync"),
    ("sdxl", 32, 2, 0.3, 1, 50, 4, "bf16", "pcpp"),         # SDXL-shaped: stride-2 and upsample halos
    ("sdxl", 32, 4, 0.8, 2, 50, 5, "bf16", "pcpp"),
]

# CFG device split: 2 x n processes, branch groups of n patches + the per-step
# eps swap between partners
SPLIT = [
    # model, H, n, p, w, S, steps, precision, scheme
    ("tiny", 32, 1, 0.0, 1, 4, 4, "bf16", "pcpp"),
    ("tiny", 32, 2, 0.25, 1, 4, 4, "fp32", "pcpp"),
    ("sdxl", 32, 2, 0.3, 1, 50, 4, "bf16", "pcpp"),
]


@pytest.mark.parametrize("split", [False, True], ids=["batch2", "cfgsplit"])
@pytest.mark.parametrize("case", CASES + SPLIT, ids=lambda c: "-".join(map(str, c)))
def test_peer_backend_multiprocess_bitwise_equals_loopback(cuda_ok, case, split, tmp_path):
    model, H, n, p, w, S, steps, prec, scheme = case
    if split != (case in SPLIT):
        pytest.skip("case list of the other mode")
    out = tmp_path / "res.json"
    nproc = 2 * n if split else n
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={29500 + (os.getpid() % 400)}",
           os.path.join(ROOT, "tests", "_peer_worker.py"), "--same-gpu", "--model", model, "--H", str(H),
           "--p", str(p), "--w", str(w), "--S", str(S), "--steps", str(steps), "--precision", prec,
           "--scheme", scheme, "--out", str(out)] + (["--cfg-split"] if split else [])
    # heuristic GEMM configurations: every process (ranks and the loopback reference) picks the same
    # split-K / tile choice, so the comparison can be bitwise (plan-time autotuning is timing-dependent)
    env = dict(os.environ, PYTHONPATH=ROOT, PCPP_AUTOTUNE="0")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(out.read_text())
    print(res)
    assert res["backend"] == 2
    assert res["ok"], res
    if split:
        assert res["bytes_eps"] == 2 * n * (H // n) * H * 16
