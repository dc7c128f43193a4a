"""Per-op device-time table (PCPP_OP_TIMING) of one async step of an n-patch loopback plan at 1024^2."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PCPP_OP_TIMING", "1")
import numpy as np, torch
from paper_2412_02962_b200 import inputs, pcpp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
p = {1: 0.0, 2: 0.3, 4: 0.8, 8: 0.8}[n]
res = int(sys.argv[2]) if len(sys.argv) > 2 else 128
tune = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "gemm_tune_b200.txt")
os.environ.setdefault("PCPP_TUNE_FILE", tune)
blob = inputs.make_weight_blob(inputs.init_specs(pcpp.manifest("sdxl")))
cfg = pcpp.make_config(model="sdxl", num_steps=50, precision="bf16", scheme="pcpp", backend="loopback")
pl = pcpp.Plan(res, res, 4, n, p, 4 if n > 1 else 0, cfg, blob)
pl.pcpp_set_cond(inputs.make_cond(1280))
lat = torch.from_numpy(np.ascontiguousarray(inputs.make_latent(res, res))).cuda()
for k in range(6):
    pl.pcpp_step(lat, k)
torch.cuda.synchronize()
pl.pcpp_profile(lat, 31, 0, 1)
pl.close()
