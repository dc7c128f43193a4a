"""One async step of an n-patch loopback plan at 1024^2 (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2412_02962_b200 import inputs, pcpp
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
p = {2: 0.3, 4: 0.8, 8: 0.8}[n]
os.environ.setdefault("PCPP_TUNE_FILE", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "gemm_tune_b200.txt"))
blob = inputs.make_weight_blob(inputs.init_specs(pcpp.manifest("sdxl")))
cfg = pcpp.make_config(model="sdxl", num_steps=50, precision="bf16", scheme="pcpp", backend="loopback")
pl = pcpp.Plan(128, 128, 4, n, p, 4, cfg, blob)
pl.pcpp_set_cond(inputs.make_cond(1280))
lat = torch.from_numpy(np.ascontiguousarray(inputs.make_latent(128, 128))).cuda()
for k in range(7):
    pl.pcpp_step(lat, k)
torch.cuda.synchronize()
pl.close()
