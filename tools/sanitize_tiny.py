"""The tiny (or SDXL-shaped 32x32) PCPP path (n = 2 loopback, bf16 tcgen05 kernels, eager launches) for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import model as M
from paper_2412_02962_b200 import inputs, pcpp
model = sys.argv[1] if len(sys.argv) > 1 else "tiny"
blob = inputs.round_to_bf16(inputs.make_weight_blob(M.weight_specs(model)))
cfg = pcpp.make_config(model=model, num_steps=4 if model == "tiny" else 50, precision="bf16", graphs=False)
plan = pcpp.Plan(32, 32, 4, 2, 0.25 if model == "tiny" else 0.3, 1, cfg, blob)
plan.pcpp_set_cond(inputs.make_cond(512 if model == "tiny" else 1280))
lat = torch.from_numpy(np.array(inputs.make_latent(32, 32))).cuda()
for k in range(3):
    plan.pcpp_step(lat, k)
torch.cuda.synchronize()
plan.close()
print("ok", float(lat.abs().mean()))
