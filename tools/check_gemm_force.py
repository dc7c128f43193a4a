"""Op-level check of one forced GEMM configuration (PCPP_GEMM_FORCE, read once per process) against a
torch fp32 reference on the same bf16 operands, over small-M shapes (1x1 and 3x3, residual, temb)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F
from paper_2412_02962_b200 import pcpp
torch.manual_seed(0)
worst = 0.0
for rows, W, Cin, Cout, taps in ((4, 32, 1280, 1280, 1), (4, 32, 1280, 1280, 9), (8, 64, 640, 640, 9), (2, 32, 256, 256, 1),
                                 (16, 128, 320, 320, 9), (4, 48, 640, 384, 1)):
    pad = 1 if taps == 9 else 0
    x = torch.randn(rows + 2 * pad, 2, W, Cin, device="cuda").bfloat16()
    if pad:
        x[0].zero_(); x[-1].zero_()
    w = (torch.randn(Cout, taps * Cin, device="cuda") / (taps * Cin) ** 0.5).bfloat16()
    b = torch.randn(Cout, device="cuda")
    t = torch.randn(2, Cout, device="cuda")
    res = torch.randn(rows, 2, W, Cout, device="cuda").bfloat16()
    y = torch.empty(rows, 2, W, Cout, device="cuda", dtype=torch.bfloat16)
    pcpp.pcpp_op_conv(x, rows, 2, W, Cin, taps, 1, w, b, t, res, y, Cout)
    torch.cuda.synchronize()
    xi = x.float().permute(1, 3, 0, 2)                                   # [B][C][rows+2p][W]
    wk = w.float().view(Cout, 3, 3, Cin).permute(0, 3, 1, 2) if taps == 9 else w.float().view(Cout, Cin, 1, 1)
    ref = F.conv2d(xi, wk, padding=(0, 1) if taps == 9 else 0)           # rows padded by the halo rows
    ref = ref.permute(2, 0, 3, 1) + b + t[None, :, None, :] + res.float()
    err = ((y.float() - ref).norm() / ref.norm()).item()
    worst = max(worst, err)
    print(f"rows={rows} W={W} Cin={Cin} Cout={Cout} taps={taps}: rel-L2 {err:.2e}", flush=True)
print("FORCE", os.environ.get("PCPP_GEMM_FORCE"), "worst", f"{worst:.2e}", "OK" if worst < 1e-2 else "FAIL")
