"""Mainloop time per K step (first operand stage landed -> last MMA issued, median over CTAs) of the 1-CTA
GEMM for several tile widths BN and grid sizes, from the PCPP_GEMM_TRACE stamps: separates the
per-SM operand feed (bytes per K step: A 16 KB + B BN x 128 B) from the MMA time (BN / 2 clk at 128 x BN x 16)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) == 1:
    for bn in (64, 128, 160, 256):
        env = dict(os.environ, PCPP_GEMM_FORCE=f"{bn},1,0", PCPP_GEMM_TRACE="1")
        subprocess.run([sys.executable, __file__, str(bn)], env=env, cwd=ROOT)
    sys.exit(0)
sys.path.insert(0, ROOT)
import numpy as np
from paper_2412_02962_b200 import pcpp
from tools.graph_timing import g_conv
bn = int(sys.argv[1])
for rows, N in ((4, 1280), (32, 1280), (32, 3840)):
    ms, tf = g_conv(rows, 32, 1280, N, 1, 1)
    n, tr = pcpp.pcpp_debug_gemm_trace()
    t = tr[(n - 1) % 32].astype(np.float64)
    t = t[t[:, 0] > 0]
    ml = np.median(t[:, 3] - t[:, 2]) / 1e3
    ksteps = 20 * (-(-(rows * 64 // 128) * (N // bn) // 148))      # k-steps of the busiest CTA
    kb = 16 + bn * 128 / 1024
    print(f"BN={bn:3d} M={rows * 64:5d} N={N}: {ms * 1e3:6.2f} us/launch, CTAs={len(t)}, mainloop {ml:5.2f} us for "
          f"{ksteps} k-steps = {ml * 1e3 / ksteps:6.1f} ns/k-step ({ml * 1965 / ksteps:5.0f} clk; MMA {bn * 2:4d} clk), "
          f"feed {kb:.0f} KB/k-step -> {kb * 1024 / (ml * 1965 / ksteps):5.1f} B/clk", flush=True)
