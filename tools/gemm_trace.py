"""GEMM launch timeline from the PCPP_GEMM_TRACE %globaltimer stamps: 12 back-to-back launches of one
shape replayed in a CUDA graph; per launch the phases (median over CTAs, us) relative to the first CTA's
entry, and the gap to the previous launch's last CTA exit."""
import os, sys
os.environ["PCPP_GEMM_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2412_02962_b200 import pcpp
from tools.graph_timing import g_conv

SHAPES = [(4, 32, 1280, 1280, 1, 1), (32, 32, 1280, 1280, 1, 1), (32, 32, 1280, 3840, 1, 1), (4, 32, 1280, 1280, 9, 1),
          (2, 32, 64, 64, 1, 1)]
EPI = os.environ.get("EPI", "bias")          # epilogue operands: none | bias | bias+temb | bias+temb+res
for sh in SHAPES:
    ms, tf = g_conv(*sh, res="res" in EPI, bias="bias" in EPI, temb="temb" in EPI)
    n, tr = pcpp.pcpp_debug_gemm_trace()
    tr = tr.astype(np.float64)
    launches = []
    for k in range(12):                       # the last 12 launches of this shape (ring slot = launch % 32)
        t = tr[(n - 12 + k) % 32]
        used = t[:, 0] > 0
        launches.append(t[used])
    launches.sort(key=lambda t: t[:, 0].min())
    print(f"[{EPI}] shape rows={sh[0]} W={sh[1]} K={sh[2]} N={sh[3]} taps={sh[4]}: {ms * 1e3:.2f} us/launch ({tf:.0f} TF/s), CTAs={len(launches[-1])}")
    prev_end = None
    for t in launches:
        e = t[:, 0].min()
        rel = lambda i: np.median(t[:, i] - e) / 1e3
        gap = (e - prev_end) / 1e3 if prev_end is not None else float("nan")
        print(f"   gap {gap:6.2f}  wait {rel(1):5.2f}  first-stage {rel(2):5.2f}  last-mma {rel(3):5.2f}  acc {rel(4):5.2f}"
              f"  epi-done {rel(5):5.2f}  exit {rel(6):5.2f}  last-exit {(t[:, 6].max() - e) / 1e3:5.2f}  entry-spread {(t[:, 0].max() - e) / 1e3:5.2f}")
        prev_end = t[:, 6].max()
