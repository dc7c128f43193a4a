"""Attention kernel timing at the 1024^2 step's shapes (CUDA events, back-to-back launches)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_02962_b200 import pcpp
from tools.bench_ops import t_attn
SHAPES = [("L1 n=1", 64, 64, 640, (64,)), ("L2 n=1", 32, 32, 1280, (32,)),
                             ("L1 n=8 p=.8", 8, 64, 640, (6, 8, 6)), ("L2 n=8 p=.8", 4, 32, 1280, (3, 4, 3))]
for name, h, W, C, rows in SHAPES[:int(sys.argv[1]) if len(sys.argv) > 1 else 4]:
    ms, gf = t_attn(h, W, C, rows)
    ex = h * W * sum(rows) * W * (C // 64) * 2
    print(f"{name:14s} {ms*1e3:8.1f} us  {gf/1e3:7.1f} TF/s  exp2 {ex/ms/1e9:6.2f} T/s ({ex/ms/1e9/4.63*100:4.1f}% of MUFU)")
