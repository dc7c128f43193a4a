"""Per-shape timing of libpcpp's contraction kernels (pcpp_op_conv / pcpp_op_attention) at the
1024^2 SDXL-shaped step's shapes, CUDA events, warm L2 (each shape replayed back to back)."""
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_02962_b200 import pcpp  # noqa: E402


def t_conv(rows, W, Cin, Cout, taps, stride, iters=20):
    pad = 1 if taps == 9 else 0
    x = torch.randn(rows + 2 * pad, 2, W, Cin, device="cuda").bfloat16()
    w = (torch.randn(Cout, taps * Cin, device="cuda") / (taps * Cin) ** 0.5).bfloat16()
    y = torch.empty(rows // stride, 2, W // stride, Cout, device="cuda", dtype=torch.bfloat16)
    b = torch.zeros(Cout, device="cuda")
    for _ in range(3):
        pcpp.pcpp_op_conv(x, rows, 2, W, Cin, taps, stride, w, b, None, None, y, Cout)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        pcpp.pcpp_op_conv(x, rows, 2, W, Cin, taps, stride, w, b, None, None, y, Cout)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    fl = 2.0 * (rows // stride) * 2 * (W // stride) * Cout * taps * Cin
    return ms, fl / ms / 1e9


def t_attn(h, W, C, rows, iters=20):
    q = torch.randn(h, 2, W, C, device="cuda").bfloat16()
    kvs = [torch.randn(r, 2, W, 2 * C, device="cuda").bfloat16() for r in rows]
    o = torch.empty_like(q)
    for _ in range(3):
        pcpp.pcpp_op_attention(q, kvs, list(rows), h, 2, W, C, o)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        pcpp.pcpp_op_attention(q, kvs, list(rows), h, 2, W, C, o)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    fl = 4.0 * h * W * sum(rows) * W * C * 2
    return ms, fl / ms / 1e9


if __name__ == "__main__":
    convs = [("L0 conv 320", 128, 128, 320, 320, 9, 1), ("L0 conv 960->320", 128, 128, 960, 320, 9, 1),
             ("L0 down s2", 128, 128, 320, 320, 9, 2), ("L1 conv 640", 64, 64, 640, 640, 9, 1),
             ("L1 conv 1920->640", 64, 64, 1920, 640, 9, 1), ("L1 qkv", 64, 64, 640, 1920, 1, 1),
             ("L1 proj", 64, 64, 640, 640, 1, 1), ("L2 conv 1280", 32, 32, 1280, 1280, 9, 1),
             ("L2 conv 2560->1280", 32, 32, 2560, 1280, 9, 1), ("L2 qkv", 32, 32, 1280, 3840, 1, 1),
             ("L2 proj", 32, 32, 1280, 1280, 1, 1), ("L1 down s2", 64, 64, 640, 640, 9, 2)]
    for name, *a in convs:
        ms, tf = t_conv(*a)
        print(f"{name:22s} {ms * 1e3:9.1f} us  {tf:7.1f} TF/s")
    for name, *a in [("attn L1 n=1", 64, 64, 640, (64,)), ("attn L2 n=1", 32, 32, 1280, (32,)),
                     ("attn L1 n=8 p=.8", 8, 64, 640, (6, 8, 6)), ("attn L2 n=8", 4, 32, 1280, (3, 4, 3))]:
        ms, tf = t_attn(*a)
        print(f"{name:22s} {ms * 1e3:9.1f} us  {tf:7.1f} TF/s")


def t_gn(rows, W, C, iters=20):
    x = torch.randn(rows, 2, W, C, device="cuda").bfloat16()
    y = torch.empty_like(x)
    g = torch.ones(C, device="cuda"); b = torch.zeros(C, device="cuda")
    m = torch.empty(2, 32, 2, device="cuda", dtype=torch.float64)
    for _ in range(3):
        pcpp.pcpp_op_groupnorm(x, rows, 2, W, C, g, b, 1, y, m)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        pcpp.pcpp_op_groupnorm(x, rows, 2, W, C, g, b, 1, y, m)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    e0.record()
    for _ in range(iters):
        y.copy_(x)
    e1.record()
    torch.cuda.synchronize()
    ms_copy = e0.elapsed_time(e1) / iters
    nb = x.numel() * 2
    return ms, 3 * nb / ms / 1e6, ms_copy, 2 * nb / ms_copy / 1e6


if __name__ == "__main__":
    for shape in [(128, 128, 320), (128, 128, 960), (64, 64, 640), (32, 32, 1280), (32, 32, 2560)]:
        ms, gbs, mc, gc = t_gn(*shape)
        print(f"GN {shape}: {ms * 1e3:7.1f} us ({gbs:6.0f} GB/s of 3x bytes)   torch copy {mc * 1e3:6.1f} us ({gc:6.0f} GB/s)")
