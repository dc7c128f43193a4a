"""Kernel timing by CUDA-graph replay (no host launch overhead): `reps` launches of one op captured in
a graph, replayed after a warm replay, CUDA events around the replay.  Usage as a module or:
  python tools/graph_timing.py attn-scaling | gemm-scaling"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_02962_b200 import pcpp


def _time_graph(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(2):
            fn(s.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn(s.cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def g_attn(h, W, C, rows, B=2):
    q = torch.randn(h, B, W, C, device="cuda").bfloat16()
    kvs = [torch.randn(r, B, W, 2 * C, device="cuda").bfloat16() for r in rows]
    o = torch.empty_like(q)
    return _time_graph(lambda st: pcpp.pcpp_op_attention(q, kvs, list(rows), h, B, W, C, o, stream=st))


def g_conv(rows, W, Cin, Cout, taps, stride, res=False, B=2, bias=True, temb=False):
    pad = 1 if taps == 9 else 0
    x = torch.randn(rows + 2 * pad, B, W, Cin, device="cuda").bfloat16()
    w = (torch.randn(Cout, taps * Cin, device="cuda") / (taps * Cin) ** 0.5).bfloat16()
    y = torch.empty(rows // stride, B, W // stride, Cout, device="cuda", dtype=torch.bfloat16)
    r = torch.randn_like(y) if res else None
    b = torch.zeros(Cout, device="cuda") if bias else None
    t = torch.zeros(B, Cout, device="cuda") if temb else None
    ms = _time_graph(lambda st: pcpp.pcpp_op_conv(x, rows, B, W, Cin, taps, stride, w, b, t, r, y, Cout, stream=st))
    return ms, 2.0 * (rows // stride) * B * (W // stride) * Cout * taps * Cin / (ms * 1e-3) / 1e12


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "attn-scaling"
    if what == "attn-scaling":
        for heads in (1, 2, 8, 16, 18, 19, 20, 37, 40):
            for rows in ((32,), (16,), (64,)):
                if heads not in (1, 18, 20) and rows != (32,):
                    continue
                ms = g_attn(32, 32, 64 * heads, rows)
                print(f"attn heads={heads:3d} ctas={16 * heads:4d} kv_rows={sum(rows):3d} key_tiles={sum(rows) * 32 // 128:3d}"
                      f"  {ms * 1e3:8.2f} us", flush=True)
        for name, a in (("L1 n=1", (64, 64, 640, (64,))), ("L2 n=1", (32, 32, 1280, (32,))),
                        ("L1 n=8", (8, 64, 640, (6, 8, 6))), ("L2 n=8", (4, 32, 1280, (3, 4, 3)))):
            ms = g_attn(*a)
            h, W, C, rows = a
            ex = h * W * sum(rows) * W * (C // 64) * 2
            print(f"attn {name}  {ms * 1e3:8.2f} us  exp2 {ex / ms / 1e9:6.2f} T/s ({ex / ms / 1e9 / 4.63 * 100:4.1f}% of MUFU)", flush=True)
    else:
        for rows in (4, 8, 16, 32, 64, 128):
            for N, K in ((1280, 1280), (3840, 1280)):
                ms, tf = g_conv(rows, 32, K, N, 1, 1)
                print(f"gemm 1x1 M={rows * 64:5d} N={N} K={K}  {ms * 1e3:8.2f} us  {tf:7.1f} TF/s", flush=True)
        for rows, W, C in ((128, 128, 320), (64, 64, 640), (32, 32, 1280), (4, 32, 1280), (16, 128, 320)):
            ms, tf = g_conv(rows, W, C, C, 9, 1)
            print(f"conv3x3 rows={rows} W={W} C={C}  {ms * 1e3:8.2f} us  {tf:7.1f} TF/s", flush=True)
