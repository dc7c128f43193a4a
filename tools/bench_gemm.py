"""Device time of one conv / 1x1 GEMM shape through pcpp_op_conv, launches captured in a CUDA graph
(no host overhead).  PCPP_GEMM_FORCE="bn,splits,pair" pins the configuration (read once per process).
  python tools/bench_gemm.py rows W Cin Cout taps stride [res]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_02962_b200 import pcpp


def run(rows, W, Cin, Cout, taps, stride, res=0, iters=20):
    pad = 1 if taps == 9 else 0
    x = torch.randn(rows + 2 * pad, 2, W, Cin, device="cuda").bfloat16()
    w = (torch.randn(Cout, taps * Cin, device="cuda") / (taps * Cin) ** 0.5).bfloat16()
    y = torch.empty(rows // stride, 2, W // stride, Cout, device="cuda", dtype=torch.bfloat16)
    r = torch.randn_like(y) if res else None
    b = torch.zeros(Cout, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(2):
            pcpp.pcpp_op_conv(x, rows, 2, W, Cin, taps, stride, w, b, None, r, y, Cout, stream=s.cuda_stream)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(iters):
                pcpp.pcpp_op_conv(x, rows, 2, W, Cin, taps, stride, w, b, None, r, y, Cout, stream=s.cuda_stream)
        g.replay(); s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); g.replay(); e1.record(s); s.synchronize()
    ms = e0.elapsed_time(e1) / iters
    fl = 2.0 * (rows // stride) * 2 * (W // stride) * Cout * taps * Cin
    return ms, fl / ms / 1e9


if __name__ == "__main__":
    a = [int(v) for v in sys.argv[1:]]
    ms, tf = run(*a)
    print(f"{os.environ.get('PCPP_GEMM_FORCE', 'heuristic'):12s} {a}: {ms * 1e3:8.1f} us  {tf:7.1f} TF/s")
