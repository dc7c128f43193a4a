"""Attention kernel timing vs grid size and key count at the level-2 geometry (32x32 tokens per
(b, head), B = 2): separates the per-CTA fixed cost, the per-key-tile cost and wave quantisation."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.bench_ops import t_attn
for heads in (1, 2, 8, 16, 18, 19, 20, 37, 40):
    for rows in ((32,), (16,), (64,)):
        if heads not in (1, 18, 20) and rows != (32,):
            continue
        ms, _ = t_attn(32, 32, 64 * heads, rows)
        ctas = 8 * heads * 2
        print(f"heads={heads:3d} ctas={ctas:4d} kv_rows={sum(rows):3d} key_tiles={sum(rows) * 32 // 128:3d}  {ms * 1e3:8.2f} us", flush=True)
