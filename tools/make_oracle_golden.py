"""Write the committed oracle golden trajectories (tests/golden/traj_*.npz) -- TEST INFRASTRUCTURE.

Imports only ``oracle/`` (the fp64 CPU implementation written from PAPER.md) and the seeded input
generators of ``paper_2412_02962_b200/inputs.py`` (no method arithmetic).  Nothing here touches
libpcpp: every stored value is the oracle's.  The GPU tests (tests/test_gpu_golden.py) replay the
same seeded inputs through libpcpp and compare per step and on the final latent (north star:
rel-L2 <= 1e-5 fp32, <= 2e-2 bf16).

Cases:
  * X1 (SDXL-shaped 1024^2, 128x128x4 latent) at n in {1, 2, 4, 8}: w = 1 warm-up + 2 async steps of
    the 50-step ladder, p = 0.3 at n = 2, 0.8 at n = 4, 8, bf16 and fp32 weights;
  * SW: X1 at n = 8, p in {0, .125, .25, .5, 1}, w = 1, 2 steps, bf16;
  * SDXL-shaped 32x32 latent at n = 2 (p = 0.3) and n = 8 (p = 0.8): all 50 DDIM steps, w = 4
    (P:173), bf16 and fp32.
Each file stores xs[k] = the gathered latent after step k (float32; the oracle runs in float64 and
float32 storage adds <= 6e-8 relative error), plus the case metadata and a checksum of the inputs.

usage: python tools/make_oracle_golden.py [--only NAME_SUBSTR] [--list]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import model as M            # noqa: E402
from oracle import pcpp as OP            # noqa: E402
from paper_2412_02962_b200 import inputs  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def cases():
    """(name, model, H, n, p, w, S, precision, scheme, max_steps)."""
    c = []
    for prec in ("bf16", "fp32"):
        for n, p in ((1, 0.0), (2, 0.3), (4, 0.8), (8, 0.8)):
            c.append((f"x1_n{n}_{prec}", "sdxl", 128, n, p, 1, 50, prec, "pcpp", 3))
    for p in (0.0, 0.125, 0.25, 0.5, 1.0):
        c.append((f"sw_p{p}_bf16", "sdxl", 128, 8, p, 1, 50, "bf16", "pcpp", 2))
    for prec in ("bf16", "fp32"):
        c.append((f"sdxl32_n2_p0.3_s50_{prec}", "sdxl", 32, 2, 0.3, 4, 50, prec, "pcpp", 50))
        c.append((f"sdxl32_n8_p0.8_s50_{prec}", "sdxl", 32, 8, 0.8, 4, 50, prec, "pcpp", 50))
    return c


def input_digest(blob, xT, cond) -> str:
    h = hashlib.sha256()
    for a in (blob, xT, cond):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--list", action="store_true")
    a = ap.parse_args()
    todo = [c for c in cases() if a.only in c[0]]
    if a.list:
        for c in todo:
            print(c)
        return
    blobs = {}
    for name, model, H, n, p, w, S, prec, scheme, ms in todo:
        path = os.path.join(OUT, f"traj_{name}.npz")
        if os.path.exists(path):
            print("exists:", path)
            continue
        if model not in blobs:
            blobs[model] = inputs.make_weight_blob(M.weight_specs(model))
        blob = blobs[model]
        wts = inputs.round_to_bf16(blob) if prec == "bf16" else blob
        xT = inputs.make_latent(H, H)
        cond = inputs.make_cond(M.arch(model)["temb"])
        cfg = OP.Config(model=model, H=H, W=H, n=n, p=p, warmup=w, steps=S, scheme=scheme)
        t0 = time.time()
        out = OP.sample(cfg, wts, xT, cond, max_steps=ms)
        dt = time.time() - t0
        meta = dict(name=name, model=model, H=H, W=H, n=n, p=p, warmup=w, steps=S, precision=prec,
                    scheme=scheme, max_steps=ms, scheduler="ddim", guidance=5.0,
                    inputs_sha16=input_digest(blob, xT, cond), oracle_seconds=round(dt, 1),
                    modes=out["modes"], generator="tools/make_oracle_golden.py (oracle/ only)")
        np.savez(path, xs=np.stack(out["xs"]).astype(np.float32), meta=json.dumps(meta))
        print(f"wrote {path} ({dt:.1f} s)", flush=True)


if __name__ == "__main__":
    main()
