"""Multi-process worker for the PEER backend test (tests/test_gpu_peer.py) -- run under torchrun.

One process per rank; every rank builds a PCPP_COMM_PEER plan for its own patch, the ranks exchange
their 64-byte IPC arena handles over gloo and connect, then run `steps` pcpp_step calls (warm-up +
async) and one pcpp_sample.  Rank 0 re-runs the same case on the LOOPBACK backend (all n virtual ranks
in one process) and compares: the trajectories must be bitwise identical (same kernels, same data,
only the transport differs).  With --same-gpu every rank uses cuda:0 (the GPU box of the tests has
one GPU: the processes share it, so the pushes are same-device stores through the IPC mappings and
the flag barriers synchronise separate CUDA contexts); otherwise rank r uses cuda:LOCAL_RANK.
Writes a JSON verdict to --out (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="tiny")
    ap.add_argument("--H", type=int, default=32)
    ap.add_argument("--p", type=float, default=0.25)
    ap.add_argument("--w", type=int, default=1)
    ap.add_argument("--S", type=int, default=4)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--precision", default="bf16")
    ap.add_argument("--scheme", default="pcpp")
    ap.add_argument("--same-gpu", action="store_true")
    ap.add_argument("--cfg-split", action="store_true", help="CFG device split: world = 2 x patches")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2412_02962_b200 import inputs, pcpp
    from tests import _data

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = 0 if a.same_gpu else int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    n = world // 2 if a.cfg_split else world
    patch = rank % n
    blob = _data.blob(a.model)
    wts = inputs.round_to_bf16(blob) if a.precision == "bf16" else blob
    cond = _data.cond(a.model)
    xT = np.array(_data.latent(a.H, a.H))
    h = a.H // n

    cfg = pcpp.make_config(model=a.model, num_steps=a.S, precision=a.precision, scheme=a.scheme,
                           backend="peer", rank=rank, world=world, cfg_split=a.cfg_split)
    plan = pcpp.Plan(a.H, a.H, 4, n, a.p, a.w, cfg, wts)
    plan.pcpp_set_cond(cond)
    handles = [None] * world
    dist.all_gather_object(handles, plan.pcpp_peer_handle())
    plan.pcpp_peer_connect(handles)
    lat = torch.from_numpy(np.ascontiguousarray(xT[patch * h:(patch + 1) * h])).cuda()
    xs = []
    for k in range(a.steps):
        plan.pcpp_step(lat, k)
        torch.cuda.synchronize()
        xs.append(lat.cpu().numpy().copy())
    x0 = plan.pcpp_sample(np.ascontiguousarray(xT[patch * h:(patch + 1) * h]), cond) if a.S <= 8 else None
    info = plan.pcpp_query()
    allx = [None] * world
    dist.all_gather_object(allx, (xs, x0))
    plan.close()                          # collective (final barrier before the arenas are unmapped)

    if rank == 0:
        cfg2 = pcpp.make_config(model=a.model, num_steps=a.S, precision=a.precision, scheme=a.scheme,
                                backend="loopback", cfg_split=a.cfg_split)
        lp = pcpp.Plan(a.H, a.H, 4, n, a.p, a.w, cfg2, wts)
        lp.pcpp_set_cond(cond)
        full = torch.from_numpy(xT.copy()).cuda()
        ref = []
        for k in range(a.steps):
            lp.pcpp_step(full, k)
            torch.cuda.synchronize()
            ref.append(full.cpu().numpy().copy())
        ref_x0 = lp.pcpp_sample(xT, cond) if a.S <= 8 else None
        lp.close()
        steps = []
        for k in range(a.steps):
            for br in range(world // n):          # every branch group holds the whole trajectory
                got = np.concatenate([allx[br * n + r][0][k] for r in range(n)], axis=0)
                steps.append(int(np.sum(got != ref[k])))
        res = {"case": vars(a), "mismatches_per_step": steps, "backend": info["backend"], "bytes_eps": info["bytes_eps"],
               "bytes_counted_async": info["bytes_counted_async"],
               "finite": bool(all(np.isfinite(x).all() for x in ref))}
        if ref_x0 is not None:
            res["x0_mismatch_per_rank"] = [int(np.sum(allx[r][1] != ref_x0)) for r in range(world)]
        res["ok"] = all(m == 0 for m in steps) and all(m == 0 for m in res.get("x0_mismatch_per_rank", [0])) \
            and info["backend"] == pcpp.COMM_PEER and res["finite"]
        with open(a.out, "w") as f:
            json.dump(res, f)
        print(json.dumps(res))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
