"""Multi-process (gloo, CPU) checks of the N > 1 host logic.  The NCCL data path itself needs
several GPUs; what can go wrong on the host is checked here with world_size 2 and 4:
  * every rank's NCCL issue schedule (pcpp_plan_schedule) pairs up: the k-th send a -> b matches
    the k-th recv b <- a (bytes, class, exchange group) -- the tagless in-order matching App. A
     relies on; every all-gather group is issued by all ranks in the same order;
  * the bench plumbing: the 128-byte NCCL id broadcast, patch slicing, max-over-ranks timing.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_02962_b200 import pcpp

CASES = [("sdxl", 128, 0.8, "pcpp"), ("sdxl", 128, 0.3, "fullmap"), ("tiny", 32, 0.25, "pcpp"), ("sdxl", 32, 1.0, "pcpp")]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        # NCCL-id broadcast exactly as bench.py does it (uint8 tensor from rank 0)
        idt = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            idt.copy_(torch.from_numpy(np.frombuffer(np.random.default_rng(5).bytes(128), dtype=np.uint8).copy()))
        dist.broadcast(idt, 0)
        ids = [None] * world
        dist.all_gather_object(ids, bytes(idt.numpy().tobytes()))
        assert all(i == ids[0] for i in ids)
        scheds = {}
        for model, H, p, scheme in CASES:
            cfg = pcpp.make_config(model=model, scheme=scheme, backend="nccl", rank=rank, world=world,
                                   nccl_id=ids[rank])
            for sync in (0, 1):
                scheds[(model, H, p, scheme, sync)] = pcpp.pcpp_plan_schedule(H, H, 4, world, p, 1, cfg, sync)
        allsch = [None] * world
        dist.all_gather_object(allsch, scheds)
        # patch slicing + max-over-ranks timing
        x = np.arange(32 * 8 * 4, dtype=np.float32).reshape(32, 8, 4)
        h = 32 // world
        parts = [None] * world
        dist.all_gather_object(parts, x[rank * h:(rank + 1) * h])
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            assert np.array_equal(np.concatenate(parts, axis=0), x)
            assert t.item() == world
            q.put(("ok", allsch))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("err", repr(e)))


def _check_matching(allsch, world):
    for key in allsch[0]:
        per = [allsch[r][key] for r in range(world)]
        ags = [[(b, c, g) for (op, peer, b, c, g) in s if op == 2] for s in per]
        assert all(a == ags[0] for a in ags), key
        for a in range(world):
            for b in range(world):
                if a == b:
                    continue
                sends = [(by, c, g) for (op, peer, by, c, g) in per[a] if op == 0 and peer == b]
                recvs = [(by, c, g) for (op, peer, by, c, g) in per[b] if op == 1 and peer == a]
                assert sends == recvs, (key, a, b)
                if abs(a - b) > 1:
                    assert not sends, "p2p only between neighbouring patches (§3.2)"


@pytest.mark.parametrize("world", [2, 4])
def test_nccl_schedules_pair_up_across_ranks(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    status, payload = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert status == "ok", payload
    _check_matching(payload, world)
    # async PCPP groups are p2p only; warm-up attention groups are all-gathers
    sch = payload[0][("sdxl", 128, 0.8, "pcpp", 0)]
    assert any(op in (0, 1) and cls == 0 for op, _, _, cls, _ in sch)
    assert not any(op == 2 and cls == 0 for op, _, _, cls, _ in sch)
    warm = payload[0][("sdxl", 128, 0.8, "pcpp", 1)]
    assert any(op == 2 and cls == 0 for op, _, _, cls, _ in warm)
