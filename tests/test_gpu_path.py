"""Whole-path parity: libpcpp (through the C ABI, loopback backend = n virtual ranks on one GPU)
against the fp64 oracle on the same seeded inputs.  Tolerances (north star / SURVEY §8(c)):
rel-L2 <= 1e-5 in fp32 mode and <= 2e-2 in bf16 mode, per step and on the final latent."""
import functools

import numpy as np
import pytest

from oracle import model as M
from oracle import pcpp as OP
from paper_2412_02962_b200 import inputs, pcpp
from tests import _data

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-5, "bf16": 2e-2}


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


@functools.lru_cache(maxsize=None)
def weights(model, precision):
    b = _data.blob(model)
    return inputs.round_to_bf16(b) if precision == "bf16" else b


@functools.lru_cache(maxsize=None)
def oracle_run(model, H, n, p, w, S, precision, scheme, max_steps, scheduler="ddim", noise_seed=0):
    cfg = OP.Config(model=model, H=H, W=H, n=n, p=p, warmup=w, steps=S, scheme=scheme, scheduler=scheduler,
                    noise_seed=noise_seed)
    out = OP.sample(cfg, weights(model, precision), _data.latent(H, H), _data.cond(model), max_steps=max_steps)
    return out["xs"]


def lib_run(model, H, n, p, w, S, precision, scheme, max_steps, kernels="auto", graphs=True, scheduler="ddim",
            noise_seed=0, cfg_split=False):
    import torch
    cfg = pcpp.make_config(model=model, num_steps=S, precision=precision, scheme=scheme, kernels=kernels,
                           graphs=graphs, scheduler=scheduler, noise_seed=noise_seed, cfg_split=cfg_split)
    plan = pcpp.Plan(H, H, 4, n, p, w, cfg, weights(model, precision))
    plan.pcpp_set_cond(_data.cond(model))
    lat = torch.from_numpy(np.array(_data.latent(H, H))).cuda()
    xs = []
    for k in range(max_steps):
        plan.pcpp_step(lat, k)
        torch.cuda.synchronize()
        xs.append(lat.cpu().numpy().copy())
    info = plan.pcpp_query()
    plan.close()
    return xs, info


CASES = [
    # model, H, n, p, w, S, precision, scheme, max_steps
    ("tiny", 32, 2, 0.25, 1, 4, "fp32", "pcpp", 4),      # config T
    ("tiny", 32, 2, 0.25, 1, 4, "bf16", "pcpp", 4),
    ("tiny", 32, 1, 0.25, 0, 4, "fp32", "pcpp", 4),
    ("tiny", 32, 4, 0.5, 1, 4, "fp32", "pcpp", 4),
    ("tiny", 32, 4, 0.0, 1, 4, "fp32", "pcpp", 3),
    ("tiny", 32, 4, 0.5, 2, 4, "fp32", "fullmap", 4),
    ("tiny", 32, 2, 1.0, 1, 4, "fp32", "sync", 3),
    ("tiny", 32, 8, 1.0, 1, 4, "bf16", "pcpp", 3),
    ("sdxl", 32, 2, 0.3, 1, 50, "fp32", "pcpp", 2),
    ("sdxl", 32, 8, 0.8, 1, 50, "bf16", "pcpp", 2),
    ("sdxl", 32, 1, 0.0, 0, 50, "bf16", "pcpp", 2),
    ("sdxl", 32, 4, 0.8, 1, 50, "bf16", "fullmap", 2),            # X2 analogue: DistriFusion-style
]

# config SW analogue: conditioning-fraction sweep at n = 8 (SDXL-shaped, 32x32 latent)
SWEEP = [("sdxl", 32, 8, p, 1, 50, "bf16", "pcpp", 2) for p in (0.0, 0.125, 0.25, 0.5, 1.0)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(map(str, c)))
def test_path_matches_oracle(cuda_ok, case):
    model, H, n, p, w, S, precision, scheme, ms = case
    ref = oracle_run(*case)
    got, info = lib_run(*case)
    errs = [rel_l2(g, r) for g, r in zip(got, ref)]
    print(case, "rel-L2 per step:", ["%.2e" % e for e in errs], "tc:", info["tc_kernels"])
    assert all(e <= TOL[precision] for e in errs), errs


@pytest.mark.parametrize("case", SWEEP, ids=lambda c: f"p{c[3]}")
def test_sweep_cond_fraction_matches_oracle_and_ledger(cuda_ok, case):
    from oracle import ledger
    model, H, n, p, w, S, precision, scheme, ms = case
    ref = oracle_run(*case)
    got, info = lib_run(*case)
    errs = [rel_l2(g, r) for g, r in zip(got, ref)]
    print(case, "rel-L2 per step:", ["%.2e" % e for e in errs])
    assert all(e <= TOL[precision] for e in errs), errs
    want = ledger.physical_bytes(model, H, H, n, p, 2, "pcpp_async")
    assert info["bytes_counted_async"] == [want[c] for c in ("attn", "conv", "gn")]


def test_bf16_simt_and_tc_agree_with_oracle(cuda_ok):
    case = ("tiny", 32, 2, 0.25, 1, 4, "bf16", "pcpp", 4)
    ref = oracle_run(*case)
    for kern in ("simt", "auto"):
        got, _ = lib_run(*case, kernels=kern)
        errs = [rel_l2(g, r) for g, r in zip(got, ref)]
        assert all(e <= TOL["bf16"] for e in errs), (kern, errs)


def test_graph_replay_equals_eager_bitwise(cuda_ok):
    case = ("tiny", 32, 4, 0.5, 1, 4, "bf16", "pcpp", 4)
    a, _ = lib_run(*case, graphs=True)
    b, _ = lib_run(*case, graphs=False)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_step_protocol_errors(cuda_ok):
    import torch
    cfg = pcpp.make_config(model="tiny", num_steps=4, precision="bf16")
    plan = pcpp.Plan(32, 32, 4, 2, 0.25, 1, cfg, weights("tiny", "bf16"))
    plan.pcpp_set_cond(_data.cond("tiny"))
    lat = torch.zeros(32, 32, 4, device="cuda")
    with pytest.raises(pcpp.PcppError) as e:
        plan.pcpp_step(lat, 1)                   # must start at k = 0
    assert e.value.status == pcpp.ERR_STATE
    for k in range(4):
        plan.pcpp_step(lat, k)
    with pytest.raises(pcpp.PcppError):
        plan.pcpp_step(lat, 4)                   # past the last step
    plan.pcpp_reset()
    plan.pcpp_step(lat, 0)
    torch.cuda.synchronize()
    plan.close()


def test_sample_e2e_host_buffers(cuda_ok):
    case = ("tiny", 32, 2, 0.25, 1, 4, "bf16", "pcpp", 4)
    cfg = pcpp.make_config(model="tiny", num_steps=4, precision="bf16")
    plan = pcpp.Plan(32, 32, 4, 2, 0.25, 1, cfg, weights("tiny", "bf16"))
    x0 = plan.pcpp_sample(np.array(_data.latent(32, 32)), np.array(_data.cond("tiny")))
    x0b = plan.pcpp_sample(np.array(_data.latent(32, 32)), np.array(_data.cond("tiny")))
    plan.close()
    np.testing.assert_array_equal(x0, x0b)       # deterministic, reset works
    assert rel_l2(x0, oracle_run(*case)[-1]) <= TOL["bf16"]


@pytest.mark.parametrize("force", ["160,1,1", "128,1,1", "256,1,1", "160,1,0", "64,1,0", "128,3,0", "160,1,2", "128,1,4",
                                   "64,1,4"])
def test_forced_gemm_configs(cuda_ok, force, tmp_path):
    """Every tcgen05 GEMM variant the autotuner can pick (1-CTA / 2-CTA pair, BN, split-K through the
    fp32 workspace, cluster split-K through DSMEM (pair = 2 / 4), with and without the fused GroupNorm
    statistics) reproduces the oracle on the SDXL-shaped stack."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "xs.npy"
    env = dict(os.environ, PCPP_GEMM_FORCE=force)
    r = subprocess.run([sys.executable, "-m", "tests._force_run", str(out)], cwd=root, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    xs = np.load(out)
    ref = oracle_run("sdxl", 32, 1, 0.0, 0, 50, "bf16", "pcpp", 2)
    for k in range(2):
        assert rel_l2(xs[k], ref[k]) <= TOL["bf16"], (force, k)


DPM_CASES = [("tiny", 32, 2, 0.25, 1, 4, "fp32", "pcpp", 4), ("tiny", 32, 2, 0.25, 1, 4, "bf16", "pcpp", 4),
             ("sdxl", 32, 2, 0.3, 1, 50, "bf16", "pcpp", 3)]


@pytest.mark.parametrize("case", DPM_CASES, ids=lambda c: "-".join(map(str, c)))
def test_dpmpp2m_path_matches_oracle(cuda_ok, case):
    """The DPM-Solver++(2M) scheduler (north star "DDIM/DPM-solver", reading D23), fused with CFG in
    one elementwise kernel with its x0 history per patch, follows the oracle step by step (k = 0 is
    first order, later steps use the history)."""
    xs, _ = lib_run(*case, scheduler="dpmpp2m")
    ref = oracle_run(*case, scheduler="dpmpp2m")
    tol = TOL[case[6]]
    for k, (a, b) in enumerate(zip(xs, ref)):
        assert rel_l2(a, b) <= tol, (k, rel_l2(a, b))
    # and it is a different sampler: from step 1 on the DDIM trajectory is far further from the
    # result than the GPU's own error
    ddim = oracle_run(*case)
    k = len(xs) - 1
    assert rel_l2(ref[k], ddim[k]) > 3 * rel_l2(xs[k], ref[k])


@pytest.mark.parametrize("case", DPM_CASES, ids=lambda c: "-".join(map(str, c)))
def test_ancestral_path_matches_oracle(cuda_ok, case):
    """The ancestral sampler (Eq. 3-4 on the ladder, reading D24): the kernel's Philox4x64-10 +
    Box-Muller noise for each global latent token and step equals the oracle's, so the stochastic
    trajectories agree step by step; another seed gives another trajectory."""
    xs, _ = lib_run(*case, scheduler="ancestral", noise_seed=11)
    ref = oracle_run(*case, scheduler="ancestral", noise_seed=11)
    tol = TOL[case[6]]
    for k, (a, b) in enumerate(zip(xs, ref)):
        assert rel_l2(a, b) <= tol, (k, rel_l2(a, b))
    other = oracle_run(*case, scheduler="ancestral", noise_seed=12)
    assert rel_l2(ref[0], other[0]) > 3 * rel_l2(xs[0], ref[0])


def test_nccl_config_with_one_patch_runs_the_local_path(cuda_ok):
    """A one-patch plan configured for NCCL has no neighbour: the library runs it on the local
    (loopback) path -- no communicator, no exchange -- and says so in pcpp_query.backend; the sample is
    bitwise the loopback plan's.  (The multi-process exchange itself is tests/test_gpu_peer.py; the
    NCCL send/recv realisation needs >= 2 GPUs, which the in-round GPU box does not have.)"""
    import torch
    blob = weights("tiny", "bf16")
    cond = _data.cond("tiny")
    xT = np.array(_data.latent(32, 32), dtype=np.float32)          # writable copy
    outs = []
    for backend in ("loopback", "nccl"):
        kw = {}
        if backend == "nccl":
            kw = dict(rank=0, world=1, nccl_id=pcpp.pcpp_get_unique_id())
        cfg = pcpp.make_config(model="tiny", num_steps=4, precision="bf16", backend=backend, **kw)
        plan = pcpp.Plan(32, 32, 4, 1, 0.0, 0, cfg, blob)
        x0 = torch.empty((32, 32, 4), dtype=torch.float32).pin_memory()
        xt = torch.from_numpy(xT).pin_memory()
        ch = torch.from_numpy(np.ascontiguousarray(cond, dtype=np.float32)).pin_memory()
        plan.pcpp_sample_into(xt.data_ptr(), ch.data_ptr(), x0.data_ptr())
        outs.append(x0.numpy().copy())
        assert plan.pcpp_query()["backend"] == pcpp.COMM_LOOPBACK
        plan.close()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("case", [("tiny", 32, 2, 0.25, 1, 4, "bf16", "pcpp", 4), ("tiny", 32, 4, 0.5, 1, 4, "fp32", "pcpp", 4),
                                  ("tiny", 32, 4, 0.5, 2, 4, "bf16", "fullmap", 4)], ids=lambda c: "-".join(map(str, c)))
@pytest.mark.parametrize("delay", ["0", "60"])
def test_async_exchange_protocol_bitwise(cuda_ok, case, delay):
    """SURVEY §4.6 race / ordering check on one GPU: with PCPP_LOOPBACK_ASYNC the exchanges run on the
    comm stream with the NCCL backend's event protocol (issued behind the producer, consumed one step
    later, parity buffers, fork / join in the captured step graph), optionally behind an injected
    per-exchange delay of 60-300 k cycles; the trajectory is bitwise the synchronous loopback's."""
    import os
    ref, _ = lib_run(*case)
    os.environ["PCPP_LOOPBACK_ASYNC"] = "1"
    os.environ["PCPP_XCH_DELAY"] = delay
    try:
        got, _ = lib_run(*case)
    finally:
        del os.environ["PCPP_LOOPBACK_ASYNC"]
        del os.environ["PCPP_XCH_DELAY"]
    for k, (a, b) in enumerate(zip(got, ref)):
        assert np.array_equal(a, b), k


@pytest.mark.gpu
def test_comm_off_debug_mode(cuda_ok):
    """SURVEY §8(d) COMM_OFF: warm-up steps are unchanged, async steps skip the exchange (so the
    trajectory departs from the method's -- proving the switch removes the transfers), and switching
    it back off after a reset restores the method's trajectory bitwise."""
    import torch
    model, H, n, p, w, S = "tiny", 32, 4, 0.5, 1, 4
    ref, _ = lib_run(model, H, n, p, w, S, "fp32", "pcpp", 4)
    cfg = pcpp.make_config(model=model, num_steps=S, precision="fp32", scheme="pcpp")
    plan = pcpp.Plan(H, H, 4, n, p, w, cfg, weights(model, "fp32"))
    plan.pcpp_set_cond(_data.cond(model))

    def traj():
        lat = torch.from_numpy(np.array(_data.latent(H, H))).cuda()
        plan.pcpp_reset()
        xs = []
        for k in range(4):
            plan.pcpp_step(lat, k)
            torch.cuda.synchronize()
            xs.append(lat.cpu().numpy().copy())
        return xs

    plan.pcpp_debug_comm_off(True)
    off = traj()
    plan.pcpp_debug_comm_off(False)
    back = traj()
    plan.close()
    assert np.array_equal(off[0], ref[0])                # warm-up step still exchanges
    assert not np.array_equal(off[2], ref[2])            # async steps read older stale bands
    for k in range(4):
        assert np.array_equal(back[k], ref[k]), k


# CFG device split (§2.2): 2 x n virtual ranks, branch b over the n patches as
# batch 1, eps swapped between partners every step.  Same arithmetic as batch 2 per rank (reading
# D27), so the oracle of the same (n, p) is the reference.
SPLIT = [
    ("tiny", 32, 1, 0.0, 0, 4, "fp32", "pcpp", 4),
    ("tiny", 32, 2, 0.25, 1, 4, "fp32", "pcpp", 4),
    ("tiny", 32, 4, 0.5, 1, 4, "bf16", "pcpp", 3),
    ("tiny", 32, 2, 0.5, 1, 4, "fp32", "fullmap", 3),
    ("sdxl", 32, 2, 0.3, 1, 50, "bf16", "pcpp", 3),
    ("sdxl", 32, 4, 0.8, 1, 50, "bf16", "pcpp", 3),
    ("sdxl", 32, 2, 0.3, 1, 50, "fp32", "pcpp", 2),
]


@pytest.mark.parametrize("case", SPLIT, ids=lambda c: "-".join(map(str, c)))
def test_cfg_split_matches_oracle(cuda_ok, case):
    ref = oracle_run(*case)
    got, info = lib_run(*case, cfg_split=True)
    errs = [rel_l2(g, r) for g, r in zip(got, ref)]
    print(case, "cfg_split rel-L2 per step:", ["%.2e" % e for e in errs])
    assert all(e <= TOL[case[6]] for e in errs), errs
    n, H = case[2], case[1]
    assert info["bytes_eps"] == 2 * n * (H // n) * H * 16
    assert info["simt_fallbacks"] == 0
