"""Network-level pins for the oracle."""
import numpy as np
import pytest

from oracle import model as M
from oracle import pcpp
from oracle.schedule import cfg_combine, ddim_step, ddim_timesteps
from tests import _data
from tests import torch_ref

CASES = {"tiny": (32, 32), "sdxl": (16, 16)}


def _inputs(model, H, W):
    return _data.blob(model), _data.latent(H, W), _data.cond(model)


def test_manifest_consistency():
    for model in ("tiny", "sdxl"):
        blob, xT, c = _inputs(model, *CASES[model])
        P = M.Params(model, blob)
        ctx = M.Ctx(1, 0.0, "sync")
        M.unet(ctx, P, model, [xT[:, :, :]], M.timestep_embedding(P, model, 501, c))
        assert P.used == set(P.t), "every manifest tensor is used exactly by the forward"
        # layer inventory of the SDXL-shaped stack (App. A): 40 conv3x3, 46 GN, 70 attention
        if model == "sdxl":
            assert ctx.count == {"conv": 40, "gn": 46, "attn": 70}


@pytest.mark.parametrize("model", ["tiny", "sdxl"])
def test_P1_one_patch_equals_unpartitioned_network(model):
    H, W = CASES[model]
    blob, xT, c = _inputs(model, H, W)
    P = M.Params(model, blob)
    for tau in (981, 1):
        emb = M.timestep_embedding(P, model, tau, c)
        for mode in ("sync", "async"):
            prev = None
            if mode == "async":       # async with n=1 reads nothing from anyone
                c0 = M.Ctx(1, 0.3, "sync"); M.unet(c0, P, model, [xT], emb); prev = c0.nxt
            ctx = M.Ctx(1, 0.3, mode, prev=prev)
            e = M.unet(ctx, P, model, [xT.astype(np.float64)], emb)[0]
            ref = torch_ref.eps(model, blob, xT, tau, c)
            np.testing.assert_allclose(e, ref, atol=1e-11 * max(1.0, np.abs(ref).max()))
            assert ctx.ledger == []


@pytest.mark.parametrize("n,p,scheme", [(2, 0.25, "pcpp"), (4, 0.5, "pcpp"), (4, 0.0, "fullmap")])
def test_P2_all_sync_equals_single_device(n, p, scheme):
    # w >= S: every step synchronous == single device for every n and p
    cfg1 = pcpp.Config(model="tiny", n=1, p=0.0, warmup=4, steps=4)
    cfgn = pcpp.Config(model="tiny", n=n, p=p, warmup=4, steps=4, scheme=scheme)
    blob, xT, c = _inputs("tiny", 32, 32)
    a = pcpp.sample(cfg1, blob, xT, c)
    b = pcpp.sample(cfgn, blob, xT, c)
    for xa, xb in zip(a["xs"], b["xs"]):
        np.testing.assert_allclose(xb, xa, atol=1e-12 * np.abs(xa).max())


def test_sampler_trajectory_matches_torch_reference_n1():
    # the whole sampler at n=1 against torch eps + an independent CFG/DDIM transcription
    blob, xT, c = _inputs("tiny", 32, 32)
    out = pcpp.sample(pcpp.Config(model="tiny", n=1, p=0.0, warmup=1, steps=4), blob, xT, c)
    x = xT.astype(np.float64)
    for k, tau in enumerate(ddim_timesteps(4)):
        e = torch_ref.eps("tiny", blob, x, tau, c)
        x = ddim_step(x, cfg_combine(e[0], e[1], 5.0), 4, k)
        np.testing.assert_allclose(out["xs"][k], x, atol=1e-11 * np.abs(x).max())


def test_P3_full_conditioning_zero_staleness_n2():
    # n=2, p=1, fresh neighbours: attention sees the full map, halos and GN fresh -> single device
    blob, xT, c = _inputs("tiny", 32, 32)
    cfg = pcpp.Config(model="tiny", n=2, p=1.0)
    e_fresh, _ = pcpp.forward_pair(cfg, blob, xT, 751, c, "fresh", "fresh")
    ref = torch_ref.eps("tiny", blob, xT, 751, c)
    np.testing.assert_allclose(np.concatenate(e_fresh, axis=1), ref, atol=1e-11)
    # negative control: n=4, p=1 misses non-neighbour patches
    e4, _ = pcpp.forward_pair(pcpp.Config(model="tiny", n=4, p=1.0), blob, xT, 751, c, "fresh", "fresh")
    assert np.abs(np.concatenate(e4, axis=1) - ref).max() > 1e-4


@pytest.mark.parametrize("model,n,p", [("tiny", 2, 0.25), ("tiny", 4, 0.5), ("tiny", 4, 0.0),
                                       ("tiny", 2, 1.0), ("sdxl", 4, 0.5), ("sdxl", 2, 0.25)])
def test_P6_time_invariant_input_staleness_plumbing(model, n, p):
    # fresh(x, tau) writes the store; async(x, tau) reading it must reproduce fresh exactly
    H, W = CASES[model]
    blob, xT, c = _inputs(model, H, W)
    e1, e2 = pcpp.forward_pair(pcpp.Config(model=model, n=n, p=p), blob, xT, 501, c, "fresh", "async")
    for a, b in zip(e1, e2):
        np.testing.assert_allclose(b, a, atol=1e-11 * max(1.0, np.abs(a).max()))
    # FULLMAP analogue: a sync pass then an async FULLMAP pass on the same input
    e1, e2 = pcpp.forward_pair(pcpp.Config(model=model, n=n, p=p, scheme="fullmap"),
                               blob, xT, 501, c, "sync", "async")
    for a, b in zip(e1, e2):
        np.testing.assert_allclose(b, a, atol=1e-11 * max(1.0, np.abs(a).max()))


def test_async_differs_from_sync_and_tracks_it():
    # sanity on the default tiny config: stale partial context changes the result, but not wildly
    blob, xT, c = _inputs("tiny", 32, 32)
    a = pcpp.sample(pcpp.Config(), blob, xT, c)
    s = pcpp.sample(pcpp.Config(scheme="sync"), blob, xT, c)
    np.testing.assert_array_equal(a["xs"][0], s["xs"][0])          # step 0 is warm-up
    d = np.linalg.norm(a["x0"] - s["x0"]) / np.linalg.norm(s["x0"])
    assert 1e-6 < d < 0.5
    assert a["modes"] == ["sync", "async", "async", "async"]


# ---- the SDXL transformer block variant ('_xf' models, reading D25/D26) ----------
def test_xf_manifest_consistency_and_sdxl_size():
    blob, xT, c = _inputs("tiny_xf", 32, 32)
    P = M.Params("tiny_xf", blob)
    M.unet(M.Ctx(1, 0.0, "sync"), P, "tiny_xf", [xT], M.timestep_embedding(P, "tiny_xf", 501, c), _data.context("tiny_xf"))
    assert P.used == set(P.t), "every manifest tensor is used exactly by the forward"
    # with SDXL's transformer blocks the SDXL-shaped stack has SDXL's UNet size (2.567 B parameters)
    n = sum(int(np.prod(s)) for _, s, _ in M.manifest("sdxl_xf"))
    assert 2.55e9 < n < 2.58e9, n


def test_xf_requires_context():
    blob, xT, c = _inputs("tiny_xf", 32, 32)
    P = M.Params("tiny_xf", blob)
    with pytest.raises(ValueError):
        M.unet(M.Ctx(1, 0.0, "sync"), P, "tiny_xf", [xT], M.timestep_embedding(P, "tiny_xf", 501, c))


@pytest.mark.parametrize("tau", [981, 1])
def test_P1_xf_one_patch_equals_unpartitioned_network(tau):
    blob, xT, c = _inputs("tiny_xf", 32, 32)
    ctxt = _data.context("tiny_xf")
    P = M.Params("tiny_xf", blob)
    emb = M.timestep_embedding(P, "tiny_xf", tau, c)
    e = M.unet(M.Ctx(1, 0.3, "sync"), P, "tiny_xf", [xT.astype(np.float64)], emb, ctxt)[0]
    ref = torch_ref.eps("tiny_xf", blob, xT, tau, c, ctxt)
    np.testing.assert_allclose(e, ref, atol=1e-11 * max(1.0, np.abs(ref).max()))


@pytest.mark.parametrize("n,p", [(2, 0.25), (4, 0.5)])
def test_P2_P6_xf(n, p):
    blob, xT, c = _inputs("tiny_xf", 32, 32)
    ctxt = _data.context("tiny_xf")
    # P2: all-synchronous n-patch sampling == single device
    a = pcpp.sample(pcpp.Config(model="tiny_xf", n=1, p=0.0, warmup=3, steps=3), blob, xT, c, context=ctxt)
    b = pcpp.sample(pcpp.Config(model="tiny_xf", n=n, p=p, warmup=3, steps=3), blob, xT, c, context=ctxt)
    for xa, xb in zip(a["xs"], b["xs"]):
        np.testing.assert_allclose(xb, xa, atol=1e-12 * np.abs(xa).max())
    # P6: fresh then async on the same input reproduces fresh (the new layers are patch-local)
    e1, e2 = pcpp.forward_pair(pcpp.Config(model="tiny_xf", n=n, p=p), blob, xT, 501, c, "fresh", "async", ctxt)
    for u, v in zip(e1, e2):
        np.testing.assert_allclose(v, u, atol=1e-11 * max(1.0, np.abs(u).max()))
    # P3: n = 2, p = 1, fresh == single device (cross-attention and FF change nothing in the argument)
    if n == 2:
        ef, _ = pcpp.forward_pair(pcpp.Config(model="tiny_xf", n=2, p=1.0), blob, xT, 751, c, "fresh", "fresh", ctxt)
        ref = torch_ref.eps("tiny_xf", blob, xT, 751, c, ctxt)
        np.testing.assert_allclose(np.concatenate(ef, axis=1), ref, atol=1e-11 * max(1.0, np.abs(ref).max()))


def test_timestep_embedding_known_answer():
    """Reading D19 pinned by a hand-derived vector: with lin1 selecting sinusoid entries 32 (cos) and
    64 + 48 (sin) of the tiny model (half = 64, f_j = 10^(-4 j / 64)), lin2 = identity on those two
    units and zero biases, tau = 1000 gives f_32 = 1/100, f_48 = 1/1000, so
    emb = [silu(cos 10), silu(sin 1), 0, ...] for the uncond branch and emb + c for the cond one."""
    import math
    man = M.manifest("tiny")
    blob = np.zeros(sum(int(np.prod(s)) for _, s, _ in man))
    offs, off = {}, 0
    for name, shape, _ in man:
        offs[name] = (off, shape)
        off += int(np.prod(shape))
    o1, (T, S) = offs["time.lin1.w"]
    blob[o1 + 0 * S + 32] = 1.0                 # hidden 0 <- sinusoid[32] = cos(tau f_32)
    blob[o1 + 1 * S + 64 + 48] = 1.0            # hidden 1 <- sinusoid[64 + 48] = sin(tau f_48)
    o2, _ = offs["time.lin2.w"]
    blob[o2 + 0 * T + 0] = 1.0
    blob[o2 + 1 * T + 1] = 1.0
    c = np.zeros(T); c[5] = 2.5
    emb = M.timestep_embedding(M.Params("tiny", blob), "tiny", 1000, c)
    silu = lambda v: v / (1.0 + math.exp(-v))
    want = np.zeros(T); want[0] = silu(math.cos(10.0)); want[1] = silu(math.sin(1.0))
    np.testing.assert_allclose(emb[0], want, atol=1e-13)
    want[5] = 2.5
    np.testing.assert_allclose(emb[1], want, atol=1e-13)
