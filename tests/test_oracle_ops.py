"""Op-level pins for oracle/model.py: special cases that reduce to library
routines (torch.nn.functional, fp64) and closed forms."""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import model as M
from oracle.schedule import band_rows

rng = np.random.default_rng(123)


def _full_to_patches(x, n):
    h = x.shape[1] // n
    return [x[:, i * h:(i + 1) * h].copy() for i in range(n)]


@pytest.mark.parametrize("stride", [1, 2])
@pytest.mark.parametrize("n", [1, 2, 4])
def test_conv3x3_sync_patches_equal_full_conv(n, stride):
    # P5: fresh-halo patch conv == full-image conv (torch conv2d, zero padding 1)
    x = rng.standard_normal((2, 16, 12, 8))
    w = rng.standard_normal((5, 3, 3, 8))
    b = rng.standard_normal(5)
    ctx = M.Ctx(n, 0.5, "sync")
    y = np.concatenate(M.conv3x3(ctx, _full_to_patches(x, n), w, b, stride), axis=1)
    ref = F.conv2d(torch.from_numpy(x).permute(0, 3, 1, 2), torch.from_numpy(w).permute(0, 3, 1, 2),
                   torch.from_numpy(b), stride=stride, padding=1).permute(0, 2, 3, 1).numpy()
    np.testing.assert_allclose(y, ref, atol=1e-12)
    # halo reads: each interior boundary contributes one row per direction (top only for stride 2)
    assert len(ctx.ledger) == (n - 1) * (2 if stride == 1 else 1)


def test_conv_async_uses_stale_rows():
    x_old = rng.standard_normal((2, 8, 6, 4))
    x_new = rng.standard_normal((2, 8, 6, 4))
    w = rng.standard_normal((3, 3, 3, 4)); b = np.zeros(3)
    c0 = M.Ctx(2, 0.5, "sync")
    M.conv3x3(c0, _full_to_patches(x_old, 2), w, b)
    c1 = M.Ctx(2, 0.5, "async", prev=c0.nxt)
    y = M.conv3x3(c1, _full_to_patches(x_new, 2), w, b)
    # the same conv on the hybrid image: rank 0 sees rank 1's stale first row, and v.v.
    hyb0 = np.concatenate([x_new[:, :4], x_old[:, 4:5]], axis=1)
    ref0 = F.conv2d(torch.from_numpy(hyb0).permute(0, 3, 1, 2), torch.from_numpy(w).permute(0, 3, 1, 2),
                    padding=1).permute(0, 2, 3, 1).numpy()[:, :4]
    np.testing.assert_allclose(y[0], ref0, atol=1e-12)
    hyb1 = np.concatenate([x_old[:, 3:4], x_new[:, 4:]], axis=1)
    ref1 = F.conv2d(torch.from_numpy(hyb1).permute(0, 3, 1, 2), torch.from_numpy(w).permute(0, 3, 1, 2),
                    padding=1).permute(0, 2, 3, 1).numpy()[:, 1:]
    np.testing.assert_allclose(y[1], ref1, atol=1e-12)


@pytest.mark.parametrize("act", [False, True])
@pytest.mark.parametrize("n", [1, 2, 4])
def test_groupnorm_sync_equals_full(n, act):
    x = rng.standard_normal((2, 8, 6, 64)) * 3 + 1
    g, b = rng.standard_normal(64), rng.standard_normal(64)
    ctx = M.Ctx(n, 0.5, "sync")
    y = np.concatenate(M.group_norm(ctx, _full_to_patches(x, n), g, b, act), axis=1)
    ref = F.group_norm(torch.from_numpy(x).permute(0, 3, 1, 2), 32, torch.from_numpy(g),
                       torch.from_numpy(b), eps=1e-5)
    if act:
        ref = F.silu(ref)
    np.testing.assert_allclose(y, ref.permute(0, 2, 3, 1).numpy(), atol=1e-12)


def test_groupnorm_corrected_stats_algebra():
    # reading D7: M_hat = M_{t+1} - m_{i,t+1} + m_{i,t}; with rank 1 unchanged between steps,
    # rank 0's corrected stats equal the fresh global stats of the new image exactly
    x_old = rng.standard_normal((2, 8, 4, 64))
    x_new = x_old.copy(); x_new[:, :4] = rng.standard_normal((2, 4, 4, 64)) * 2
    g, b = np.ones(64), np.zeros(64)
    c0 = M.Ctx(2, 0.5, "sync")
    M.group_norm(c0, _full_to_patches(x_old, 2), g, b, False)
    c1 = M.Ctx(2, 0.5, "async", prev=c0.nxt)
    y = M.group_norm(c1, _full_to_patches(x_new, 2), g, b, False)
    ref = F.group_norm(torch.from_numpy(x_new).permute(0, 3, 1, 2), 32, eps=1e-5).permute(0, 2, 3, 1).numpy()
    np.testing.assert_allclose(y[0], ref[:, :4], atol=1e-12)


def _sdpa(x, wq, wk, wv, wo, bo):
    B, H, W, C = x.shape
    t = torch.from_numpy(x.reshape(B, H * W, C))
    q, k, v = t @ torch.from_numpy(wq).T, t @ torch.from_numpy(wk).T, t @ torch.from_numpy(wv).T
    hs = lambda z: z.reshape(B, H * W, C // 64, 64).transpose(1, 2)
    o = F.scaled_dot_product_attention(hs(q), hs(k), hs(v)).transpose(1, 2).reshape(B, H * W, C)
    return (o @ torch.from_numpy(wo).T + torch.from_numpy(bo)).reshape(B, H, W, C).numpy()


def _attn_w(C):
    s = 1 / math.sqrt(C)
    return [rng.standard_normal((C, C)) * s for _ in range(4)] + [rng.standard_normal(C)]


@pytest.mark.parametrize("n", [1, 2, 4])
def test_attention_sync_equals_full_sdpa(n):
    x = rng.standard_normal((2, 8, 4, 128))
    W = _attn_w(128)
    ctx = M.Ctx(n, 0.25, "sync")
    y = np.concatenate(M.attention(ctx, _full_to_patches(x, n), *W), axis=1)
    np.testing.assert_allclose(y, _sdpa(x, *W), atol=1e-12)


def test_attention_p1_fresh_two_patches_equals_full():
    # P3 at op level: n=2, p=1, fresh context covers the whole image
    x = rng.standard_normal((2, 8, 4, 64))
    W = _attn_w(64)
    y = np.concatenate(M.attention(M.Ctx(2, 1.0, "fresh"), _full_to_patches(x, 2), *W), axis=1)
    np.testing.assert_allclose(y, _sdpa(x, *W), atol=1e-12)
    # negative control: n=4, p=1 misses non-adjacent patches
    y4 = np.concatenate(M.attention(M.Ctx(4, 1.0, "fresh"), _full_to_patches(x, 4), *W), axis=1)
    assert np.abs(y4 - _sdpa(x, *W)).max() > 1e-3


def test_attention_p0_is_local_only():
    # P10: p = 0 -> each patch attends to itself only (naive PP)
    x = rng.standard_normal((2, 8, 4, 64))
    W = _attn_w(64)
    c0 = M.Ctx(4, 0.0, "sync"); M.attention(c0, _full_to_patches(x, 4), *W)
    c1 = M.Ctx(4, 0.0, "async", prev=c0.nxt)
    y = M.attention(c1, _full_to_patches(x, 4), *W)
    for i, xi in enumerate(_full_to_patches(x, 4)):
        np.testing.assert_allclose(y[i], _sdpa(xi, *W), atol=1e-12)
    assert c1.ledger == []


def test_attention_closed_forms():
    # P9: all keys equal -> output = mean(V) per head (then W_o, b_o)
    C = 64
    x = rng.standard_normal((1, 4, 4, C))
    wq, wv = rng.standard_normal((C, C)), rng.standard_normal((C, C))
    wk = np.zeros((C, C))                     # every key is 0 -> uniform attention
    eye, zero = np.eye(C), np.zeros(C)
    y = M.attention(M.Ctx(1, 0.0, "sync"), [x], wq, wk, wv, eye, zero)[0]
    v = x.reshape(-1, C) @ wv.T
    np.testing.assert_allclose(y.reshape(-1, C), np.broadcast_to(v.mean(0), (16, C)), atol=1e-12)
    # softmax row closed form: [0, ln 3] -> [0.25, 0.75]; rows sum to 1
    np.testing.assert_allclose(M._softmax_rows(np.array([[0.0, math.log(3.0)]])), [[0.25, 0.75]], atol=1e-15)
    s = M._softmax_rows(np.array([[1000.0, 1000.0, 1000.0]]))
    np.testing.assert_allclose(s, [[1 / 3] * 3], atol=1e-15)


@pytest.mark.parametrize("n,p", [(2, 0.25), (4, 0.5), (4, 1.0), (8, 0.3)])
def test_attention_band_assembly_matches_masked_global_attention(n, p):
    # P4 brute force: PCPP attention == full-image attention with a -inf mask: query rows of
    # patch i see key rows [i h - r, (i+1) h + r) of a hybrid global map whose rows outside
    # patch i come from the previous step's global K/V.
    C, H, W = 64, 16, 3
    h = H // n
    r = band_rows(p, h)
    x_old = rng.standard_normal((2, H, W, C))
    x_new = rng.standard_normal((2, H, W, C))
    wq, wk, wv, wo, bo = _attn_w(C)
    c0 = M.Ctx(n, p, "sync"); M.attention(c0, _full_to_patches(x_old, n), wq, wk, wv, wo, bo)
    c1 = M.Ctx(n, p, "async", prev=c0.nxt)
    y = M.attention(c1, _full_to_patches(x_new, n), wq, wk, wv, wo, bo)
    Ko, Vo = x_old @ wk.T, x_old @ wv.T
    Kn, Vn, Qn = x_new @ wk.T, x_new @ wv.T, x_new @ wq.T
    for i in range(n):
        K, V = Ko.copy(), Vo.copy()
        K[:, i * h:(i + 1) * h], V[:, i * h:(i + 1) * h] = Kn[:, i * h:(i + 1) * h], Vn[:, i * h:(i + 1) * h]
        lo, hi = max(0, i * h - r), min(H, (i + 1) * h + r)
        mask = np.full((h * W, H * W), -np.inf)
        mask[:, lo * W:hi * W] = 0.0
        for b in range(2):
            q = Qn[b, i * h:(i + 1) * h].reshape(-1, C)
            out = np.zeros((h * W, C))
            for hd in range(C // 64):
                sl = slice(hd * 64, hd * 64 + 64)
                s = q[:, sl] @ K[b].reshape(-1, C)[:, sl].T / 8.0 + mask
                s = np.exp(s - s.max(1, keepdims=True)); s /= s.sum(1, keepdims=True)
                out[:, sl] = s @ V[b].reshape(-1, C)[:, sl]
            np.testing.assert_allclose(y[i][b].reshape(-1, C), out @ wo.T + bo, atol=1e-12)


# ---- transformer-block ops of the '_xf' models (reading D25) --------------------------------------
def test_layer_norm_equals_torch_and_closed_forms():
    import torch
    import torch.nn.functional as F
    rng = np.random.default_rng(5)
    x = rng.standard_normal((2, 3, 5, 128)) * 3 + 1
    g, b = rng.standard_normal(128), rng.standard_normal(128)
    y = M.layer_norm([x], g, b)[0]
    ref = F.layer_norm(torch.from_numpy(x), (128,), torch.from_numpy(g), torch.from_numpy(b), eps=1e-5).numpy()
    np.testing.assert_allclose(y, ref, atol=1e-12)
    # gamma = 1, beta = 0: zero mean and (nearly) unit variance per token; a constant token -> beta
    z = M.layer_norm([x], np.ones(128), np.zeros(128))[0]
    np.testing.assert_allclose(z.mean(axis=-1), 0, atol=1e-12)
    np.testing.assert_allclose(z.var(axis=-1), 1 / (1 + 1e-5 / x.var(axis=-1)), rtol=1e-10)
    c = M.layer_norm([np.full((1, 1, 1, 128), 7.0)], g, b)[0]
    np.testing.assert_allclose(c[0, 0, 0], b, atol=1e-12)


def test_cross_attention_equals_sdpa_and_closed_forms():
    import torch
    import torch.nn.functional as F
    rng = np.random.default_rng(6)
    C, D = 128, 32
    x = rng.standard_normal((2, 3, 4, C))
    ctx = rng.standard_normal((2, 77, D))
    wq, wk, wv, wo = (rng.standard_normal(s) / 8 for s in ((C, C), (C, D), (C, D), (C, C)))
    bo = rng.standard_normal(C)
    y = M.cross_attention([x], ctx, wq, wk, wv, wo, bo)[0]
    t = lambda a: torch.from_numpy(a)
    q = (t(x).reshape(2, 12, C) @ t(wq).T).reshape(2, 12, 2, 64).transpose(1, 2)
    k = (t(ctx) @ t(wk).T).reshape(2, 77, 2, 64).transpose(1, 2)
    v = (t(ctx) @ t(wv).T).reshape(2, 77, 2, 64).transpose(1, 2)
    o = F.scaled_dot_product_attention(q, k, v).transpose(1, 2).reshape(2, 12, C) @ t(wo).T + t(bo)
    np.testing.assert_allclose(y, o.reshape(2, 3, 4, C).numpy(), atol=1e-12)
    # identical context tokens -> every query sees mean(V) = that token's value
    same = np.repeat(ctx[:, :1], 77, axis=1)
    y2 = M.cross_attention([x], same, wq, wk, wv, np.eye(C), np.zeros(C))[0]
    np.testing.assert_allclose(y2, np.broadcast_to((same[:, 0] @ wv.T)[:, None, None, :], y2.shape), atol=1e-12)


def test_gelu_geglu_closed_forms():
    import torch
    import torch.nn.functional as F
    x = np.linspace(-6, 6, 121)
    np.testing.assert_allclose(M.gelu(x), F.gelu(torch.from_numpy(x)).numpy(), atol=1e-14)
    assert M.gelu(np.array([0.0]))[0] == 0.0
    np.testing.assert_allclose(M.gelu(np.array([1.0]))[0], 0.8413447460685429, atol=1e-15)  # Phi(1)
    # GEGLU: value half [I; 0], gate half [0; big I] -> FF(x) ~ x * gelu(big * x) ~ relu-gated identity
    C = 4
    w1 = np.zeros((8 * C, C)); w1[:C] = np.eye(C); w1[4 * C:5 * C] = 1e3 * np.eye(C)
    w2 = np.zeros((C, 4 * C)); w2[:, :C] = np.eye(C)
    x = np.array([[[[1.5, -2.0, 0.25, -0.125]]]])
    y = M.geglu_ff([x], w1, np.zeros(8 * C), w2, np.zeros(C))[0]
    np.testing.assert_allclose(y, x * M.gelu(1e3 * x), atol=1e-12)
    np.testing.assert_allclose(y, np.where(x > 0, 1e3 * x * x, 0.0), rtol=1e-12, atol=1e-12)
