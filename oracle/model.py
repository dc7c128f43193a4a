"""Denoiser stacks and the patch-parallel layer rules -- TEST INFRASTRUCTURE ONLY.

The paper runs SDXL's U-Net (§4; "U-Net ... with attention modules",
P:17 §2.1).  No checkpoint exists offline, so (reading D18) the stack is the
SDXL-shaped random-init topology of SURVEY.md App. A:

  RB(a->b) = GN(a) -> SiLU -> conv3x3(a->b) + bias + temb_b
             -> GN(b) -> SiLU -> conv3x3(b->b)  (+ skip: x, or 1x1(a->b) if a != b)
  AS(C, d) = GN(C) -> proj_in -> d x [h <- h + W_o MHSA(h)] -> proj_out -> + input

with 70 self-attention layers, 40 conv3x3, 46 GroupNorms (the counts that
reproduce Table 1).  TINY is the config-T toy stack.

Layer rules across patches (§3.3), per rank i of n, step t:
  * attention: Q from the local fresh patch only; K/V =
      [lower r rows of i-1 ; local ; upper r rows of i+1], the neighbour rows
      stale from step t+1 (Eq. 1), r = band_rows(p, h_l) at that
      layer's resolution (reading D3).  Warm-up: full fresh map (D10).
      FULLMAP (DistriFusion): all other ranks' stale K/V.
  * GroupNorm ("same approach in DistriFusion"; reading D7): fresh local
      sums m_i, stale global sums M:  M_hat = M_{t+1} - m_{i,t+1} + m_{i,t}.
  * conv3x3 ("leave the AllGather ... as it is"; reading D8): 1-row halos
      of the conv input from the neighbours, stale from step t+1; zero padding
      at true image borders.
  * everything else is patch-local.

Modes: 'sync' = warm-up / exact single-device semantics (fresh neighbours,
full-map attention); 'async' = the stale PCPP (or FULLMAP) rules above;
'fresh' = debug mode for pin P6: partial bands / halos / GN sums taken fresh
from this pass.

Weight layouts (one flat float32 blob, manifest order):
  conv  [Cout, 3, 3, Cin]   (tap-major, Cin innermost)
  lin   [out, in]
  vectors [C]

Pins: tests/test_oracle_model.py (n=1 vs an independent torch.nn.functional
forward; all-sync vs single device for any n, p; fresh-vs-async invariant P6;
masked full-image attention brute force P4; op-level conv/GN/SDPA vs torch).
"""
from __future__ import annotations

import math

import numpy as np

from .schedule import band_rows

G_GROUPS = 32
GN_EPS = 1e-5
LN_EPS = 1e-5
HEAD_DIM = 64


def _erf(x):
    from scipy.special import erf       # library primitive (the error function)
    return erf(x)

# ----------------------------------------------------------------------------
# Architecture description
# ----------------------------------------------------------------------------


CTX_LEN = 77          # text tokens of the cross-attention context (SDXL's CLIP length; reading D26)


def arch(model: str) -> dict:
    """Channel widths / depths.  SDXL: App. A; TINY: config T.  The '_xf' variants
     replace each attention layer of an AS stack by SDXL's full transformer block
    (LayerNorm, self-attention, LayerNorm, cross-attention to a 77-token context, LayerNorm, GEGLU
    feed-forward; reading D25), with a context of dimension ctx_dim (SDXL 2048)."""
    base, xf = (model[:-3], True) if model.endswith("_xf") else (model, False)
    if base == "sdxl":
        return dict(model=model, base=base, xf=xf, C0=320, chans=[320, 640, 1280], depth=[0, 2, 10],
                    temb=1280, sin_dim=320, levels=3, ctx_dim=2048)
    if base == "tiny":
        return dict(model=model, base=base, xf=xf, C0=128, chans=[128], depth=[1], temb=512,
                    sin_dim=128, levels=1, ctx_dim=256)
    raise ValueError(model)


def _rb_specs(pre, cin, cout, T):
    s = [(f"{pre}.gn1.g", (cin,), "gamma"), (f"{pre}.gn1.b", (cin,), "beta"),
         (f"{pre}.conv1.w", (cout, 3, 3, cin), "conv"), (f"{pre}.conv1.b", (cout,), "bias"),
         (f"{pre}.temb.w", (cout, T), "lin"), (f"{pre}.temb.b", (cout,), "bias"),
         (f"{pre}.gn2.g", (cout,), "gamma"), (f"{pre}.gn2.b", (cout,), "beta"),
         (f"{pre}.conv2.w", (cout, 3, 3, cout), "conv_res"), (f"{pre}.conv2.b", (cout,), "bias")]
    if cin != cout:
        s += [(f"{pre}.skip.w", (cout, cin), "lin"), (f"{pre}.skip.b", (cout,), "bias")]
    return s


def _as_specs(pre, C, depth, xf=False, ctx_dim=0):
    s = [(f"{pre}.gn.g", (C,), "gamma"), (f"{pre}.gn.b", (C,), "beta"),
         (f"{pre}.proj_in.w", (C, C), "lin"), (f"{pre}.proj_in.b", (C,), "bias")]
    for d in range(depth):
        a = f"{pre}.attn{d}"
        if xf:
            s += [(f"{a}.ln1.g", (C,), "gamma"), (f"{a}.ln1.b", (C,), "beta")]
        s += [(f"{a}.wq", (C, C), "lin"), (f"{a}.wk", (C, C), "lin"),
              (f"{a}.wv", (C, C), "lin"), (f"{a}.wo", (C, C), f"lin_res{depth}"),
              (f"{a}.bo", (C,), "bias")]
        if xf:   # reading D25: cross-attention (no q/k/v bias, as SDXL) and the GEGLU feed-forward
            s += [(f"{a}.ln2.g", (C,), "gamma"), (f"{a}.ln2.b", (C,), "beta"),
                  (f"{a}.xq", (C, C), "lin"), (f"{a}.xk", (C, ctx_dim), "lin"), (f"{a}.xv", (C, ctx_dim), "lin"),
                  (f"{a}.xo", (C, C), f"lin_res{depth}"), (f"{a}.xbo", (C,), "bias"),
                  (f"{a}.ln3.g", (C,), "gamma"), (f"{a}.ln3.b", (C,), "beta"),
                  (f"{a}.ff1.w", (8 * C, C), "lin"), (f"{a}.ff1.b", (8 * C,), "bias"),
                  (f"{a}.ff2.w", (C, 4 * C), f"lin_res{depth}"), (f"{a}.ff2.b", (C,), "bias")]
    s += [(f"{pre}.proj_out.w", (C, C), "lin_res1"), (f"{pre}.proj_out.b", (C,), "bias")]
    return s


def _blocks(model: str):
    """The forward program as a list of block records, in forward order.

    Each record: (kind, prefix, args).  Used by both manifest() and unet().
    kinds: conv_in, rb, as, down, up, out, push (skip), pop (skip concat).
    """
    a = arch(model)
    C = a["chans"]
    B = []
    if a["base"] == "tiny":
        B.append(("conv_in", "conv_in", (4, C[0])))
        for j in range(2):
            B.append(("rb", f"blk{j}.rb", (C[0], C[0])))
            B.append(("as", f"blk{j}.as", (C[0], a["depth"][0])))
        B.append(("out", "out", (C[0],)))
        return B
    # SDXL-shaped (App. A)
    B.append(("conv_in", "conv_in", (4, C[0])))
    B.append(("push", None, (C[0],)))
    cin = C[0]
    for lvl in range(3):
        for j in range(2):
            B.append(("rb", f"down{lvl}.{j}.rb", (cin, C[lvl])))
            cin = C[lvl]
            if a["depth"][lvl]:
                B.append(("as", f"down{lvl}.{j}.as", (C[lvl], a["depth"][lvl])))
            B.append(("push", None, (C[lvl],)))
        if lvl < 2:
            B.append(("down", f"down{lvl}.ds", (C[lvl],)))
            B.append(("push", None, (C[lvl],)))
    B.append(("rb", "mid.rb0", (C[2], C[2])))
    B.append(("as", "mid.as", (C[2], a["depth"][2])))
    B.append(("rb", "mid.rb1", (C[2], C[2])))
    # skip channel stack, to know concat widths
    stack = [C[0], C[0], C[0], C[0], C[1], C[1], C[1], C[2], C[2]]
    cur = C[2]
    for lvl in (2, 1, 0):
        for j in range(3):
            sk = stack.pop()
            B.append(("pop", None, (sk,)))
            B.append(("rb", f"up{lvl}.{j}.rb", (cur + sk, C[lvl])))
            cur = C[lvl]
            if a["depth"][lvl]:
                B.append(("as", f"up{lvl}.{j}.as", (C[lvl], a["depth"][lvl])))
        if lvl > 0:
            B.append(("up", f"up{lvl}.us", (C[lvl],)))
    B.append(("out", "out", (C[0],)))
    return B


def manifest(model: str) -> list[tuple[str, tuple, str]]:
    """Ordered (name, shape, kind) list of every parameter, forward order."""
    a = arch(model)
    T, S = a["temb"], a["sin_dim"]
    m = [("time.lin1.w", (T, S), "lin"), ("time.lin1.b", (T,), "bias"),
         ("time.lin2.w", (T, T), "lin"), ("time.lin2.b", (T,), "bias")]
    for kind, pre, args in _blocks(model):
        if kind == "conv_in":
            cin, cout = args
            m += [("conv_in.w", (cout, 3, 3, cin), "conv"), ("conv_in.b", (cout,), "bias")]
        elif kind == "rb":
            m += _rb_specs(pre, args[0], args[1], T)
        elif kind == "as":
            m += _as_specs(pre, args[0], args[1], a["xf"], a["ctx_dim"])
        elif kind in ("down", "up"):
            c = args[0]
            m += [(f"{pre}.conv.w", (c, 3, 3, c), "conv"), (f"{pre}.conv.b", (c,), "bias")]
        elif kind == "out":
            c = args[0]
            m += [("out.gn.g", (c,), "gamma"), ("out.gn.b", (c,), "beta"),
                  ("conv_out.w", (4, 3, 3, c), "conv"), ("conv_out.b", (4,), "bias")]
    return m


def init_spec(shape, kind) -> tuple[int, float, float]:
    """(numel, mean, std) for the seeded generator -- reading D17."""
    n = int(np.prod(shape))
    if kind == "gamma":
        return n, 1.0, 0.1
    if kind in ("beta", "bias"):
        return n, 0.0, 0.1
    if kind == "conv":
        return n, 0.0, 1.0 / math.sqrt(9 * shape[3])
    if kind == "conv_res":
        return n, 0.0, 1.0 / math.sqrt(9 * shape[3]) / math.sqrt(2.0)
    if kind == "lin":
        return n, 0.0, 1.0 / math.sqrt(shape[1])
    if kind.startswith("lin_res"):
        d = int(kind[len("lin_res"):])
        return n, 0.0, 1.0 / math.sqrt(shape[1]) / math.sqrt(2.0 * d)
    raise ValueError(kind)


def weight_specs(model: str):
    return [init_spec(shape, kind) for _, shape, kind in manifest(model)]


# (The same rule, derived from names/shapes only, lives in paper_2412_02962_b200/inputs.py
#  for callers that hold the library's manifest; tests/test_abi.py checks the two agree.)


class Params:
    """Name -> float64 array view over the flat blob (manifest order)."""

    def __init__(self, model: str, blob: np.ndarray):
        blob = np.asarray(blob, dtype=np.float64)
        self.t = {}
        off = 0
        for name, shape, _ in manifest(model):
            n = int(np.prod(shape))
            self.t[name] = blob[off:off + n].reshape(shape)
            off += n
        if off != blob.size:
            raise ValueError(f"blob has {blob.size} values, manifest needs {off}")
        self.used = set()

    def __call__(self, name):
        self.used.add(name)
        return self.t[name]


# ----------------------------------------------------------------------------
# The cross-patch context: what each rank may read from its neighbours
# ----------------------------------------------------------------------------


class Ctx:
    """n simulated ranks at one step.

    prev: the stale store written by the previous step (layer id -> data);
    nxt : the store this step writes (written in every mode, so the first async
          step reads the last warm-up step).
    ledger: (kind, lid, src, dst, elements) for every datum a rank reads from
          another rank -- the counted communication ledger.
    """

    def __init__(self, n: int, p: float, mode: str, scheme: str = "pcpp", prev=None):
        assert mode in ("sync", "async", "fresh")
        assert scheme in ("pcpp", "fullmap")
        self.n, self.p, self.mode, self.scheme = n, p, mode, scheme
        self.prev = prev if prev is not None else {}
        self.nxt = {}
        self.count = {"conv": 0, "gn": 0, "attn": 0}
        self.ledger = []

    def lid(self, kind):
        i = self.count[kind]
        self.count[kind] += 1
        return f"{kind}{i}"

    def read(self, kind, lid, src, dst, elems):
        if src != dst and elems > 0:
            self.ledger.append((kind, lid, src, dst, int(elems)))


# ----------------------------------------------------------------------------
# Layer ops over lists of patches xs[i]: float64 [B, h, W, C]
# ----------------------------------------------------------------------------


def silu(x):
    return x / (1.0 + np.exp(-x))


def conv3x3(ctx: Ctx, xs, w, b, stride=1):
    """3x3 conv, padding 1, on each rank's patch with 1-row halos (reading D8).

    Halos: top from rank i-1's last input row, bottom from rank i+1's first
    row; zeros at the true image border.  'sync'/'fresh' take this step's rows,
    'async' the stored rows of step t+1.  A stride-2 conv needs only the top
    halo: output row o reads input rows 2o-1, 2o, 2o+1.
    w: [Cout, 3, 3, Cin].
    """
    n = ctx.n
    lid = ctx.lid("conv")
    for i, x in enumerate(xs):
        ctx.nxt[(lid, i)] = {"top": x[:, 0].copy(), "bot": x[:, -1].copy()}
    out = []
    for i, x in enumerate(xs):
        Bn, h, W, Cin = x.shape
        zero = np.zeros((Bn, W, Cin))
        if i == 0:
            top = zero
        else:
            top = xs[i - 1][:, -1] if ctx.mode in ("sync", "fresh") else ctx.prev[(lid, i - 1)]["bot"]
            ctx.read("conv", lid, i - 1, i, top.size)
        if i == n - 1 or stride == 2:
            bot = zero
        else:
            bot = xs[i + 1][:, 0] if ctx.mode in ("sync", "fresh") else ctx.prev[(lid, i + 1)]["top"]
            ctx.read("conv", lid, i + 1, i, bot.size)
        xp = np.concatenate([top[:, None], x, bot[:, None]], axis=1)      # rows -1..h
        xp = np.pad(xp, ((0, 0), (0, 0), (1, 1), (0, 0)))                 # cols -1..W
        ho, wo = h // stride, W // stride
        y = np.zeros((Bn, ho, wo, w.shape[0]))
        for dr in range(3):
            for dw in range(3):
                patch = xp[:, dr:dr + stride * ho:stride, dw:dw + stride * wo:stride, :]
                y += patch @ w[:, dr, dw, :].T
        out.append(y + b)
    return out


def group_norm(ctx: Ctx, xs, gamma, beta, act: bool):
    """GroupNorm(32) with fresh local + stale global statistics (reading D7).

    m_i = (sum x, sum x^2) per (batch, group) over rank i's patch;
    sync/fresh: M = sum_j m_j (this step); async: M_hat = M_{t+1} - m_{i,t+1} + m_i.
    mu = M1/N, var = max(M2/N - mu^2, 0), N = H_l W_l C/G (global count);
    y = gamma (x - mu)/sqrt(var + eps) + beta, then SiLU if act.
    """
    n = ctx.n
    lid = ctx.lid("gn")
    Bn, h, W, C = xs[0].shape
    cg = C // G_GROUPS
    ms = []
    for x in xs:
        xg = x.reshape(Bn, h * W, G_GROUPS, cg)
        ms.append(np.stack([xg.sum(axis=(1, 3)), (xg * xg).sum(axis=(1, 3))], axis=-1))  # [B,G,2]
    M_fresh = np.zeros_like(ms[0])
    for j in range(n):                       # rank order
        M_fresh = M_fresh + ms[j]
    ctx.nxt[(lid, "m")] = [m.copy() for m in ms]
    ctx.nxt[(lid, "M")] = M_fresh.copy()
    Ncount = n * h * W * cg
    out = []
    for i, x in enumerate(xs):
        for j in range(n):
            ctx.read("gn", lid, j, i, ms[j].size)
        if ctx.mode in ("sync", "fresh") or n == 1:
            # n = 1: M_{t+1} - m_{0,t+1} + m_0 = m_0 = M_fresh exactly (no other rank exists)
            M = M_fresh
        else:
            M = ctx.prev[(lid, "M")] - ctx.prev[(lid, "m")][i] + ms[i]
        mu = M[..., 0] / Ncount                                   # [B, G]
        var = np.maximum(M[..., 1] / Ncount - mu * mu, 0.0)
        rstd = 1.0 / np.sqrt(var + GN_EPS)
        xg = x.reshape(Bn, h, W, G_GROUPS, cg)
        y = (xg - mu[:, None, None, :, None]) * rstd[:, None, None, :, None]
        y = y.reshape(Bn, h, W, C) * gamma + beta
        out.append(silu(y) if act else y)
    return out


def _softmax_rows(s):
    s = s - s.max(axis=-1, keepdims=True)
    e = np.exp(s)
    return e / e.sum(axis=-1, keepdims=True)


def attention(ctx: Ctx, hs, wq, wk, wv, wo, bo):
    """Partially conditioned multi-head self-attention (§3.3; Fig. 3).

    Q from the local patch; K/V context in token order [top band; local;
    bottom band] (reading D13).  heads = C/64, scale 1/sqrt(64) (reading D12).
    Returns W_o O + b_o (the caller adds the residual).
    """
    n, p = ctx.n, ctx.p
    lid = ctx.lid("attn")
    Bn, h, W, C = hs[0].shape
    r = band_rows(p, h)
    qs = [x @ wq.T for x in hs]
    ks = [x @ wk.T for x in hs]
    vs = [x @ wv.T for x in hs]
    for i in range(n):
        ctx.nxt[(lid, i)] = {"k": ks[i].copy(), "v": vs[i].copy()}
    out = []
    for i in range(n):
        blocks_k, blocks_v = [], []
        if ctx.mode == "sync":
            for j in range(n):
                blocks_k.append(ks[j]); blocks_v.append(vs[j])
                ctx.read("attn", lid, j, i, ks[j].size + vs[j].size)
        elif ctx.mode == "async" and ctx.scheme == "fullmap":
            for j in range(n):
                if j == i:
                    kj, vj = ks[i], vs[i]
                else:
                    kj, vj = ctx.prev[(lid, j)]["k"], ctx.prev[(lid, j)]["v"]
                    ctx.read("attn", lid, j, i, kj.size + vj.size)
                blocks_k.append(kj); blocks_v.append(vj)
        else:  # pcpp async (stale bands) or fresh (fresh bands)
            src = (lambda j: {"k": ks[j], "v": vs[j]}) if ctx.mode == "fresh" else \
                  (lambda j: ctx.prev[(lid, j)])
            if i > 0 and r > 0:
                d = src(i - 1)
                blocks_k.append(d["k"][:, h - r:]); blocks_v.append(d["v"][:, h - r:])
                ctx.read("attn", lid, i - 1, i, 2 * d["k"][:, h - r:].size)
            blocks_k.append(ks[i]); blocks_v.append(vs[i])
            if i < n - 1 and r > 0:
                d = src(i + 1)
                blocks_k.append(d["k"][:, :r]); blocks_v.append(d["v"][:, :r])
                ctx.read("attn", lid, i + 1, i, 2 * d["k"][:, :r].size)
        K = np.concatenate(blocks_k, axis=1)
        V = np.concatenate(blocks_v, axis=1)
        Q = qs[i]
        nq, nk = h * W, K.shape[1] * W
        O = np.zeros((Bn, nq, C))
        for bb in range(Bn):
            q = Q[bb].reshape(nq, C)
            k = K[bb].reshape(nk, C)
            v = V[bb].reshape(nk, C)
            for hd in range(C // HEAD_DIM):
                sl = slice(hd * HEAD_DIM, (hd + 1) * HEAD_DIM)
                S = (q[:, sl] @ k[:, sl].T) / math.sqrt(HEAD_DIM)
                O[bb, :, sl] = _softmax_rows(S) @ v[:, sl]
        out.append(O.reshape(Bn, h, W, C) @ wo.T + bo)
    return out


def layer_norm(xs, gamma, beta):
    """LayerNorm over the channels of every token (reading D25; eps = 1e-5, biased variance):
    y = gamma (x - mean_c x) / sqrt(var_c x + eps) + beta.  Patch-local: no exchange."""
    out = []
    for x in xs:
        mu = x.mean(axis=-1, keepdims=True)
        var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
        out.append((x - mu) / np.sqrt(var + LN_EPS) * gamma + beta)
    return out


def cross_attention(hs, context, wq, wk, wv, wo, bo):
    """Multi-head cross-attention of every token to the 77-token context (reading D25/D26):
    Q = X W_q, K = ctx W_k, V = ctx W_v (no bias), heads = C/64, scale 1/8, O W_o + b_o.
    context: [B=2, 77, ctx_dim] (b = 0 uncond, b = 1 cond).  Patch-local: no exchange."""
    out = []
    for x in hs:
        Bn, h, W, C = x.shape
        O = np.zeros((Bn, h * W, C))
        for bb in range(Bn):
            q = x[bb].reshape(h * W, C) @ wq.T
            k = context[bb] @ wk.T
            v = context[bb] @ wv.T
            for hd in range(C // HEAD_DIM):
                sl = slice(hd * HEAD_DIM, (hd + 1) * HEAD_DIM)
                S = (q[:, sl] @ k[:, sl].T) / math.sqrt(HEAD_DIM)
                O[bb, :, sl] = _softmax_rows(S) @ v[:, sl]
        out.append(O.reshape(Bn, h, W, C) @ wo.T + bo)
    return out


def gelu(x):
    """Exact GELU x Phi(x) = x (1 + erf(x / sqrt 2)) / 2 (SDXL's GEGLU uses the exact form; D25)."""
    return 0.5 * x * (1.0 + _erf(x / math.sqrt(2.0)))


def geglu_ff(xs, w1, b1, w2, b2):
    """GEGLU feed-forward (reading D25): u = X W_1 + b_1 (8C), split into the value a (first 4C)
    and the gate g (last 4C); FF(X) = (a * gelu(g)) W_2 + b_2."""
    out = []
    for x in xs:
        u = x @ w1.T + b1
        half = u.shape[-1] // 2
        out.append((u[..., :half] * gelu(u[..., half:])) @ w2.T + b2)
    return out


def upsample2(xs):
    """Nearest x2 (SDXL Upsample2D), patch-local: low rows [i h, (i+1) h) map to
    high rows [2 i h, 2 (i+1) h)."""
    return [np.repeat(np.repeat(x, 2, axis=1), 2, axis=2) for x in xs]


def linear(xs, w, b):
    return [x @ w.T + b for x in xs]


def timestep_embedding(P: Params, model: str, tau: int, cond: np.ndarray) -> np.ndarray:
    """temb (reading D19): sinusoid [cos(tau f_j), sin(tau f_j)],
    f_j = exp(-ln(1e4) j / half) -> Linear -> SiLU -> Linear; the cond branch
    (b = 1) adds c, the uncond branch (b = 0) adds nothing (reading D11)."""
    a = arch(model)
    half = a["sin_dim"] // 2
    f = np.exp(-math.log(10000.0) * np.arange(half, dtype=np.float64) / half)
    e = np.concatenate([np.cos(tau * f), np.sin(tau * f)])
    hdn = silu(P("time.lin1.w") @ e + P("time.lin1.b"))
    emb = P("time.lin2.w") @ hdn + P("time.lin2.b")
    return np.stack([emb, emb + np.asarray(cond, dtype=np.float64)])      # [B=2, T]


def resblock(ctx, P, pre, xs, emb):
    """RB(a->b), App. A.  xs may be the channel concat [h, skip] (SDXL order)."""
    h = group_norm(ctx, xs, P(f"{pre}.gn1.g"), P(f"{pre}.gn1.b"), act=True)
    h = conv3x3(ctx, h, P(f"{pre}.conv1.w"), P(f"{pre}.conv1.b"))
    t = silu(emb) @ P(f"{pre}.temb.w").T + P(f"{pre}.temb.b")          # [B, Cout]
    h = [y + t[:, None, None, :] for y in h]
    h = group_norm(ctx, h, P(f"{pre}.gn2.g"), P(f"{pre}.gn2.b"), act=True)
    h = conv3x3(ctx, h, P(f"{pre}.conv2.w"), P(f"{pre}.conv2.b"))
    cin, cout = xs[0].shape[-1], h[0].shape[-1]
    skip = linear(xs, P(f"{pre}.skip.w"), P(f"{pre}.skip.b")) if cin != cout else xs
    return [a + s for a, s in zip(h, skip)]


def attn_stack(ctx, P, pre, xs, depth, context=None):
    """AS(C, d), App. A.  With a context (the '_xf' models) every layer is SDXL's transformer
    block (reading D25): h += SA(LN1 h) [PCPP bands of K/V of LN1 h]; h += CA(LN2 h, ctx);
    h += FF(LN3 h)."""
    g = group_norm(ctx, xs, P(f"{pre}.gn.g"), P(f"{pre}.gn.b"), act=False)
    h = linear(g, P(f"{pre}.proj_in.w"), P(f"{pre}.proj_in.b"))
    for d in range(depth):
        a = f"{pre}.attn{d}"
        x = layer_norm(h, P(f"{a}.ln1.g"), P(f"{a}.ln1.b")) if context is not None else h
        o = attention(ctx, x, P(f"{a}.wq"), P(f"{a}.wk"), P(f"{a}.wv"), P(f"{a}.wo"), P(f"{a}.bo"))
        h = [x + y for x, y in zip(h, o)]
        if context is not None:
            x = layer_norm(h, P(f"{a}.ln2.g"), P(f"{a}.ln2.b"))
            o = cross_attention(x, context, P(f"{a}.xq"), P(f"{a}.xk"), P(f"{a}.xv"), P(f"{a}.xo"), P(f"{a}.xbo"))
            h = [x + y for x, y in zip(h, o)]
            x = layer_norm(h, P(f"{a}.ln3.g"), P(f"{a}.ln3.b"))
            o = geglu_ff(x, P(f"{a}.ff1.w"), P(f"{a}.ff1.b"), P(f"{a}.ff2.w"), P(f"{a}.ff2.b"))
            h = [x + y for x, y in zip(h, o)]
    o = linear(h, P(f"{pre}.proj_out.w"), P(f"{pre}.proj_out.b"))
    return [x + y for x, y in zip(o, xs)]


def unet(ctx: Ctx, P: Params, model: str, latents, emb, context=None):
    """eps_theta over n patches, both CFG branches as batch 2 (b=0 uncond, b=1 cond).

    latents: list over ranks of [h, W, 4] float64.  context: [2, 77, ctx_dim] for the '_xf'
    models (required there), else None.  Returns list of [2, h, W, 4].
    """
    if arch(model)["xf"] != (context is not None):
        raise ValueError("the '_xf' models need a context, the others take none")
    if context is not None:
        context = np.asarray(context, dtype=np.float64)
    xs = [np.stack([x, x]).astype(np.float64) for x in latents]
    skips = []
    h = None
    for kind, pre, args in _blocks(model):
        if kind == "conv_in":
            h = conv3x3(ctx, xs, P("conv_in.w"), P("conv_in.b"))
        elif kind == "push":
            skips.append(h)
        elif kind == "pop":
            s = skips.pop()
            h = [np.concatenate([a, b], axis=-1) for a, b in zip(h, s)]
        elif kind == "rb":
            h = resblock(ctx, P, pre, h, emb)
        elif kind == "as":
            h = attn_stack(ctx, P, pre, h, args[1], context)
        elif kind == "down":
            h = conv3x3(ctx, h, P(f"{pre}.conv.w"), P(f"{pre}.conv.b"), stride=2)
        elif kind == "up":
            h = conv3x3(ctx, upsample2(h), P(f"{pre}.conv.w"), P(f"{pre}.conv.b"))
        elif kind == "out":
            h = group_norm(ctx, h, P("out.gn.g"), P("out.gn.b"), act=True)
            h = conv3x3(ctx, h, P("conv_out.w"), P("conv_out.b"))
    return h
