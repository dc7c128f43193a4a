"""Independent single-device reference forward, written with torch.nn.functional
library routines in float64 on the CPU (NCHW layout).

Used only to pin the oracle: the oracle's n-rank code
path must reduce to this unpartitioned network when nothing is partitioned
(n = 1) or when every step is synchronous.  It transcribes SURVEY App. A on its
own (it does not call oracle.model's ops or block walker); it reads the flat
weight blob by the manifest's (name, shape) order only.
"""
from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F

from oracle.model import manifest


def load(model, blob):
    t, off = {}, 0
    for name, shape, _ in manifest(model):
        n = int(np.prod(shape))
        t[name] = torch.from_numpy(np.asarray(blob[off:off + n], dtype=np.float64).reshape(shape))
        off += n
    return t


def conv(x, w, b, stride=1):
    # blob layout [Cout, 3, 3, Cin] -> torch [Cout, Cin, 3, 3]
    return F.conv2d(x, w.permute(0, 3, 1, 2).contiguous(), b, stride=stride, padding=1)


def gn(x, g, b, act):
    y = F.group_norm(x, 32, g, b, eps=1e-5)
    return F.silu(y) if act else y


def lin(x, w, b):  # x NCHW -> per-pixel linear
    return torch.einsum("bchw,oc->bohw", x, w) + b[None, :, None, None]


def mhsa(x, wq, wk, wv, wo, bo):
    B, C, H, W = x.shape
    tok = x.permute(0, 2, 3, 1).reshape(B, H * W, C)
    q, k, v = tok @ wq.T, tok @ wk.T, tok @ wv.T
    nh = C // 64

    def heads(z):
        return z.reshape(B, H * W, nh, 64).transpose(1, 2)

    o = F.scaled_dot_product_attention(heads(q), heads(k), heads(v))
    o = o.transpose(1, 2).reshape(B, H * W, C) @ wo.T + bo
    return o.reshape(B, H, W, C).permute(0, 3, 1, 2)


def temb(t, model, tau, cond):
    T = 1280 if model.startswith("sdxl") else 512
    sd = 320 if model.startswith("sdxl") else 128
    half = sd // 2
    freqs = torch.exp(-math.log(10000.0) * torch.arange(half, dtype=torch.float64) / half)
    e = torch.cat([torch.cos(tau * freqs), torch.sin(tau * freqs)])
    e = F.linear(F.silu(F.linear(e, t["time.lin1.w"], t["time.lin1.b"])), t["time.lin2.w"], t["time.lin2.b"])
    c = torch.from_numpy(np.asarray(cond, dtype=np.float64))
    assert c.numel() == T
    return torch.stack([e, e + c])


def resblock(t, pre, x, emb):
    h = conv(gn(x, t[f"{pre}.gn1.g"], t[f"{pre}.gn1.b"], True), t[f"{pre}.conv1.w"], t[f"{pre}.conv1.b"])
    h = h + F.linear(F.silu(emb), t[f"{pre}.temb.w"], t[f"{pre}.temb.b"])[:, :, None, None]
    h = conv(gn(h, t[f"{pre}.gn2.g"], t[f"{pre}.gn2.b"], True), t[f"{pre}.conv2.w"], t[f"{pre}.conv2.b"])
    if f"{pre}.skip.w" in t:
        x = lin(x, t[f"{pre}.skip.w"], t[f"{pre}.skip.b"])
    return x + h


def ln(x, g, b):   # LayerNorm over channels of every pixel (NCHW)
    return F.layer_norm(x.permute(0, 2, 3, 1), (x.shape[1],), g, b, eps=1e-5).permute(0, 3, 1, 2)


def mhca(x, ctx, wq, wk, wv, wo, bo):   # cross-attention to ctx [B, 77, D] (diffusers Attention, no qkv bias)
    B, C, H, W = x.shape
    tok = x.permute(0, 2, 3, 1).reshape(B, H * W, C)
    q, k, v = tok @ wq.T, ctx @ wk.T, ctx @ wv.T
    nh = C // 64
    o = F.scaled_dot_product_attention(q.reshape(B, -1, nh, 64).transpose(1, 2), k.reshape(B, -1, nh, 64).transpose(1, 2),
                                       v.reshape(B, -1, nh, 64).transpose(1, 2))
    o = o.transpose(1, 2).reshape(B, H * W, C) @ wo.T + bo
    return o.reshape(B, H, W, C).permute(0, 3, 1, 2)


def ff(x, w1, b1, w2, b2):   # diffusers GEGLU: proj -> chunk(2) -> value * gelu(gate) -> Linear
    u = lin(x, w1, b1)
    a, g = u.chunk(2, dim=1)
    return lin(a * F.gelu(g), w2, b2)


def attn_stack(t, pre, x, depth, ctx=None):
    h = lin(gn(x, t[f"{pre}.gn.g"], t[f"{pre}.gn.b"], False), t[f"{pre}.proj_in.w"], t[f"{pre}.proj_in.b"])
    for d in range(depth):
        a = f"{pre}.attn{d}"
        y = ln(h, t[f"{a}.ln1.g"], t[f"{a}.ln1.b"]) if ctx is not None else h
        h = h + mhsa(y, t[f"{a}.wq"], t[f"{a}.wk"], t[f"{a}.wv"], t[f"{a}.wo"], t[f"{a}.bo"])
        if ctx is not None:
            h = h + mhca(ln(h, t[f"{a}.ln2.g"], t[f"{a}.ln2.b"]), ctx, t[f"{a}.xq"], t[f"{a}.xk"], t[f"{a}.xv"],
                         t[f"{a}.xo"], t[f"{a}.xbo"])
            h = h + ff(ln(h, t[f"{a}.ln3.g"], t[f"{a}.ln3.b"]), t[f"{a}.ff1.w"], t[f"{a}.ff1.b"], t[f"{a}.ff2.w"],
                       t[f"{a}.ff2.b"])
    return x + lin(h, t[f"{pre}.proj_out.w"], t[f"{pre}.proj_out.b"])


def eps(model, blob, x_hw4, tau, cond, context=None):
    """Full-image eps for both CFG branches: returns [2, H, W, 4] float64.  context [2, 77, D] for
    the '_xf' models (SDXL's transformer blocks)."""
    t = load(model, blob)
    ctx = None if context is None else torch.from_numpy(np.asarray(context, dtype=np.float64))
    emb = temb(t, model, tau, cond)
    x = torch.from_numpy(np.asarray(x_hw4, dtype=np.float64)).permute(2, 0, 1)[None].repeat(2, 1, 1, 1)
    h = conv(x, t["conv_in.w"], t["conv_in.b"])
    if model.startswith("tiny"):
        for j in range(2):
            h = resblock(t, f"blk{j}.rb", h, emb)
            h = attn_stack(t, f"blk{j}.as", h, 1, ctx)
    else:
        chans, depth = [320, 640, 1280], [0, 2, 10]
        skips = [h]
        for lvl in range(3):
            for j in range(2):
                h = resblock(t, f"down{lvl}.{j}.rb", h, emb)
                if depth[lvl]:
                    h = attn_stack(t, f"down{lvl}.{j}.as", h, depth[lvl], ctx)
                skips.append(h)
            if lvl < 2:
                h = conv(h, t[f"down{lvl}.ds.conv.w"], t[f"down{lvl}.ds.conv.b"], stride=2)
                skips.append(h)
        h = resblock(t, "mid.rb0", h, emb)
        h = attn_stack(t, "mid.as", h, depth[2], ctx)
        h = resblock(t, "mid.rb1", h, emb)
        for lvl in (2, 1, 0):
            for j in range(3):
                h = torch.cat([h, skips.pop()], dim=1)
                h = resblock(t, f"up{lvl}.{j}.rb", h, emb)
                if depth[lvl]:
                    h = attn_stack(t, f"up{lvl}.{j}.as", h, depth[lvl], ctx)
            if lvl > 0:
                h = F.interpolate(h, scale_factor=2, mode="nearest")
                h = conv(h, t[f"up{lvl}.us.conv.w"], t[f"up{lvl}.us.conv.b"])
        assert not skips
    h = conv(gn(h, t["out.gn.g"], t["out.gn.b"], True), t["conv_out.w"], t["conv_out.b"])
    return h.permute(0, 2, 3, 1).numpy()
