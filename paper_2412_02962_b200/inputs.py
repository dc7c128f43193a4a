"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no conv, norm, attention,
schedule, CFG or band logic). It only turns a weight *spec list* -- which each
side derives from its own model description -- into random numbers, and draws
the latent x_T and the condition vector c.  The oracle (``oracle/``) and the
CUDA path (``libpcpp``) never import each other; this is the one module both
sides' callers use (task rule: "only the seeded input generators serve both").

Seeds follow SURVEY.md §8(c): weights 0, x_T 1, c 2 (numpy PCG64).
Reading D17: random init, W ~ N(0, std^2) with std chosen per tensor
by the model description; GN gamma ~ 1 + 0.1 N(0,1), beta ~ 0.1 N(0,1); biases
~ 0.1 N(0,1) so that every bias path is visible in the parity tests.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

SEED_WEIGHTS = 0
SEED_XT = 1
SEED_COND = 2
SEED_CONTEXT = 3


def init_specs(manifest) -> list[tuple[int, float, float]]:
    """(numel, mean, std) per manifest entry [(name, shape), ...] -- reading D17.

    conv [Cout,3,3,Cin]: std 1/sqrt(9 Cin) (x 1/sqrt(2) for a ResBlock's conv2);
    linear [out,in]: std 1/sqrt(in) (x 1/sqrt(2 depth) for W_o of an attention stack of that
    depth, x 1/sqrt(2) for proj_out); GN gamma 1 + 0.1 z, GN beta / biases 0.1 z.
    The rule reads only names and shapes, so both sides can derive it from their own manifest.
    """
    names = [n for n, _ in manifest]
    depth = {}
    for n in names:
        if n.endswith(".wo"):
            pre = n[: n.rindex(".attn")]
            depth[pre] = depth.get(pre, 0) + 1
    out = []
    for name, shape in manifest:
        numel = int(np.prod(shape))
        leaf = name.rsplit(".", 1)[-1]
        if len(shape) == 4:
            std = 1.0 / np.sqrt(9 * shape[3])
            if name.endswith(".conv2.w"):
                std /= np.sqrt(2.0)
            out.append((numel, 0.0, float(std)))
        elif len(shape) == 2:
            std = 1.0 / np.sqrt(shape[1])
            if leaf in ("wo", "xo") or name.endswith(".ff2.w"):     # residual-branch outputs of a block
                std /= np.sqrt(2.0 * depth[name[: name.rindex(".attn")]])
            elif name.endswith("proj_out.w"):
                std /= np.sqrt(2.0)
            out.append((numel, 0.0, float(std)))
        elif leaf == "g":
            out.append((numel, 1.0, 0.1))
        else:                                   # GN beta ('.b' of a norm) and every bias
            out.append((numel, 0.0, 0.1))
    return out


def make_weight_blob(specs, seed: int = SEED_WEIGHTS) -> np.ndarray:
    """specs: iterable of (numel, mean, std).  Returns one flat float32 blob.

    Each tensor is mean + std * z with z drawn sequentially from one PCG64
    stream in spec order, so the blob is a pure function of (specs, seed).
    """
    specs = [(int(n), float(m), float(s)) for (n, m, s) in specs]
    total = sum(n for n, _, _ in specs)
    out = np.empty(total, dtype=np.float32)
    # fixed 1 Mi-value chunks, chunk j drawn from PCG64(SeedSequence([seed, j])):
    # independent of the thread count, so the blob is a pure function of (specs, seed)
    chunk = 1 << 20
    nchunks = (total + chunk - 1) // chunk

    def fill(j):
        g = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, j])))
        lo = j * chunk
        g.standard_normal(min(chunk, total - lo), dtype=np.float32, out=out[lo:lo + chunk])

    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
        list(ex.map(fill, range(nchunks)))
    off = 0
    for n, m, s in specs:
        seg = out[off:off + n]
        seg *= np.float32(s)
        if m:
            seg += np.float32(m)
        off += n
    return out


def round_to_bf16(a: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bfloat16 (round-to-nearest-even),
    returned as float32 holding exactly representable bf16 values.  Used so
    that bf16-mode parity runs feed both sides identical (pre-rounded) weights.
    """
    a = np.ascontiguousarray(a, dtype=np.float32)
    out = np.empty_like(a)
    src, dst = a.reshape(-1).view(np.uint32), out.reshape(-1).view(np.uint32)
    step = 1 << 24                      # chunked: the SDXL_XF blob has 2.6 G values
    for i in range(0, src.size, step):
        u = src[i:i + step].astype(np.uint64)
        lsb = (u >> 16) & 1
        dst[i:i + step] = ((u + 0x7FFF + lsb) & 0xFFFF0000).astype(np.uint32)
    return out


def make_latent(H: int, W: int, C: int = 4, seed: int = SEED_XT) -> np.ndarray:
    """x_T ~ N(0, I) as [H, W, C] float32 (row-major, C innermost)."""
    z = np.random.Generator(np.random.PCG64(seed)).standard_normal((H, W, C))
    return z.astype(np.float32)


def make_context(ctx_len: int, dim: int, seed: int = SEED_CONTEXT) -> np.ndarray:
    """Cross-attention context of the '_xf' models (reading D26): [2, ctx_len, dim] float32 ~ N(0, I);
    [0] = the unconditional branch's (SDXL encodes the empty prompt: not zeros), [1] = the prompt's."""
    z = np.random.Generator(np.random.PCG64(seed)).standard_normal((2, ctx_len, dim))
    return z.astype(np.float32)


def make_cond(dim: int, seed: int = SEED_COND) -> np.ndarray:
    """Condition vector c ~ N(0, I) of the temb dimension, float32."""
    z = np.random.Generator(np.random.PCG64(seed)).standard_normal(dim)
    return z.astype(np.float32)
