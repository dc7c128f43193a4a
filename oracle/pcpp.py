"""The PCPP sampling schedule over n simulated ranks -- TEST INFRASTRUCTURE ONLY.

Follows, in the paper's order:
  * split x_t horizontally into n patches of h = H/n rows (§3.1);
  * the first w steps are synchronous (§3.2 "initial warm-up steps where
    we perform synchronous AllGather"; w = 4 in Table 2);
  * later steps read neighbour data stale from step t+1 (§3.2; Eq. 1);
  * per rank: CFG (Eq. 2) and the DDIM update -- or DPM-Solver++(2M),
    reading D23 -- on its own patch (the scheduler is elementwise: patch-local);
  * scheme 'fullmap' is the DistriFusion baseline (§3.2): every
    attention layer reads all other ranks' stale K/V;
  * scheme 'sync' runs every step synchronously (domain parallelism).

Execution is layer-major, rank-minor inside one process; the device boundary is
simulated by the stale store.  No code is shared with libpcpp.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import model as M
from .schedule import ancestral_step, cfg_combine, ddim_step, ddim_timesteps, dpmpp_2m_step, noise_patch


@dataclass
class Config:
    model: str = "tiny"
    H: int = 32
    W: int = 32
    n: int = 2
    p: float = 0.25
    warmup: int = 1
    steps: int = 4
    guidance: float = 5.0
    scheme: str = "pcpp"          # 'pcpp' | 'fullmap' | 'sync'
    scheduler: str = "ddim"       # 'ddim' | 'dpmpp2m' (north star "DPM-solver", D23) | 'ancestral' (Eq. 3-4, D24)
    noise_seed: int = 0           # key of the counter-based noise of the ancestral sampler (D24)
    extras: dict = field(default_factory=dict)


def split(x: np.ndarray, n: int):
    """Row strips x^(i) = rows [i h, (i+1) h)."""
    H = x.shape[0]
    if H % n:
        raise ValueError("H must be divisible by n (P:39 h = H/n)")
    h = H // n
    return [x[i * h:(i + 1) * h].astype(np.float64) for i in range(n)]


def sample(cfg: Config, blob: np.ndarray, x_T: np.ndarray, cond: np.ndarray,
           record: bool = True, max_steps: int | None = None, on_step=None, context=None):
    """Run the n-patch PCPP sampler.  on_step(k), if given, is called after step k (timing hook).
    context: [2, 77, ctx_dim] cross-attention context of the '_xf' models (b = 0 uncond, 1 cond).

    Returns dict(x0=[H,W,4], xs=[x after every step], eps=[per-step eps_hat],
                 ledger=[per-step list of (kind, lid, src, dst, elems)],
                 modes=[per-step mode]).
    """
    P = M.Params(cfg.model, blob)
    n = cfg.n
    taus = ddim_timesteps(cfg.steps)
    patches = split(np.asarray(x_T), n)
    prev = None
    out = dict(xs=[], eps=[], ledger=[], modes=[])
    last = cfg.steps if max_steps is None else min(cfg.steps, max_steps)
    for k in range(last):
        sync = cfg.scheme == "sync" or k < cfg.warmup
        mode = "sync" if sync else "async"
        ctx = M.Ctx(n, cfg.p, mode, "fullmap" if cfg.scheme == "fullmap" else "pcpp", prev)
        emb = M.timestep_embedding(P, cfg.model, taus[k], cond)
        eps = M.unet(ctx, P, cfg.model, patches, emb, context)
        eps_hat = [cfg_combine(e[0], e[1], cfg.guidance) for e in eps]   # b=0 uncond, b=1 cond
        if cfg.scheduler == "dpmpp2m":
            if k == 0:
                x0_hist = [None] * n
            res = [dpmpp_2m_step(x, e, cfg.steps, k, x0p) for x, e, x0p in zip(patches, eps_hat, x0_hist)]
            patches = [r[0] for r in res]
            x0_hist = [r[1] for r in res]
        elif cfg.scheduler == "ancestral":
            h = patches[0].shape[0]
            patches = [ancestral_step(x, e, cfg.steps, k, noise_patch(cfg.noise_seed, k, i * h, h, cfg.W))
                       for i, (x, e) in enumerate(zip(patches, eps_hat))]
        else:
            patches = [ddim_step(x, e, cfg.steps, k) for x, e in zip(patches, eps_hat)]
        prev = ctx.nxt
        if on_step is not None:
            on_step(k)
        if record:
            out["xs"].append(np.concatenate(patches, axis=0))
            out["eps"].append(np.concatenate(eps_hat, axis=0))
            out["ledger"].append(ctx.ledger)
            out["modes"].append(mode)
    out["x0"] = np.concatenate(patches, axis=0)
    return out


def forward_pair(cfg: Config, blob, x, tau, cond, first_mode: str, second_mode: str, context=None):
    """Two forwards on identical (x, tau): the second reads the store the first
    wrote.  Used by pin P6 (fresh-then-async must reproduce the fresh output)."""
    P = M.Params(cfg.model, blob)
    patches = split(np.asarray(x), cfg.n)
    emb = M.timestep_embedding(P, cfg.model, tau, cond)
    scheme = "fullmap" if cfg.scheme == "fullmap" else "pcpp"
    c1 = M.Ctx(cfg.n, cfg.p, first_mode, scheme)
    e1 = M.unet(c1, P, cfg.model, patches, emb, context)
    c2 = M.Ctx(cfg.n, cfg.p, second_mode, scheme, c1.nxt)
    e2 = M.unet(c2, P, cfg.model, patches, emb, context)
    return e1, e2


def ledger_totals(entries, elem_bytes: int) -> dict:
    """Sum a step's counted ledger into bytes per class.  Activations travel at
    elem_bytes per element, the latent halos of conv_in at 4 (fp32), GN statistics
    as float64 (8 bytes)."""
    tot = {"attn": 0, "conv": 0, "gn": 0}
    for kind, lid, _src, _dst, elems in entries:
        e = 8 if kind == "gn" else (4 if lid == "conv0" else elem_bytes)   # conv0 = conv_in on the fp32 latent
        tot[kind] += elems * e
    return tot
