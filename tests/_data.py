"""Cached seeded inputs for the tests (generation of the 786 M-parameter SDXL-shaped
blob takes seconds; build it once per session)."""
import functools

from oracle import model as M
from paper_2412_02962_b200 import inputs


@functools.lru_cache(maxsize=None)
def blob(model: str):
    b = inputs.make_weight_blob(M.weight_specs(model))
    b.setflags(write=False)
    return b


@functools.lru_cache(maxsize=None)
def latent(H: int, W: int):
    x = inputs.make_latent(H, W)
    x.setflags(write=False)
    return x


@functools.lru_cache(maxsize=None)
def cond(model: str):
    c = inputs.make_cond(M.arch(model)["temb"])
    c.setflags(write=False)
    return c


@functools.lru_cache(maxsize=None)
def context(model: str):
    a = M.arch(model)
    if not a["xf"]:
        return None
    c = inputs.make_context(M.CTX_LEN, a["ctx_dim"])
    c.setflags(write=False)
    return c
