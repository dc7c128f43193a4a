"""The '_xf' models (DESIGN D25/D26): SDXL's full transformer block -- LayerNorm,
PCPP self-attention, LayerNorm, cross-attention to a 77-token context, LayerNorm, GEGLU FF -- in every
attention layer.  libpcpp (C ABI, LOOPBACK backend) against the fp64 oracle on the same seeded inputs,
per step; north-star tolerances (rel-L2 <= 1e-5 fp32, <= 2e-2 bf16)."""
import functools

import numpy as np
import pytest

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


CASES = [
    # model, H, n, p, w, S, precision, scheme, steps
    ("tiny_xf", 32, 1, 0.0, 0, 4, "fp32", "pcpp", 3),
    ("tiny_xf", 32, 2, 0.25, 1, 4, "fp32", "pcpp", 4),
    ("tiny_xf", 32, 2, 0.25, 1, 4, "bf16", "pcpp", 4),
    ("tiny_xf", 32, 4, 0.5, 1, 4, "bf16", "fullmap", 3),
    ("tiny_xf", 64, 2, 0.25, 1, 4, "bf16", "pcpp", 3),          # W = 64: two-row context tiles
    ("sdxl_xf", 32, 2, 0.3, 1, 50, "bf16", "pcpp", 2),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(map(str, c)))
def test_xf_path_matches_oracle(cuda_ok, case):
    import torch
    model, H, n, p, w, S, prec, scheme, steps = case
    wts = weights(model, prec)
    xT, cond, ctx = _data.latent(H, H), _data.cond(model), _data.context(model)
    ref = OP.sample(OP.Config(model=model, H=H, W=H, n=n, p=p, warmup=w, steps=S, scheme=scheme), wts, xT, cond,
                    max_steps=steps, context=ctx)["xs"]
    cfg = pcpp.make_config(model=model, num_steps=S, precision=prec, scheme=scheme)
    plan = pcpp.Plan(H, H, 4, n, p, w, cfg, wts)
    plan.pcpp_set_cond(cond)
    lat = torch.from_numpy(np.array(xT)).cuda()
    with pytest.raises(pcpp.PcppError):          # no context yet
        plan.pcpp_step(lat, 0)
    plan.pcpp_set_context(ctx)
    errs = []
    for k in range(steps):
        plan.pcpp_step(lat, k)
        torch.cuda.synchronize()
        errs.append(rel_l2(lat.cpu().numpy(), ref[k]))
    info = plan.pcpp_query()
    plan.close()
    print(case, "rel-L2 per step:", ["%.2e" % e for e in errs], "tc:", info["tc_kernels"])
    assert max(errs) <= TOL[prec], errs
    assert info["simt_fallbacks"] == 0


def test_set_context_rejected_for_models_without_cross_attention(cuda_ok):
    cfg = pcpp.make_config(model="tiny", num_steps=4, precision="bf16")
    plan = pcpp.Plan(32, 32, 4, 1, 0.0, 0, cfg, weights("tiny", "bf16"))
    with pytest.raises(pcpp.PcppError):
        plan.pcpp_set_context(np.zeros((2, 77, 256), np.float32))
    plan.close()
