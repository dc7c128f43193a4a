"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/pcpp.h declares,
its own model manifest equals the oracle's, its host-side plan math (band rows, byte ledger) is
bit-exact against the oracle's closed forms, and argument validation rejects bad plans."""
import os
import re

import pytest

from oracle import ledger, model as M
from oracle.schedule import band_rows
from paper_2412_02962_b200 import pcpp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "pcpp.h")).read()
    declared = set(re.findall(r"PCPP_API\s+[\w\s\*]+?\b(pcpp_\w+)\s*\(", hdr))
    assert len(declared) >= 19
    L = pcpp.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert declared == set(pcpp.SYMBOLS)


@pytest.mark.parametrize("model", ["tiny", "sdxl"])
def test_manifest_matches_oracle(model):
    assert pcpp.manifest(model) == [(n, tuple(s)) for n, s, _ in M.manifest(model)]
    assert pcpp.pcpp_weights_len(model) == sum(M.init_spec(s, k)[0] for _, s, k in M.manifest(model))


@pytest.mark.parametrize("model", ["tiny", "sdxl"])
def test_init_rule_from_library_manifest_matches_oracle(model):
    from paper_2412_02962_b200 import inputs
    a = inputs.init_specs(pcpp.manifest(model))
    b = M.weight_specs(model)
    assert len(a) == len(b)
    for x, y in zip(a, b):
        assert x[0] == y[0] and x[1] == y[1] and abs(x[2] - y[2]) < 1e-15 * max(1, y[2])


@pytest.mark.parametrize("model,H,n,p", [("sdxl", 128, 8, 0.8), ("sdxl", 128, 4, 0.8), ("sdxl", 128, 2, 0.3),
                                         ("sdxl", 256, 8, 0.8), ("sdxl", 480, 8, 0.8), ("sdxl", 128, 8, 0.0),
                                         ("sdxl", 128, 8, 0.125), ("sdxl", 128, 8, 0.25), ("sdxl", 128, 8, 0.5),
                                         ("sdxl", 128, 8, 1.0), ("tiny", 32, 2, 0.25), ("sdxl", 32, 8, 0.3),
                                         ("sdxl", 128, 1, 0.8)])
@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_plan_math_bit_exact(model, H, n, p, precision):
    es = 2 if precision == "bf16" else 4
    cfg = pcpp.make_config(model=model, precision=precision)
    info = pcpp.pcpp_plan_info(H, H, 4, n, p, 1 if n > 1 else 0, cfg)
    lay = [L for L in ledger.layer_table(model, H, H) if L["kind"] == "attn"]
    assert info["n_attn"] == len(lay)
    assert info["attn_h"] == [L["H_l"] // n for L in lay]
    assert info["attn_r"] == [band_rows(p, L["H_l"] // n) for L in lay]
    cls = ("attn", "conv", "gn")
    for key, kind in (("bytes_async", "pcpp_async"), ("bytes_warmup", "warmup"), ("bytes_fullmap", "fullmap_async")):
        want = ledger.physical_bytes(model, H, H, n, p, es, kind)
        assert info[key] == [want[c] for c in cls], key
    want = ledger.physical_bytes(model, H, H, n, p, es, "pcpp_async")
    assert info["bytes_counted_async"] == [want[c] for c in cls]
    want = ledger.physical_bytes(model, H, H, n, p, es, "warmup")
    assert info["bytes_counted_warmup"] == [want[c] for c in cls]


def test_fullmap_counted_ledger():
    cfg = pcpp.make_config(model="sdxl", scheme="fullmap")
    info = pcpp.pcpp_plan_info(128, 128, 4, 8, 0.8, 4, cfg)
    want = ledger.physical_bytes("sdxl", 128, 128, 8, 0.8, 2, "fullmap_async")
    assert info["bytes_counted_async"] == [want[c] for c in ("attn", "conv", "gn")]


@pytest.mark.parametrize("args", [
    dict(H=128, n=3, p=0.5, w=1),        # H % 4n
    dict(H=128, n=16, p=0.5, w=1),       # n > 8
    dict(H=128, n=8, p=1.5, w=1),        # p > 1 undefined
    dict(H=128, n=8, p=-0.1, w=1),
    dict(H=128, n=8, p=0.5, w=0),        # warm-up required for n > 1 (D20)
    dict(H=128, n=8, p=0.5, w=60),       # w > S
    dict(H=130, n=1, p=0.5, w=1),
])
def test_validation_rejects(args):
    cfg = pcpp.make_config(model="sdxl")
    with pytest.raises(pcpp.PcppError) as e:
        pcpp.pcpp_plan_info(args["H"], 128, 4, args["n"], args["p"], args["w"], cfg)
    assert e.value.status == pcpp.ERR_INVALID


def test_validation_channels_and_nccl_world():
    cfg = pcpp.make_config(model="sdxl")
    with pytest.raises(pcpp.PcppError):
        pcpp.pcpp_plan_info(128, 128, 3, 2, 0.5, 1, cfg)
    cfg = pcpp.make_config(model="sdxl", backend="nccl", world=4)
    with pytest.raises(pcpp.PcppError):
        pcpp.pcpp_plan_info(128, 128, 4, 2, 0.5, 1, cfg)


def test_scheduler_validation():
    """An unknown scheduler id is rejected before any allocation (PCPP_ERR_INVALID)."""
    from paper_2412_02962_b200 import pcpp
    cfg = pcpp.make_config(model="tiny", num_steps=4)
    cfg.scheduler = 7
    info = None
    with pytest.raises(pcpp.PcppError):
        info = pcpp.pcpp_plan_info(32, 32, 4, 2, 0.25, 1, cfg)
    assert info is None


@pytest.mark.parametrize("model,H,n,prec", [("sdxl", 128, 1, "bf16"), ("sdxl", 128, 8, "bf16"), ("sdxl", 480, 8, "fp32"),
                                           ("sdxl", 32, 2, "fp32"), ("tiny", 32, 2, "bf16"), ("tiny", 32, 4, "fp32")])
def test_arena_memory_plan(model, H, n, prec):
    """The liveness-based rank-arena plan (runtime.cpp plan_memory) runs host-only inside
    pcpp_plan_info, checks its own no-overlap invariant for every pair of tensors live at the same
    op (an overlap would fail the call), and shrinks the activation arena."""
    cfg = pcpp.make_config(model=model, precision=prec)
    info = pcpp.pcpp_plan_info(H, H, 4, n, 0.8 if n > 1 else 0.0, 1 if n > 1 else 0, cfg)
    assert 0 < info["arena_bytes_per_rank"] <= info["arena_bytes_unplanned"]
    if model == "sdxl":
        assert info["arena_bytes_per_rank"] < 0.75 * info["arena_bytes_unplanned"]


@pytest.mark.parametrize("model,H,n,p", [("sdxl", 128, 4, 0.8), ("sdxl", 128, 2, 0.3), ("tiny", 32, 2, 0.25), ("sdxl", 128, 1, 0.0)])
def test_cfg_split_plan_math(model, H, n, p):
    # the CFG device split: per-branch exchanges within each group, 2 x the batch-1 bytes of one
    # group = the batch-2 bytes of the same n; the eps swap moves one fp32 patch per rank and step
    base = pcpp.pcpp_plan_info(H, H, 4, n, p, 1, pcpp.make_config(model=model))
    sp = pcpp.pcpp_plan_info(H, H, 4, n, p, 1, pcpp.make_config(model=model, cfg_split=True))
    assert sp["bytes_counted_async"] == sp["bytes_async"] == base["bytes_async"]
    assert sp["bytes_counted_warmup"] == base["bytes_counted_warmup"]
    assert sp["bytes_eps"] == 2 * n * (H // n) * H * 4 * 4
    assert abs(sp["step_flops_rank_max"] * 2 - base["step_flops_rank_max"]) <= 1e-9 * base["step_flops_rank_max"]


def test_cfg_split_validation():
    C = pcpp.make_config
    with pytest.raises(pcpp.PcppError):      # NCCL would need per-branch communicators
        pcpp.pcpp_plan_info(128, 128, 4, 2, 0.3, 1, C(model="sdxl", cfg_split=True, backend="nccl", world=4, rank=0))
    with pytest.raises(pcpp.PcppError):      # PEER world must be 2 n
        pcpp.pcpp_plan_info(128, 128, 4, 2, 0.3, 1, C(model="sdxl", cfg_split=True, backend="peer", world=2, rank=0))
    with pytest.raises(pcpp.PcppError):
        pcpp.pcpp_plan_info(32, 32, 4, 2, 0.3, 1, C(model="tiny_xf", cfg_split=True))
    assert pcpp.pcpp_plan_info(128, 128, 4, 2, 0.3, 1, C(model="sdxl", cfg_split=True, backend="peer", world=4,
                                                         rank=3))["backend"] == pcpp.COMM_PEER
