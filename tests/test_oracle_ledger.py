"""Pins for the byte ledger: Table 1 and counted == closed form (P7)."""
import json
import os

import numpy as np
import pytest

from oracle import ledger, model as M, pcpp
from tests import _data

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table1.json")))


def test_table1_reproduced_from_the_stack():
    for j, res in enumerate(GOLD["resolutions"]):
        r = ledger.paper_convention("sdxl", res, GOLD["n_devices"])
        # buffer sizes round to the printed digits (reading D14: element counts)
        assert round(r["total_buffer"] / 1e9, 3 if res < 3840 else 2) == GOLD["total_buffer_G"][j]
        assert round(r["b_attn"] / 1e9, 2 if res == 1024 else 3) == GOLD["attn_G"][j]
        assert round(r["b_conv"] / 1e9, 3) == GOLD["conv2d_G"][j]
        assert round(r["b_gn"] / 1e6, 3) == GOLD["group_norm_M"][j]
        # the printed totals follow from the printed (rounded) buffer sizes by the §4 formulas
        n = GOLD["n_devices"]
        df = GOLD["total_buffer_G"][j] * (n - 1)
        pc = 2 * GOLD["attn_G"][j] + (n - 1) * (GOLD["conv2d_G"][j] + GOLD["group_norm_M"][j] / 1e3)
        assert abs(df - GOLD["distrifusion_G"][j]) < 5e-4 * max(1, GOLD["distrifusion_G"][j])
        assert abs(pc - GOLD["pcpp_G"][j]) < 2e-3 * max(1, GOLD["pcpp_G"][j])
        # and our unrounded totals agree with the printed ones to the printed precision
        assert abs(r["df"] / 1e9 - GOLD["distrifusion_G"][j]) / GOLD["distrifusion_G"][j] < 2e-3
        assert abs(r["pcpp"] / 1e9 - GOLD["pcpp_G"][j]) / GOLD["pcpp_G"][j] < 3e-3
        assert 0.68 <= r["cut"] <= 0.71                          # "around 70%"


@pytest.mark.parametrize("model,H,n,p", [("tiny", 32, 2, 0.25), ("tiny", 32, 4, 0.5),
                                         ("tiny", 32, 8, 1.0), ("tiny", 32, 4, 0.0),
                                         ("sdxl", 16, 2, 0.3), ("sdxl", 32, 8, 0.8)])
def test_counted_ledger_equals_closed_form(model, H, n, p):
    blob, xT, c = _data.blob(model), _data.latent(H, H), _data.cond(model)
    for scheme in ("pcpp", "fullmap"):
        cfg = pcpp.Config(model=model, H=H, W=H, n=n, p=p, warmup=1, steps=4, scheme=scheme)
        out = pcpp.sample(cfg, blob, xT, c, max_steps=2)
        warm = pcpp.ledger_totals(out["ledger"][0], 2)
        asyn = pcpp.ledger_totals(out["ledger"][1], 2)
        assert warm == ledger.physical_bytes(model, H, H, n, p, 2, "warmup")
        kind = "pcpp_async" if scheme == "pcpp" else "fullmap_async"
        assert asyn == ledger.physical_bytes(model, H, H, n, p, 2, kind)


def test_sdxl_1024_cut_vs_fullmap():
    # 1024^2, n=8, p=0.8 -> PCPP moves ~80% fewer bytes than FULLMAP
    a = ledger.physical_bytes("sdxl", 128, 128, 8, 0.8, 2, "pcpp_async")
    f = ledger.physical_bytes("sdxl", 128, 128, 8, 0.8, 2, "fullmap_async")
    cut = 1 - sum(a.values()) / sum(f.values())
    assert 0.75 < cut < 0.85
