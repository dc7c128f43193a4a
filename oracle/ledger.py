"""Closed-form communication bytes -- TEST INFRASTRUCTURE ONLY.

Two conventions:

1. The paper's (§4, Table 1).  b_s per layer type is the
   send-buffer size of one UNet forward; DistriFusion total = (n-1) sum b_s;
   PCPP = 2 b_attn + (n-1)(b_conv + b_gn).  Reading D14: Table 1's b_s are
   element counts (the printed totals omit the x2 bytes), reproduced with
       b_attn = sum_attn H_l W_l 2 C_l             (full-map K+V, batch 1)
       b_conv = 2 * 2 * sum_conv W_in C_in         (two 1-row halos, B = 2)
       b_gn   = 2 * 2 * 32 * 46                    (2 stats, B = 2, 32 groups)
   at n = 8 (reading D15).  Pinned by the printed digits (tests/golden/table1.json).

2. Physical bytes per step, summed over receiving ranks (what libpcpp moves):
       attn  PCPP async   : 2 (n-1) r_l W_l 2 C_l B e
       attn  warm-up / FULLMAP: (n-1) H_l W_l 2 C_l B e
       conv  stride 1     : 2 (n-1) W_in C_in B e ;  stride 2: (n-1) W_in C_in B e
                            (conv_in's input is the fp32 latent: e = 4 there)
       gn    (all-gather of local sums, float64): n (n-1) 2 G B 8
   Pinned by the oracle's counted ledger (pcpp.sample) on every config.
"""
from __future__ import annotations

from . import model as M
from .schedule import band_rows

B_CFG = 2


def layer_table(model: str, H: int, W: int):
    """Walk the stack and list every exchange-bearing layer with its geometry.

    Returns list of dicts: kind in {'conv','gn','attn'}, level, C (input
    channels for conv/gn, model width for attn), H_l, W_l (input resolution),
    stride (conv).
    """
    a = M.arch(model)
    lay = []
    lvl = 0

    def res(l):
        return H >> l, W >> l

    def rb(cin, cout):
        Hl, Wl = res(lvl)
        lay.append(dict(kind="gn", level=lvl, C=cin, H_l=Hl, W_l=Wl))
        lay.append(dict(kind="conv", level=lvl, C=cin, H_l=Hl, W_l=Wl, stride=1))
        lay.append(dict(kind="gn", level=lvl, C=cout, H_l=Hl, W_l=Wl))
        lay.append(dict(kind="conv", level=lvl, C=cout, H_l=Hl, W_l=Wl, stride=1))

    def ast(C, depth):
        Hl, Wl = res(lvl)
        lay.append(dict(kind="gn", level=lvl, C=C, H_l=Hl, W_l=Wl))
        for _ in range(depth):
            lay.append(dict(kind="attn", level=lvl, C=C, H_l=Hl, W_l=Wl))

    for kind, _pre, args in M._blocks(model):
        if kind == "conv_in":
            lay.append(dict(kind="conv", level=0, C=4, H_l=H, W_l=W, stride=1))
        elif kind == "rb":
            rb(args[0], args[1])
        elif kind == "as":
            ast(args[0], args[1])
        elif kind == "down":
            Hl, Wl = res(lvl)
            lay.append(dict(kind="conv", level=lvl, C=args[0], H_l=Hl, W_l=Wl, stride=2))
            lvl += 1
        elif kind == "up":
            lvl -= 1
            Hl, Wl = res(lvl)
            lay.append(dict(kind="conv", level=lvl, C=args[0], H_l=Hl, W_l=Wl, stride=1))
        elif kind == "out":
            Hl, Wl = res(0)
            lay.append(dict(kind="gn", level=0, C=args[0], H_l=Hl, W_l=Wl))
            lay.append(dict(kind="conv", level=0, C=args[0], H_l=Hl, W_l=Wl, stride=1))
    return lay


def paper_convention(model: str, H_img: int, n: int = 8):
    """Table 1 reproduction from the latent H = W = H_img / 8.

    Returns dict(b_attn, b_conv, b_gn, total_buffer, df, pcpp, cut) in elements.
    """
    H = W = H_img // 8
    lay = layer_table(model, H, W)
    b_attn = sum(L["H_l"] * L["W_l"] * 2 * L["C"] for L in lay if L["kind"] == "attn")
    b_conv = 2 * B_CFG * sum(L["W_l"] * L["C"] for L in lay if L["kind"] == "conv")
    b_gn = 2 * B_CFG * M.G_GROUPS * sum(1 for L in lay if L["kind"] == "gn")
    total = b_attn + b_conv + b_gn
    df = (n - 1) * total
    pcpp = 2 * b_attn + (n - 1) * (b_conv + b_gn)
    return dict(b_attn=b_attn, b_conv=b_conv, b_gn=b_gn, total_buffer=total,
                df=df, pcpp=pcpp, cut=1.0 - pcpp / df)


def physical_bytes(model: str, H: int, W: int, n: int, p: float, elem_bytes: int,
                   kind: str = "pcpp_async") -> dict:
    """Bytes received by all ranks in one step, per class.

    kind: 'pcpp_async' | 'fullmap_async' | 'warmup'.
    """
    lay = layer_table(model, H, W)
    tot = {"attn": 0, "conv": 0, "gn": 0}
    if n == 1:
        return tot
    for L in lay:
        if L["kind"] == "attn":
            Hl, Wl, C = L["H_l"], L["W_l"], L["C"]
            if kind == "pcpp_async":
                r = band_rows(p, Hl // n)
                tot["attn"] += 2 * (n - 1) * r * Wl * 2 * C * B_CFG * elem_bytes
            else:
                tot["attn"] += (n - 1) * Hl * Wl * 2 * C * B_CFG * elem_bytes
        elif L["kind"] == "conv":
            mult = 2 if L["stride"] == 1 else 1
            e = 4 if L["C"] == 4 else elem_bytes          # conv_in reads the fp32 latent (reading D9)
            tot["conv"] += mult * (n - 1) * L["W_l"] * L["C"] * B_CFG * e
        else:
            tot["gn"] += n * (n - 1) * 2 * M.G_GROUPS * B_CFG * 8
    return tot
