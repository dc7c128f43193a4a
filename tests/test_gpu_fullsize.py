"""Parity at the bench workload's full sizes (1024^2 SDXL-shaped step, n = 1, bf16, the launch
configurations bench.py times), on sampled outputs the oracle's definitions compute one by one:
conv3x3 / 1x1 GEMMs of every level (incl. split-K and stride 2), partially conditioned attention
at level 1 and level 2, and GroupNorm.  Tolerance: bf16 storage with fp32 accumulation."""
import numpy as np
import pytest

from oracle import model as M
from paper_2412_02962_b200 import inputs, pcpp

pytestmark = pytest.mark.gpu


def bf(x):
    return inputs.round_to_bf16(np.asarray(x, np.float32)).astype(np.float64)


def T(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda().to(torch.bfloat16)


# (rows_in, W_in, Cin, Cout, taps, stride): level 0/1/2 convs, the up-block concat widths, 1x1s
SHAPES = [(128, 128, 320, 320, 9, 1), (64, 64, 640, 640, 9, 1), (32, 32, 1280, 1280, 9, 1),
          (32, 32, 2560, 1280, 9, 1), (128, 128, 960, 320, 9, 1), (128, 128, 320, 320, 9, 2),
          (64, 64, 640, 640, 9, 2), (32, 32, 1280, 3840, 1, 1), (64, 64, 1920, 640, 1, 1)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_conv_fullsize_sampled(cuda_ok, shape):
    import torch
    rows, W, Cin, Cout, taps, stride = shape
    rng = np.random.default_rng(1)
    pad = 1 if taps == 9 else 0
    x = bf(rng.standard_normal((rows + 2 * pad, 2, W, Cin)))
    w = bf(rng.standard_normal((Cout, 3, 3, Cin) if taps == 9 else (Cout, Cin)) / np.sqrt(taps * Cin))
    bias = rng.standard_normal(Cout).astype(np.float32)
    ro, wo = rows // stride, W // stride
    res = bf(rng.standard_normal((ro, 2, wo, Cout)))
    y = torch.empty((ro, 2, wo, Cout), device="cuda", dtype=torch.bfloat16)
    pcpp.pcpp_op_conv(T(x), rows, 2, W, Cin, taps, stride, T(w), torch.from_numpy(bias).cuda(), None, T(res), y, Cout)
    torch.cuda.synchronize()
    got = y.float().cpu().numpy()
    idx = [(rng.integers(ro), rng.integers(2), rng.integers(wo), rng.integers(Cout)) for _ in range(256)]
    idx += [(0, 0, 0, 0), (ro - 1, 1, wo - 1, Cout - 1), (0, 1, wo - 1, 3), (ro - 1, 0, 0, Cout // 2)]
    err = 0.0
    for (r, b, c, n) in idx:
        acc = bias[n] + res[r, b, c, n]
        if taps == 9:
            for dr in range(3):
                for dw in range(3):
                    ri, wi = r * stride + dr - 1, c * stride + dw - 1
                    if 0 <= wi < W:
                        acc += x[ri + 1, b, wi] @ w[n, dr, dw]
        else:
            acc += x[r, b, c] @ w[n]
        err = max(err, abs(got[r, b, c, n] - acc) / (1.0 + abs(acc)))
    assert err < 2e-2, err


@pytest.mark.parametrize("geo", [(64, 64, 640, (64,)), (32, 32, 1280, (32,)), (8, 64, 640, (6, 8, 6))])
def test_attention_fullsize_sampled(cuda_ok, geo):
    import torch
    h, W, Cm, rows = geo
    rng = np.random.default_rng(2)
    q = bf(rng.standard_normal((h, 2, W, Cm)))
    srcs = [bf(rng.standard_normal((r, 2, W, 2 * Cm))) for r in rows]
    out = torch.empty((h, 2, W, Cm), device="cuda", dtype=torch.bfloat16)
    pcpp.pcpp_op_attention(T(q), [T(s) for s in srcs], list(rows), h, 2, W, Cm, out)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    K = np.concatenate([s[..., :Cm] for s in srcs], axis=0)
    V = np.concatenate([s[..., Cm:] for s in srcs], axis=0)
    worst = 0.0
    for _ in range(12):
        r, b, w = rng.integers(h), rng.integers(2), rng.integers(W)
        for hd in range(Cm // 64):
            sl = slice(hd * 64, hd * 64 + 64)
            s = (K[:, b, :, sl].reshape(-1, 64) @ q[r, b, w, sl]) / 8.0
            p = M._softmax_rows(s[None])[0]
            ref = p @ V[:, b, :, sl].reshape(-1, 64)
            worst = max(worst, np.abs(got[r, b, w, sl] - ref).max() / (np.abs(ref).max() + 1e-3))
    assert worst < 2e-2, worst


@pytest.mark.parametrize("shape", [(128, 128, 320), (64, 64, 1920), (32, 32, 2560)])
def test_groupnorm_fullsize(cuda_ok, shape):
    import torch
    rows, W, Cm = shape
    rng = np.random.default_rng(3)
    x = bf(rng.standard_normal((rows, 2, W, Cm)) * 1.5 + 0.3)
    g = (1 + 0.1 * rng.standard_normal(Cm)).astype(np.float32)
    be = (0.1 * rng.standard_normal(Cm)).astype(np.float32)
    y = torch.empty((rows, 2, W, Cm), device="cuda", dtype=torch.bfloat16)
    m = torch.empty((2, 32, 2), device="cuda", dtype=torch.float64)
    pcpp.pcpp_op_groupnorm(T(x), rows, 2, W, Cm, torch.from_numpy(g).cuda(), torch.from_numpy(be).cuda(), 1, y, m)
    torch.cuda.synchronize()
    ctx = M.Ctx(1, 0.0, "sync")
    ref = M.group_norm(ctx, [np.transpose(x, (1, 0, 2, 3))], g.astype(np.float64), be.astype(np.float64), True)[0]
    np.testing.assert_allclose(m.cpu().numpy(), ctx.nxt[("gn0", "m")][0], rtol=1e-6, atol=1e-3)
    got = np.transpose(y.float().cpu().numpy(), (1, 0, 2, 3))
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-2


@pytest.mark.parametrize("n", [1, 2])
def test_bench_workload_bf16_matches_fp32_path(cuda_ok, n):
    """The bench's whole 1024^2 step, in the launch configuration bench.py times (tcgen05 kernels,
    GEMM table profiles/gemm_tune_b200.txt, CUDA graphs), against the same plan in fp32 with the
    SIMT kernels -- the path the oracle parity tests pin at small sizes: one DDIM step (and, for
    n = 2, the warm-up then an async step with stale bands) agree to the bf16 tolerance."""
    import torch
    blob = inputs.make_weight_blob(inputs.init_specs(pcpp.manifest("sdxl")))
    xT = np.array(inputs.make_latent(128, 128), dtype=np.float32)
    cond = inputs.make_cond(1280)
    p, w = (0.0, 0) if n == 1 else (0.3, 1)
    steps = 1 if n == 1 else 2
    outs = {}
    for prec, kern in (("bf16", "auto"), ("fp32", "simt")):
        cfg = pcpp.make_config(model="sdxl", num_steps=50, precision=prec, kernels=kern)
        plan = pcpp.Plan(128, 128, 4, n, p, w, cfg, blob)
        plan.pcpp_set_cond(cond)
        lat = torch.from_numpy(xT.copy()).cuda()
        for k in range(steps):
            plan.pcpp_step(lat, k)
        torch.cuda.synchronize()
        outs[prec] = lat.cpu().numpy().astype(np.float64)
        plan.close()
    err = float(np.linalg.norm(outs["bf16"] - outs["fp32"]) / np.linalg.norm(outs["fp32"]))
    assert err <= 2e-2, err


@pytest.mark.parametrize("geo", [(256, 4, 0.8, "fp32"), (480, 8, 0.8, "bf16")], ids=["X2-2048px-n4", "X3-3840px-n8"])
def test_large_resolution_tc_matches_simt_path(cuda_ok, geo):
    """SURVEY §8(d) X2 / X3 geometries (256^2 and 480^2 latents, the paper's 2048^2 / 3840^2 images) in
    the loopback backend (all n ranks on this GPU): the warm-up step (full-map attention over 16k /
    57.6k tokens per head) and one async step with stale bands, tcgen05 bf16 path vs the SIMT path
    (fp32 at X2; bf16 storage at X3, where 8 fp32 rank arenas exceed one GPU's HBM).  Exercises
    > 2^31-byte activation offsets, thousands of GEMM / attention tiles and the arena memory plan."""
    import torch
    H, n, p, ref_prec = geo
    blob = inputs.make_weight_blob(inputs.init_specs(pcpp.manifest("sdxl")))
    xT = np.array(inputs.make_latent(H, H), dtype=np.float32)
    cond = inputs.make_cond(1280)
    outs = {}
    for key, prec, kern in (("tc", "bf16", "auto"), ("simt", ref_prec, "simt")):
        cfg = pcpp.make_config(model="sdxl", num_steps=50, precision=prec, kernels=kern)
        plan = pcpp.Plan(H, H, 4, n, p, 1, cfg, blob)
        plan.pcpp_set_cond(cond)
        lat = torch.from_numpy(xT.copy()).cuda()
        xs = []
        for k in range(2):
            plan.pcpp_step(lat, k)
            torch.cuda.synchronize()
            xs.append(lat.cpu().numpy().astype(np.float64))
        outs[key] = xs
        plan.close()
        del lat
        torch.cuda.empty_cache()
    for k in range(2):
        a, b = outs["tc"][k], outs["simt"][k]
        assert np.isfinite(a).all(), k
        err = float(np.linalg.norm(a - b) / np.linalg.norm(b))
        assert err <= 2e-2, (k, err)
