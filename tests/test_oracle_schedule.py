"""Pins for oracle/schedule.py against closed forms and the paper's numbers."""
import json
import math
import os

import numpy as np
import pytest

from oracle import schedule as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_alpha_bar_is_product_of_alphas():
    # P:70 §3.1: alpha_bar_t = prod_{s<=t} alpha_s; checked against numpy's cumprod
    b = S.betas()
    assert b.shape == (1000,)
    assert np.all(np.diff(b) > 0) and 0 < b[0] < b[-1] < 1
    np.testing.assert_allclose(S.alpha_bars(), np.cumprod(1.0 - b), rtol=1e-12)
    # scaled_linear endpoints (reading D2)
    assert math.isclose(b[0], 0.00085, rel_tol=1e-12) and math.isclose(b[-1], 0.012, rel_tol=1e-12)


def test_ddim_timesteps_leading_spacing():
    assert S.ddim_timesteps(4) == [751, 501, 251, 1]
    t50 = S.ddim_timesteps(json.load(open(os.path.join(GOLD, "paper_settings.json")))["ddim_steps"]["value"])
    assert len(t50) == 50 and t50[0] == 981 and t50[-1] == 1 and all(a - b == 20 for a, b in zip(t50, t50[1:]))


@pytest.mark.parametrize("steps", [4, 50])
def test_ddim_step_closed_form(steps):
    # P8: feeding the exact noise back reproduces the forward-marginal at tau_prev
    rng = np.random.default_rng(0)
    x0 = rng.standard_normal((8, 8, 4))
    eps = rng.standard_normal((8, 8, 4))
    ab = S.alpha_bars()
    taus = S.ddim_timesteps(steps)
    for k, tau in enumerate(taus):
        x = math.sqrt(ab[tau]) * x0 + math.sqrt(1 - ab[tau]) * eps
        prev = tau - 1000 // steps
        ap = ab[prev] if prev >= 0 else ab[0]
        want = math.sqrt(ap) * x0 + math.sqrt(1 - ap) * eps
        np.testing.assert_allclose(S.ddim_step(x, eps, steps, k), want, atol=1e-12, rtol=0)


def test_cfg_identities():
    rng = np.random.default_rng(1)
    u, c = rng.standard_normal(16), rng.standard_normal(16)
    np.testing.assert_allclose(S.cfg_combine(u, c, 1.0), c, atol=1e-15)   # s = 1 -> eps_c
    np.testing.assert_array_equal(S.cfg_combine(u, u, 5.0), u)          # eps_c = eps_u -> eps_u
    np.testing.assert_allclose(S.cfg_combine(np.zeros(16), c, 5.0), 5 * c)  # s = 5
    # linearity: cfg(a,b,s) + cfg(b,a,s) = a + b
    np.testing.assert_allclose(S.cfg_combine(u, c, 5.0) + S.cfg_combine(c, u, 5.0), u + c, atol=1e-12)


def test_ddpm_mean_closed_form():
    # Eq. 3 with eps_hat = 0 is x / sqrt(alpha_t); with x = sqrt(ab) x0 + sqrt(1-ab) eps and
    # eps_hat = eps it equals the posterior mean coefficient form (Ho et al. Eq. 11)
    rng = np.random.default_rng(2)
    x = rng.standard_normal(10)
    t = 500
    a = 1 - S.betas()[t]
    np.testing.assert_allclose(S.ddpm_mean(x, np.zeros(10), t), x / math.sqrt(a), rtol=1e-14)
    x0, e = rng.standard_normal(10), rng.standard_normal(10)
    ab, abp = S.alpha_bars()[t], S.alpha_bars()[t - 1]
    xt = math.sqrt(ab) * x0 + math.sqrt(1 - ab) * e
    b = S.betas()[t]
    post = (math.sqrt(abp) * b / (1 - ab)) * x0 + (math.sqrt(a) * (1 - abp) / (1 - ab)) * xt
    np.testing.assert_allclose(S.ddpm_mean(xt, e, t), post, atol=1e-12)


def test_band_rows_rule():
    # Eq. 1 'p h' rows; reading D1: floor with 1e-9 guard, >=1 when p>0, <=h
    assert S.band_rows(0.0, 16) == 0
    assert S.band_rows(0.25, 16) == 4
    assert S.band_rows(1.0, 16) == 16
    assert S.band_rows(0.3, 10) == 3          # 0.3*10 = 2.9999999999999996 in binary
    assert S.band_rows(0.01, 4) == 1
    assert S.band_rows(0.8, 8) == 6 and S.band_rows(0.8, 4) == 3
    for h in range(1, 129):
        prev = 0
        for k in range(0, 1001):
            r = S.band_rows(k / 1000, h)
            assert 0 <= r <= h and r >= prev          # monotone in p
            if k:
                assert r == min(h, max(1, (k * h) // 1000))   # exact integer form of floor(p h)
            prev = r
    with pytest.raises(ValueError):
        S.band_rows(1.5, 8)                       # p > 1 undefined


# ---- DPM-Solver++(2M) (north star "DDIM/DPM-solver"; reading D23) --------------------------------
from oracle import schedule as SCH  # noqa: E402  (S is used for step counts below)

def test_dpmpp_first_order_equals_ddim():
    """The first-order DPM-Solver++ update is algebraically the DDIM (eta = 0) update."""
    rng = np.random.default_rng(7)
    x = rng.standard_normal((8, 8, 4))
    e = rng.standard_normal((8, 8, 4))
    for S, k in [(50, 0), (4, 0), (4, 3), (10, 9)]:
        ref = SCH.ddim_step(x, e, S, k)
        got, _ = SCH.dpmpp_2m_step(x, e, S, k, x0_prev=np.full_like(x, 1e9))   # history must be ignored
        assert np.max(np.abs(got - ref)) <= 1e-12 * (1 + np.max(np.abs(ref)))


def test_dpmpp_exact_on_exact_trajectory():
    """If the model returns the true eps of x_tau = alpha x0 + sigma eps, every 2M step lands on
    alpha' x0 + sigma' eps (x0 predictions agree, so the second-order correction vanishes)."""
    rng = np.random.default_rng(8)
    x0 = rng.standard_normal((4, 4, 4))
    eps = rng.standard_normal((4, 4, 4))
    S = 20
    ab = SCH.alpha_bars()
    taus = SCH.ddim_timesteps(S)
    x = math.sqrt(ab[taus[0]]) * x0 + math.sqrt(1 - ab[taus[0]]) * eps
    hist = None
    for k in range(S):
        x, hist = SCH.dpmpp_2m_step(x, eps, S, k, hist)
        prev = taus[k] - 1000 // S
        a = ab[prev] if prev >= 0 else ab[0]
        assert np.max(np.abs(x - (math.sqrt(a) * x0 + math.sqrt(1 - a) * eps))) <= 1e-10


def _one_step_errors(a, b, S):
    """Local error of one step from tau_k (k = S/2: the same point of the ladder for every S) for
    the "model" x0(lambda) = a + b lambda, against the closed-form solution of the data-prediction
    ODE x'/sigma' = x/sigma + F(lambda') - F(lambda), F(lam) = e^lam (a + b (lam - 1)); the 2M
    history is the exact x0 at the previous ladder point."""
    ab = SCH.alpha_bars()
    taus = SCH.ddim_timesteps(S)
    k = S // 2
    at, ap, aq = ab[taus[k]], ab[taus[k] - 1000 // S], ab[taus[k - 1]]
    lt, lp, lq = SCH._lam(at), SCH._lam(ap), SCH._lam(aq)
    F = lambda lam: math.exp(lam) * (a + b * (lam - 1.0))
    x = np.array([0.8])
    exact = math.sqrt(1 - ap) * (x[0] / math.sqrt(1 - at) + F(lp) - F(lt))
    eps = (x - math.sqrt(at) * (a + b * lt)) / math.sqrt(1 - at)
    x2, _ = SCH.dpmpp_2m_step(x, eps, S, k, np.array([a + b * lq]))
    x1 = SCH.ddim_step(x, eps, S, k)
    return abs(float(x2[0]) - exact), abs(float(x1[0]) - exact)


def test_dpmpp_2m_local_order():
    """One 2M step has local error O(h^3) (falls ~8x per halving of the step), the first-order
    (DDIM) step O(h^2) (~4x): a dropped, mis-signed or mis-weighted history term breaks the order."""
    e2, e1 = zip(*[_one_step_errors(0.3, -0.7, S) for S in (20, 40, 100)])
    assert 6.0 < e2[0] / e2[1] < 10.0, e2
    assert 3.0 < e1[0] / e1[1] < 5.0, e1
    assert e2[2] < e1[2] / 20, (e1, e2)


# ---- ancestral sampler (Eq. 3-4; reading D24) ------------------------------------------------------

def test_philox_matches_numpy():
    """The oracle's Philox4x64-10 equals numpy's Philox bit generator (which advances its counter
    before each block: Philox(counter=c) produces philox(c + 1))."""
    for key, ctr in [((5, 0), (0, 0, 0, 0)), ((2**63 + 12345, 77), (41, 3, 0, 0)), ((0, 0), (2**64 - 2, 9, 1, 0))]:
        bg = np.random.Philox(key=np.array(key, dtype=np.uint64), counter=np.array(ctr, dtype=np.uint64))
        want = [int(v) for v in bg.random_raw(4)]
        c1 = list(ctr)
        c1[0] = (c1[0] + 1) % 2**64
        if c1[0] == 0:
            c1[1] += 1
        assert SCH.philox4x64_10(c1, key) == want


def test_noise_is_standard_normal():
    z = np.concatenate([SCH.noise_token(3, k, g) for k in range(4) for g in range(2500)])
    assert abs(z.mean()) < 0.03 and abs(z.std() - 1.0) < 0.03
    assert abs(np.mean(z ** 4) - 3.0) < 0.2                    # Gaussian kurtosis
    assert SCH.noise_token(3, 1, 7).tolist() != SCH.noise_token(3, 2, 7).tolist()


def test_ancestral_reduces_to_eq3_eq4_on_full_ladder():
    """With S = 1000 (adjacent timesteps) the eta = 1 update's mean is Eq. 3's mu and its variance
    the DDPM posterior variance (1 - ab_{t-1})/(1 - ab_t) beta_t: the sampler is Eq. 4."""
    rng = np.random.default_rng(4)
    x = rng.standard_normal((4, 4, 4))
    e = rng.standard_normal((4, 4, 4))
    ab = SCH.alpha_bars()
    be = SCH.betas()
    for k in (1, 500, 998):                     # tau_0 = 1000 lies past the 1000-entry table
        t = SCH.ddim_timesteps(1000)[k]
        mean = SCH.ancestral_step(x, e, 1000, k, np.zeros_like(x))
        np.testing.assert_allclose(mean, SCH.ddpm_mean(x, e, t), rtol=1e-9, atol=1e-9)
        sig = SCH.ancestral_coeffs(1000, k)[4]
        assert abs(sig ** 2 - (1 - ab[t - 1]) / (1 - ab[t]) * be[t]) <= 1e-12


def test_box_muller_known_answer_invariants():
    """Reading D24's z, pinned by invariants of the Box-Muller map rather than its formula: for each
    word pair, z_a^2 + z_b^2 = -2 ln u1 and atan2(z_b, z_a) = 2 pi u2 (mod 2 pi), with u1, u2 the
    documented 53-bit uniforms of numpy's independent Philox4x64 words.  A swapped cos / sin, a wrong
    shift or a mis-paired word fails one of them."""
    import math
    from oracle.schedule import noise_token
    for seed, k, g in ((0, 0, 0), (12, 3, 517), (2 ** 40 + 7, 49, 65535)):
        # numpy's Philox increments its 256-bit counter before the first block: start one below (g, k, 0, 0)
        c = (g + (k << 64) - 1) % (1 << 256)
        bg = np.random.Philox(counter=np.array([(c >> (64 * i)) & (2 ** 64 - 1) for i in range(4)], dtype=np.uint64),
                              key=np.array([seed, 0], dtype=np.uint64))
        words = [int(v) for v in bg.random_raw(4)]
        z = noise_token(seed, k, g)
        for j in range(2):
            u1 = ((words[2 * j] >> 11) + 0.5) * 2.0 ** -53
            u2 = (words[2 * j + 1] >> 11) * 2.0 ** -53
            za, zb = z[2 * j], z[2 * j + 1]
            assert abs(za * za + zb * zb - (-2.0 * math.log(u1))) <= 1e-12 * max(1.0, -2.0 * math.log(u1))
            ang = math.atan2(zb, za) % (2 * math.pi)
            assert abs(ang - (2 * math.pi * u2) % (2 * math.pi)) <= 1e-9
