"""Noise schedule, DDIM update, classifier-free guidance, band-row rule.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* CFG, Eq. 2 (§3.1): eps_hat = eps_u + s (eps_c - eps_u), s = 5 (§4).
* Sampler: "50-step DDIM sampler" (§4).  The paper gives no schedule;
  reading D2: SDXL's public scheduler configuration --
  scaled_linear betas in [0.00085, 0.012] over 1000 training steps,
  'leading' spacing with steps_offset 1, final alpha_bar_prev = alpha_bar[0],
  eta = 0 (deterministic, no noise).
* Eq. 3-4: DDPM ancestral mean; provided for the closed-form pin that
  ties alpha, beta and alpha_bar together (not used by the DDIM sampler).
* rows(p, h): Eq. 1 takes "p h" rows of a neighbour; reading D1:
  floor(p h + 1e-9), at least one row when p > 0, at most h.

* DPM-Solver++(2M) (north star "DDIM/DPM-solver"; reading D23): data-prediction multistep on
  the same timestep ladder; first order at k = 0 (and at the last step when S < 15).

Pins (tests/test_oracle_schedule.py): alpha_bar = prod(1 - beta); DDIM step on
an exact x_tau = sqrt(ab) x0 + sqrt(1-ab) eps returns sqrt(ab') x0 +
sqrt(1-ab') eps; CFG identities s=1 -> eps_c, eps_c = eps_u -> eps_u; the
printed p values of Fig. 4 give integer row counts; DPM-Solver++ first
order == DDIM; on an exact trajectory every 2M step is exact; against the closed-form
solution of the data-prediction ODE for x0 linear in lambda the 2M sampler converges at
order 2 (the first-order sampler at order 1).
"""
from __future__ import annotations

import math

import numpy as np

NUM_TRAIN_TIMESTEPS = 1000
BETA_START = 0.00085
BETA_END = 0.012


def betas() -> np.ndarray:
    """scaled_linear: beta_t = (linspace(sqrt(b0), sqrt(b1), 1000))^2, t = 0..999."""
    return np.linspace(math.sqrt(BETA_START), math.sqrt(BETA_END),
                       NUM_TRAIN_TIMESTEPS, dtype=np.float64) ** 2


def alpha_bars() -> np.ndarray:
    """alpha_bar_t = prod_{s<=t} (1 - beta_s)  (P:70 'ᾱ_t = Π α_s')."""
    a = 1.0 - betas()
    out = np.empty_like(a)
    acc = 1.0
    for t in range(a.shape[0]):       # explicit running product, no cumprod
        acc *= a[t]
        out[t] = acc
    return out


def ddim_timesteps(num_steps: int) -> list[int]:
    """'leading' spacing with steps_offset=1: tau_k = (S-1-k)*(1000//S) + 1."""
    ratio = NUM_TRAIN_TIMESTEPS // num_steps
    return [(num_steps - 1 - k) * ratio + 1 for k in range(num_steps)]


def ddim_coeffs(num_steps: int, k: int) -> tuple[float, float, float, float]:
    """(alpha_bar_tau, alpha_bar_prev) -> the four DDIM scalars for step k.

    Returns (sqrt(ab), sqrt(1-ab), sqrt(ab_prev), sqrt(1-ab_prev)).
    prev timestep = tau - 1000//S; alpha_bar_prev = alpha_bar[0] when prev < 0
    (set_alpha_to_one = False, reading D2).
    """
    ab = alpha_bars()
    tau = ddim_timesteps(num_steps)[k]
    prev = tau - NUM_TRAIN_TIMESTEPS // num_steps
    a_t = ab[tau]
    a_p = ab[prev] if prev >= 0 else ab[0]
    return math.sqrt(a_t), math.sqrt(1.0 - a_t), math.sqrt(a_p), math.sqrt(1.0 - a_p)


def cfg_combine(eps_u: np.ndarray, eps_c: np.ndarray, s: float) -> np.ndarray:
    """Eq. 2: eps_hat = eps_u + s (eps_c - eps_u)."""
    return eps_u + s * (eps_c - eps_u)


def ddim_step(x: np.ndarray, eps_hat: np.ndarray, num_steps: int, k: int) -> np.ndarray:
    """Deterministic DDIM (eta = 0) update for step k (P:134 '50-step DDIM').

    x0_hat = (x - sqrt(1-ab) eps) / sqrt(ab);  x' = sqrt(ab') x0_hat + sqrt(1-ab') eps.
    """
    sa, s1a, sp, s1p = ddim_coeffs(num_steps, k)
    x0 = (x - s1a * eps_hat) / sa
    return sp * x0 + s1p * eps_hat


def dpmpp_2m_second_order(num_steps: int, k: int) -> bool:
    """Reading D23: DPM-Solver++(2M) takes a first-order step at k = 0 (no history) and, for
    S < 15, at the final step (diffusers' lower_order_final); second order otherwise."""
    if k == 0:
        return False
    if num_steps < 15 and k == num_steps - 1:
        return False
    return True


def _lam(ab: float) -> float:
    """lambda_t = log(alpha_t / sigma_t), alpha_t = sqrt(ab), sigma_t = sqrt(1 - ab)."""
    return 0.5 * math.log(ab) - 0.5 * math.log(1.0 - ab)


def dpmpp_2m_step(x: np.ndarray, eps_hat: np.ndarray, num_steps: int, k: int, x0_prev):
    """DPM-Solver++(2M) (Lu et al. 2022, data-prediction multistep, Algorithm 2) on the DDIM
    timestep ladder of reading D2 (north star: "the DDIM/DPM-solver scheduler update").

      x0_k = (x - sigma_k eps) / alpha_k,   h = lambda' - lambda_k
      first order:  x' = (sigma'/sigma_k) x - alpha' (e^{-h} - 1) x0_k        (== DDIM)
      second order: r = h_prev / h,  D = (1 + 1/(2r)) x0_k - (1/(2r)) x0_{k-1}
                    x' = (sigma'/sigma_k) x - alpha' (e^{-h} - 1) D

    Returns (x', x0_k); x0_k is the history the next step needs.
    """
    ab = alpha_bars()
    taus = ddim_timesteps(num_steps)
    step = NUM_TRAIN_TIMESTEPS // num_steps

    def abar(t):
        return ab[t] if t >= 0 else ab[0]

    a_t = abar(taus[k])
    a_p = abar(taus[k] - step)
    alpha_t, sigma_t = math.sqrt(a_t), math.sqrt(1.0 - a_t)
    alpha_p, sigma_p = math.sqrt(a_p), math.sqrt(1.0 - a_p)
    h = _lam(a_p) - _lam(a_t)
    x0 = (x - sigma_t * eps_hat) / alpha_t
    if dpmpp_2m_second_order(num_steps, k):
        h_prev = _lam(a_t) - _lam(abar(taus[k - 1]))
        r = h_prev / h
        D = (1.0 + 1.0 / (2.0 * r)) * x0 - (1.0 / (2.0 * r)) * x0_prev
    else:
        D = x0
    return (sigma_p / sigma_t) * x - alpha_p * math.expm1(-h) * D, x0


# ---- ancestral (DDPM, Eq. 3-4) sampling on the ladder; reading D24 ------------------------------
PHILOX_M = (0xD2E7470EE14C6C93, 0xCA5A826395121157)
PHILOX_W = (0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B)
_M64 = (1 << 64) - 1


def philox4x64_10(ctr, key):
    """Philox4x64-10 (Salmon et al., SC'11) on a 4 x 64-bit counter and 2 x 64-bit key, in Python
    integers.  Pinned against numpy.random.Philox (tests/test_oracle_schedule.py)."""
    c = [int(v) & _M64 for v in ctr]
    k0, k1 = int(key[0]) & _M64, int(key[1]) & _M64
    for _ in range(10):
        p0 = PHILOX_M[0] * c[0]
        p1 = PHILOX_M[1] * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k0, p1 & _M64, (p0 >> 64) ^ c[3] ^ k1, p0 & _M64]
        k0 = (k0 + PHILOX_W[0]) & _M64
        k1 = (k1 + PHILOX_W[1]) & _M64
    return c


def noise_token(seed: int, k: int, g: int) -> np.ndarray:
    """The 4 standard normals of latent token g (= global row * W + column) at step k (reading D24):
    words = Philox4x64-10(counter = (g, k, 0, 0), key = (seed, 0)); Box-Muller on the word pairs
    (w0, w1) and (w2, w3) with u = (w >> 11) * 2^-53 (u1 shifted by half an ulp so log(u1) is finite)."""
    w = philox4x64_10((g, k, 0, 0), (seed, 0))
    out = np.empty(4)
    for j in range(2):
        u1 = ((w[2 * j] >> 11) + 0.5) * 2.0 ** -53
        u2 = (w[2 * j + 1] >> 11) * 2.0 ** -53
        rad = math.sqrt(-2.0 * math.log(u1))
        out[2 * j] = rad * math.cos(2.0 * math.pi * u2)
        out[2 * j + 1] = rad * math.sin(2.0 * math.pi * u2)
    return out


def noise_patch(seed: int, k: int, row0: int, h: int, W: int) -> np.ndarray:
    """z for rows [row0, row0 + h) of the [H][W][4] latent at step k (pure-Python loop: small cases)."""
    z = np.empty((h, W, 4))
    for r in range(h):
        for w in range(W):
            z[r, w] = noise_token(seed, k, (row0 + r) * W + w)
    return z


def ancestral_coeffs(num_steps: int, k: int):
    """Reading D24: DDIM with eta = 1 on the D2 ladder (Song et al.: eta = 1 is the DDPM ancestral
    sampler) -- sigma^2 = (1 - ab')/(1 - ab) (1 - ab/ab'); returns (sqrt(ab), sqrt(1-ab), sqrt(ab'),
    sqrt(1 - ab' - sigma^2), sigma)."""
    sa, s1a, sp, s1p = ddim_coeffs(num_steps, k)
    a, ap = sa * sa, sp * sp
    var = (1.0 - ap) / (1.0 - a) * (1.0 - a / ap)
    return sa, s1a, sp, math.sqrt(max(1.0 - ap - var, 0.0)), math.sqrt(var)


def ancestral_step(x: np.ndarray, eps_hat: np.ndarray, num_steps: int, k: int, z: np.ndarray) -> np.ndarray:
    """x' = sqrt(ab') x0 + sqrt(1 - ab' - sigma^2) eps + sigma z,  x0 = (x - sqrt(1-ab) eps)/sqrt(ab).
    On the full 1000-step ladder the mean is Eq. 3 and sigma^2 the posterior variance, so this
    is Eq. 4 x_{t-1} = mu + sigma_t z."""
    sa, s1a, sp, ce, sig = ancestral_coeffs(num_steps, k)
    x0 = (x - s1a * eps_hat) / sa
    return sp * x0 + ce * eps_hat + sig * z


def ddpm_mean(x: np.ndarray, eps_hat: np.ndarray, t: int) -> np.ndarray:
    """Eq. 3: mu = (x_t - beta_t / sqrt(1 - ab_t) eps_hat) / sqrt(alpha_t)."""
    b = betas()[t]
    ab = alpha_bars()[t]
    return (x - b / math.sqrt(1.0 - ab) * eps_hat) / math.sqrt(1.0 - b)


def band_rows(p: float, h: int) -> int:
    """Eq. 1 'upper/lower p h of' a neighbour patch of height h.

    Reading D1: 0 if p == 0, else min(h, max(1, floor(p h + 1e-9))).
    """
    if not (0.0 <= p <= 1.0):
        raise ValueError("p must lie in [0, 1] (p > 1 is undefined, P:209 §6)")
    if p == 0.0:
        return 0
    return min(h, max(1, int(math.floor(p * h + 1e-9))))
