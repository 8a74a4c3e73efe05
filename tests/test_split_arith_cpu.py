"""CPU emulation of the tensor paths' split arithmetic (no GPU): the FP16
hi/lo products the tcgen05 kernels accumulate in FP32, for

  * the difference form of contract_tc.cu / contract_tcw.cu: a = x - z in FP32,
    a s_i = ah + al (s_i a power of two from max |a_i|), u 2^15 = uh + ul,
    y s_i 2^15 ~ sum(uh ah + uh al + ul ah);
  * the pre-split form of contract_tcp.cu: x s_i = bh + bl once per dataset
    (s_i from max |x_i|), y = acc inv_i + Delta with Delta = fp32(<u, -z>),
    evaluated as one FMA.

Both must give the sign of the FP64 y = <u, x_i - z> for every pair outside
the halfspace tie zone |y| < 1e-6 max(|x_i|, |z|) (the tier-1 contract,
SURVEY §8c), on the cases that stress them: offset data (|x| >> spread), far
queries, heterogeneous coordinate scales, d = 50 and d = 200.  Rows equal to
the query are exact ties on the tensor paths by construction (a = 0) or by
index (contract_tcp's coinciding-row list) and are left out here.
"""

import numpy as np
import pytest

TIE_REL = 1e-6


def _split16(v32):
    """hi = fp16(v), lo = fp16(v - hi) with the residual formed in FP32 (the kernels' order)."""
    hi = v32.astype(np.float16)
    lo = (v32 - hi.astype(np.float32)).astype(np.float16)
    return hi.astype(np.float32), lo.astype(np.float32)


def _dir_split(U):
    v = U * 32768.0  # FP64, rounded straight to FP16 (__double2half)
    hi = v.astype(np.float16)
    lo = (v - hi.astype(np.float64)).astype(np.float16)
    return hi.astype(np.float32), lo.astype(np.float32)


def _pow2_scale(mx):
    """s = 2^(14 - E) with mx < 2^E (E clamped as the kernels do); 0 for mx == 0."""
    _, e = np.frexp(mx.astype(np.float32))
    e = np.maximum(e, -100)
    return np.where(mx > 0, np.ldexp(np.float32(1.0), 14 - e).astype(np.float32), np.float32(0.0)), e


def _acc(uh, ul, bh, bl):
    # FP16 x FP16 products are exact in FP32; FP32 accumulation (sequential here)
    prods = (uh[None, :, :] * bh[:, None, :] + uh[None, :, :] * bl[:, None, :] + ul[None, :, :] * bh[:, None, :])
    return prods.astype(np.float32).sum(axis=2, dtype=np.float32)


def _difference_form(X, z, U):
    a = (X.astype(np.float32) - z.astype(np.float32)[None, :]).astype(np.float32)
    s, _ = _pow2_scale(np.abs(a).max(axis=1))
    bh, bl = _split16((a * s[:, None]).astype(np.float32))
    uh, ul = _dir_split(U)
    return _acc(uh, ul, bh, bl)  # sign only (the per-point scale is positive)


def _presplit_form(X, z, U):
    x32 = X.astype(np.float32)
    s, e = _pow2_scale(np.abs(x32).max(axis=1))
    inv = np.where(s > 0, np.ldexp(np.float32(1.0), e - 29), np.float32(0.0)).astype(np.float32)
    bh, bl = _split16((x32 * s[:, None]).astype(np.float32))
    uh, ul = _dir_split(U)
    acc = _acc(uh, ul, bh, bl)
    delta = (U @ (-z)).astype(np.float32) + np.float32(0.0)  # FP64 shift rounded to FP32, no -0
    # one FMA: acc * inv exact (power of two), + delta rounded once
    return (acc.astype(np.float64) * inv[:, None].astype(np.float64) + delta[None, :].astype(np.float64)).astype(
        np.float32)


CASES = ["gauss", "offset", "far", "hetero"]


@pytest.mark.parametrize("d", [50, 200])
@pytest.mark.parametrize("case", CASES)
def test_split_signs_outside_tie_zone(case, d):
    rng = np.random.default_rng(7 + d)
    n, m = 600, 48
    X = rng.standard_normal((n, d))
    if case == "offset":
        X = X + 500.0
    if case == "hetero":
        X = X * rng.uniform(0.05, 20.0, size=d)
    z = X[3] + 1e-3 * rng.standard_normal(d)
    if case == "far":
        z = X[3] + 1e3
    U = rng.standard_normal((m, d))
    U /= np.linalg.norm(U, axis=1)[:, None]
    y = X @ U.T - (U @ z)[None, :]
    zone = np.abs(y) < TIE_REL * np.maximum(np.linalg.norm(X, axis=1), np.linalg.norm(z))[:, None]
    for form in (_difference_form, _presplit_form):
        got = form(X, z, U)
        wrong = (np.sign(got) != np.sign(y)) & ~zone
        assert not wrong.any(), (form.__name__, case, d, int(wrong.sum()))
