"""CPU restatement of K4's table-driven FP64 exponential (csrc/evaluate.cu,
`exp_neg_scaled`) and its error bound.  No GPU: the bit-level algorithm is
replayed in numpy (FMAs emulated in long double) and compared with
long-double exp, pinning the constants and the <= 2.3e-16 (1 + |L|) relative
error per term that DESIGN.md §3/§4 rely on.  The kernel itself is checked
against the reference's goldens by the GPU tests."""

import math

import numpy as np

K = 2954.639443740597  # 2048 / ln 2 (evaluate.cu EXP_K)
C1, C2, C3 = 3.384507717577858e-04, 5.72744624517204e-08, 6.461528672932365e-12
SHIFT = 6755399441055744.0  # 1.5 * 2^52
NMIN = -1022 * 2048


def _fma(a, b, c):
    return (np.longdouble(a) * np.longdouble(b) + np.longdouble(c)).astype(np.float64)


def _table():
    """Table words as the host builds them: bits of 2^(j/2048) minus (j << 9) in the high word."""
    t = np.array([float(np.exp2(np.longdouble(j) / 2048)) for j in range(2048)])
    bits = t.view(np.uint64).copy()
    bits -= (np.arange(2048, dtype=np.uint64) << np.uint64(9)) << np.uint64(32)
    return bits


def exp_neg_scaled(d2, g, tab):
    s = _fma(d2, -g, SHIFT)
    nd = s - SHIFT
    f = _fma(-g, d2, -nd)
    sb = s.view(np.int64)
    lo = (sb & 0xFFFFFFFF).astype(np.uint64)
    tw = tab[(lo & np.uint64(2047)).astype(np.int64)]
    hi = ((tw >> np.uint64(32)) + (lo << np.uint64(9))) & np.uint64(0xFFFFFFFF)
    Ts = ((hi << np.uint64(32)) | (tw & np.uint64(0xFFFFFFFF))).view(np.float64)
    p = _fma(f, _fma(f, _fma(f, C3, C2), C1), 1.0)
    with np.errstate(all="ignore"):
        return np.where(sb >= np.int64(0x4338000000000000) + NMIN, Ts * p, 0.0)


def test_constants():
    ln2 = math.log(2.0)
    assert K == 2048 / ln2
    assert C1 == ln2 / 2048 and C2 == (ln2 / 2048) ** 2 / 2 and C3 == (ln2 / 2048) ** 3 / 6


def test_relative_error_bound():
    rng = np.random.default_rng(0)
    inv = np.exp(rng.uniform(-6, 6, 200_000))  # 1 / (2 w^2) over 5 decades of widths
    L = -rng.random(200_000) * np.where(rng.random(200_000) < 0.5, 3.0, 700.0)
    d2 = -L / inv
    g = inv * K
    e = exp_neg_scaled(d2, g, _table())
    ref = np.exp(-np.longdouble(d2) * np.longdouble(inv))
    rel = np.abs((e - ref) / ref).astype(np.float64)
    assert np.max(rel / (1.0 + np.abs(L))) <= 2.5e-16


def test_underflow_flush_and_zero():
    tab = _table()
    d2 = np.array([0.0, 707.0, 710.0, 745.5, 800.0, 1e6, 1e30, 1e300])
    e = exp_neg_scaled(d2, np.full(d2.size, K), tab)  # L = -d2
    assert e[0] == 1.0
    assert abs(e[1] / math.exp(-707.0) - 1) < 1e-12
    # below 2^-1022 (and far beyond the 1.5*2^52 shift range) the term is exactly 0
    assert np.all(e[2:] == 0.0)
