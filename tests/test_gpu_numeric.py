"""Device numeric core vs the reference's WidenedFloat64 ops (interval.hpp:38-103),
bit-for-bit, on edge cases and random operands (proj/tests/test_interval.cpp)."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

EDGE = [0.0, -0.0, 1.0, -1.0, 0.1, 0.2, 0.3, 1e-300, -1e-300, 5e-324, -5e-324, 2.2250738585072014e-308,
        1.7976931348623157e308, -1.7976931348623157e308, np.inf, -np.inf, 2.0 ** -500, 2.0 ** -501, 2.0 ** 1020,
        2.0 ** 1023, 3.0, 1.0 / 3.0, 2.0 ** -80, 1.5, 2.5, 1e16, 1e-16, 0.5]


def gpu_ops(op, a, b):
    from paper_2007_10868_b200 import _lib
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    out = np.empty_like(a)
    vp = ctypes.c_void_p
    _lib.check(_lib.lib.pc_scalar_ops(op, a.ctypes.data_as(vp), b.ctypes.data_as(vp),
                                      out.ctypes.data_as(vp), len(a)))
    return out


def operands():
    rng = np.random.default_rng(20260801)
    e = np.array(EDGE)
    A, B = np.meshgrid(e, e)
    a, b = [A.ravel()], [B.ravel()]
    n = 400_000
    mant = rng.random(n) - 0.5
    for scale in (1e-6, 1e6, 64.0, 1.0, 1e-150, 1e150, 1e300):
        a.append(mant * scale)
        b.append((rng.random(n) - 0.5) * scale)
    # near-cancelling pairs, exact dyadic pairs, random bit patterns
    x = rng.random(n)
    a.append(x); b.append(-x * (1 + rng.integers(-3, 4, n) * 2.0 ** -52))
    a.append(rng.integers(-64, 65, n) / 64.0); b.append(rng.integers(-256, 257, n) / 256.0)
    bits = rng.integers(0, 2 ** 63, 2 * n, dtype=np.int64).view(np.float64)
    bits = bits[np.isfinite(bits)]
    m = len(bits) // 2
    a.append(bits[:m]); b.append(bits[m:2 * m])
    return np.concatenate(a), np.concatenate(b)


def same_bits(x, y):
    return np.array_equal(x.view(np.int64), y.view(np.int64))


@pytest.mark.parametrize("op", [0, 1, 2, 3, 4, 5, 6])
def test_scalar_ops_match_reference(port, op):
    a, b = operands()
    if op in (4, 5):  # the reference only divides by positive intervals' endpoints
        b = np.abs(b)
        b[b == 0] = 1.0
    g = gpu_ops(op, a, b)
    r = port.scalar_ops(op, a, b)
    bad = ~((g == r) | (np.isnan(g) & np.isnan(r)))
    assert not bad.any(), (op, a[bad][:4], b[bad][:4], g[bad][:4], r[bad][:4])
    nn = ~np.isnan(r)
    assert same_bits(g[nn], r[nn]), op


def test_direction_generic_add(port):
    a, b = operands()
    assert same_bits(gpu_ops(7, a, b), port.scalar_ops(1, a, b))
    assert same_bits(gpu_ops(8, a, b), port.scalar_ops(0, a, b))


def test_nextafter_bits():
    a, _ = operands()
    a = a[~np.isnan(a)]
    assert same_bits(gpu_ops(9, a, a), np.nextafter(a, np.inf))
    assert same_bits(gpu_ops(10, a, a), np.nextafter(a, -np.inf))


def test_band_forms(port):
    """madd_band's compare-free outward steps (kernels.cuh) equal the reference
    ops for every in-band operand: products with |a*b| in [2^-499, 2^999] (or a
    zero factor), sums of operands below 2^1000 (zero results compare by value:
    the band forms may give -0 where the reference gives +0)."""
    a, b = operands()
    fin = np.isfinite(a) & np.isfinite(b)
    a, b = a[fin], b[fin]
    with np.errstate(all="ignore"):
        p = np.abs(a * b)
    pm = (a == 0) | (b == 0) | ((p >= 2.0 ** -499) & (p <= 2.0 ** 999))
    sm = (np.abs(a) < 2.0 ** 1000) & (np.abs(b) < 2.0 ** 1000) & \
         ((a == 0) | (np.abs(a) >= 2.0 ** -520)) & ((b == 0) | (np.abs(b) >= 2.0 ** -520))
    for op, ref, m in ((11, 2, pm), (12, 3, pm), (13, 0, sm), (14, 1, sm)):
        g, r = gpu_ops(op, a[m], b[m]), port.scalar_ops(ref, a[m], b[m])
        assert np.array_equal(g, r), (op, np.flatnonzero(g != r)[:4])
        nz = r != 0
        assert same_bits(g[nz], r[nz]), op


def gpu_chain_fold(acc0, terms, up):
    from paper_2007_10868_b200 import _lib
    acc0 = np.ascontiguousarray(acc0, dtype=np.float64)
    terms = np.ascontiguousarray(terms, dtype=np.float64)
    upa = np.ascontiguousarray(up, dtype=np.int32)
    out = np.empty_like(acc0)
    vp = ctypes.c_void_p
    _lib.check(_lib.lib.pc_chain_fold(terms.shape[0], terms.shape[1], acc0.ctypes.data_as(vp),
                                      terms.ctypes.data_as(vp), upa.ctypes.data_as(vp),
                                      out.ctypes.data_as(vp)))
    return out


def chain_cases(rng, n_chains, length):
    """Adversarial chains for the scan fold (scanfold.cuh): every regime that
    must leave the integer scan (ties, binade and sign changes, zero and
    subnormal accumulators, huge / infinite / tiny terms) next to the common
    one (many small inexact terms on a large accumulator)."""
    T = np.empty((n_chains, length))
    A = np.empty(n_chains)
    for c in range(n_chains):
        kind = c % 12
        if kind == 0:    # the common regime: random terms, |acc| >> |t|
            T[c] = rng.standard_normal(length) * 1e-3
            A[c] = rng.standard_normal() * 10
        elif kind == 1:  # dyadic terms: exact adds and exact half-ulp ties
            A[c] = 1.0 + rng.integers(0, 2 ** 20) * 2.0 ** -52
            T[c] = rng.integers(-4, 5, length) * 2.0 ** -53
        elif kind == 2:  # random walk through zero: sign and binade changes
            A[c] = 0.0
            T[c] = rng.standard_normal(length)
        elif kind == 3:  # accumulator near a power of two
            A[c] = 2.0 ** rng.integers(-20, 20)
            T[c] = rng.standard_normal(length) * 2.0 ** -45 * A[c]
        elif kind == 4:  # tiny terms, sometimes below the accumulator's ulp
            A[c] = rng.standard_normal()
            T[c] = rng.standard_normal(length) * 10.0 ** rng.integers(-40, -10, length)
        elif kind == 5:  # huge terms, infinities, zeros, NaN (no term)
            A[c] = rng.standard_normal() * 1e3
            T[c] = rng.standard_normal(length)
            m = rng.integers(0, 50, length)
            T[c][m == 0] = 1e300
            T[c][m == 1] = -1e300
            T[c][m == 2] = 0.0
            T[c][m == 3] = -0.0
            T[c][m == 4] = np.nan
            T[c][m == 5] = np.inf if c % 24 == 5 else T[c][m == 5]
        elif kind == 6:  # subnormal region
            A[c] = 5e-324 * rng.integers(1, 1000)
            T[c] = rng.standard_normal(length) * 1e-310
        elif kind == 7:  # signed zero starts, then exact cancellations
            A[c] = -0.0
            x = rng.integers(-8, 9, length) / 8.0
            T[c] = np.where(np.arange(length) % 2, -np.roll(x, 1), x)
        elif kind == 8:  # terms comparable to the accumulator (every link changes binade often)
            A[c] = rng.standard_normal()
            T[c] = rng.standard_normal(length) * np.abs(A[c])
        elif kind == 9:  # row-constant shape: bias products c*b, b = k/64
            A[c] = rng.integers(-32, 33) / 64.0
            T[c] = rng.standard_normal(length) * 1e-2 * rng.integers(-32, 33, length) / 64.0
        elif kind == 10:  # large magnitudes near the scan's exponent limits
            A[c] = 2.0 ** rng.integers(800, 1000) * rng.standard_normal()
            T[c] = rng.standard_normal(length) * 2.0 ** rng.integers(700, 1010)
        else:            # very small magnitudes near the limits
            A[c] = 2.0 ** rng.integers(-1000, -800) * rng.standard_normal()
            T[c] = rng.standard_normal(length) * 2.0 ** rng.integers(-1070, -820)
    return A, T


@pytest.mark.parametrize("length", [1, 31, 33, 1000, 5000])
def test_chain_fold_matches_serial(port, length):
    """The warp-scan fold == the reference's serial add_up / add_down chain,
    bit for bit, on both directions."""
    rng = np.random.default_rng(length)
    A, T = chain_cases(rng, 96, length)
    for upv in (0, 1, 2, 3, 4, 5, 8, 9, 20, 21):  # bit 0: add_up; 1: 32-link warp scan; 2: CTA scan; 3: prefetching warp scan; 4 (with 2): CTA scan with local retry
        up = np.full(len(A), upv, dtype=np.int32)
        up[::3] ^= 1
        g = gpu_chain_fold(A, T, up)
        r = port.chain_fold(A, T, up & 1)  # noqa: the device variant is chosen by the other bits
        bad = ~((g.view(np.int64) == r.view(np.int64)) | (np.isnan(g) & np.isnan(r)))
        assert not bad.any(), (np.nonzero(bad)[0][:8] % 12, g[bad][:4], r[bad][:4])
