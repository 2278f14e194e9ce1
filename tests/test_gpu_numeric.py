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
