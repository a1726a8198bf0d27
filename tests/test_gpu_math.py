"""The device fp64 division / square-root fast paths (FastMath in
csrc/hydro_physics.cuh) against the compiler's IEEE `/` and sqrt() on the
same B200: wherever the fast path reports itself in range, the bits must be
identical; outside its range the kernels recompute with the IEEE operation,
so only the in-range results matter -- but they must cover the operand
ranges the physics produces.  Host numpy (x86 IEEE) is the second witness."""
import ctypes as C

import numpy as np
import pytest

from paper_2106_13465_b200 import _lib

pytestmark = pytest.mark.gpu
_dp = C.POINTER(C.c_double)


def run(op, a, b=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(a if b is None else b, dtype=np.float64)
    n = a.size
    fast, exact = np.empty(n), np.empty(n)
    ok = np.empty(n, dtype=np.int32)
    rc = _lib.lib().hydro_gpu_math_selftest(op, a.ctypes.data_as(_dp), b.ctypes.data_as(_dp),
                                            fast.ctypes.data_as(_dp), exact.ctypes.data_as(_dp),
                                            ok.ctypes.data_as(C.POINTER(C.c_int)), n)
    assert rc == 0
    return fast, exact, ok.astype(bool)


def operands(rng, n):
    mant = rng.uniform(1.0, 2.0, n)
    expo = rng.integers(-1030, 1024, n)
    sign = rng.choice([-1.0, 1.0], n)
    x = sign * np.ldexp(mant, expo)
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 2.2250738585072014e-308,
                        1.7976931348623157e308, 1.0, -1.0, 0.4, 0.3999999999999999])
    return np.concatenate([x, special, rng.uniform(-10, 10, n // 4),
                           rng.uniform(1e-6, 1e6, n // 4)])


def bits(x):
    return x.view(np.uint64)


def test_division_fast_path_is_ieee():
    rng = np.random.default_rng(2106)
    a = operands(rng, 1 << 20)
    b = rng.permutation(operands(rng, 1 << 20))[: a.size]
    fast, exact, ok = run(0, a, b)
    assert ok.mean() > 0.85
    assert np.array_equal(bits(fast[ok]), bits(exact[ok]))
    with np.errstate(all="ignore"):
        host = a / b
    both = ok & ~np.isnan(host)
    assert np.array_equal(bits(fast[both]), bits(host[both]))


def test_division_physics_ranges_all_fast():
    rng = np.random.default_rng(1)
    a = rng.uniform(-1e9, 1e9, 1 << 20)
    b = np.concatenate([rng.uniform(1e-9, 1e9, 1 << 19), -rng.uniform(1e-9, 1e9, 1 << 19)])
    fast, exact, ok = run(0, a, b)
    assert ok.mean() > 0.999
    assert np.array_equal(bits(fast[ok]), bits(exact[ok]))
    assert np.array_equal(bits(fast[ok]), bits((a / b)[ok]))


def test_sqrt_fast_path_is_ieee():
    rng = np.random.default_rng(13465)
    x = np.abs(operands(rng, 1 << 20))
    fast, exact, ok = run(1, x)
    assert ok.mean() > 0.9
    assert np.array_equal(bits(fast[ok]), bits(exact[ok]))
    with np.errstate(all="ignore"):
        host = np.sqrt(x)
    assert np.array_equal(bits(fast[ok]), bits(host[ok]))
    # negative, zero, inf, nan never take the fast path
    f2, e2, ok2 = run(1, np.array([-1.0, 0.0, -0.0, np.inf, np.nan, 1e-310]))
    assert not ok2.any()


def test_division_zero_numerator_fast_and_signed():
    """Zero momenta are everywhere in the benchmark cases (u = v = 0 at rest):
    +-0 / a density inside the fast-pass envelope [2^-256, 2^256) must stay on
    the fast path with the IEEE sign; outside it the exact pass takes over."""
    rng = np.random.default_rng(7)
    b = np.concatenate([10.0 ** rng.uniform(-77, 77, 4096), rng.uniform(1e-6, 1e6, 4096)])
    for zero in (0.0, -0.0):
        a = np.full(b.size, zero)
        fast, exact, ok = run(4, a, b)
        assert ok.all()
        assert np.array_equal(bits(fast), bits(exact))
        assert np.array_equal(bits(fast), bits(a / b))
    # densities outside the envelope leave the fast path (exact recompute)
    for far in (1e-300, 1e-78, 1e78, 1e300):
        _, _, ok = run(4, np.zeros(1), np.full(1, far))
        assert not ok.any()
    # negative or non-normal denominators leave the fast path (exact recompute)
    _, _, ok = run(4, np.array([-0.0, 0.0, 0.0, 0.0, 1.0]),
                   np.array([-2.0, 0.0, 5e-324, np.inf, -3.0]))
    assert not ok.any()


def test_density_division_sign_or_is_ieee():
    """op 4 (velocities, internal energy: x / rho): the quotient's sign bit is
    OR-ed with the numerator's, exact for positive normal denominators."""
    rng = np.random.default_rng(11)
    a = operands(rng, 1 << 20)
    b = np.abs(rng.permutation(operands(rng, 1 << 20))[: a.size])
    fast, exact, ok = run(4, a, b)
    env = (b >= np.ldexp(1.0, -256)) & (b < np.ldexp(1.0, 256))  # the fast-pass envelope
    assert ok[env].mean() > 0.8
    assert not ok[~env].any()
    assert np.array_equal(bits(fast[ok]), bits(exact[ok]))


def test_signed_zero_division_any_denominator_sign():
    """op 2: the star-speed division (divz) -- +-0 over a negative normal
    denominator stays fast with the IEEE sign."""
    rng = np.random.default_rng(3)
    b = np.concatenate([-rng.uniform(1e-6, 1e6, 4096), rng.uniform(1e-6, 1e6, 4096)])
    for zero in (0.0, -0.0):
        a = np.full(b.size, zero)
        fast, exact, ok = run(2, a, b)
        assert ok.all()
        assert np.array_equal(bits(fast), bits(exact))
    a = rng.uniform(-5, 5, b.size)
    fast, exact, ok = run(2, a, b)
    assert ok.all() and np.array_equal(bits(fast), bits(exact))


def test_minmod_fast_equals_reference_comparisons():
    """minmod_d_fast (integer sign/zero tests, one FP64 compare) == the
    reference's slope_minmod (euler_kernel.cpp:41-47) for every non-NaN pair:
    signed zeros, infinities, denormals, ties of equal magnitude."""
    rng = np.random.default_rng(41)
    x = operands(rng, 1 << 18)
    x = x[~np.isnan(x)]
    y = rng.permutation(x)
    ties = rng.choice(x, 4096)
    edge = np.array([0.0, -0.0, np.inf, -np.inf, 5e-324, -5e-324, 1.0, -1.0])
    ea, eb = np.meshgrid(edge, edge)
    a = np.concatenate([x, ties, -ties, ea.ravel()])
    b = np.concatenate([y, ties, -ties, eb.ravel()])
    fast, exact, ok = run(3, a, b)
    assert np.array_equal(bits(fast), bits(exact))


def test_bounded_division_is_ieee_inside_the_envelope():
    """divb (p / (gamma - 1), gamma p / rho) skips the range test: for every
    numerator in [2^-256, 65 * 2^256) and denominator in the envelope
    [2^-256, 2^256) the fast path must give the IEEE quotient bit for bit."""
    rng = np.random.default_rng(2106)
    n = 1 << 20
    a = np.ldexp(rng.uniform(1.0, 2.0, n), rng.integers(-256, 262, n))
    b = np.ldexp(rng.uniform(1.0, 2.0, n), rng.integers(-256, 256, n))
    lo, hi = np.ldexp(1.0, -256), np.nextafter(np.ldexp(1.0, 256), 0.0)
    top = np.nextafter(65.0 * np.ldexp(1.0, 256), 0.0)
    a = np.concatenate([a, [lo, lo, top, top, 0.4, 1.4]])
    b = np.concatenate([b, [lo, hi, lo, hi, 0.3999999999999999, 0.4]])
    fast, exact, _ = run(5, a, b)
    assert np.array_equal(bits(fast), bits(exact))
    assert np.array_equal(bits(fast), bits(a / b))
