"""The validation suite (paper_2106_13465_b200/validation.py): the reference's
`hydrobench validate` checks (proj/src/validation.cpp) on GPU output."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2106_13465_b200 import validation as V

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built here")


def test_host_exact_solver_self_checks():
    for r in V.check_riemann_solver():
        assert r.passed, (r.name, r.detail)


@needs_ref
def test_host_exact_solver_matches_reference_flux():
    """The validation ground truth agrees with the reference's exact solver."""
    rng = np.random.default_rng(9)
    for _ in range(300):
        wl = np.array([rng.uniform(0.1, 5), rng.uniform(-2, 2), rng.uniform(-1, 1), rng.uniform(0.1, 5)])
        wr = np.array([rng.uniform(0.1, 5), rng.uniform(-2, 2), rng.uniform(-1, 1), rng.uniform(0.1, 5)])
        try:
            ref, _ = O.ref_exact_flux(wl, wr)
        except O.CheckerError:
            continue
        w = V.sample(V.exact_riemann(wl, wr), wl, wr, 0.0)
        e = w[3] / (1.4 - 1.0) + 0.5 * w[0] * (w[1] ** 2 + w[2] ** 2)
        f = np.array([w[0] * w[1], w[0] * w[1] * w[1] + w[3], w[0] * w[1] * w[2], (e + w[3]) * w[1]])
        assert np.max(np.abs(f - ref) / np.maximum(np.abs(ref), 1.0)) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("math", ["bitwise", "tolerance"])
@pytest.mark.parametrize("flux", ["hllc", "exact10"])
def test_gpu_validation_suite_passes(gpu, flux, math):
    results = V.run_validation_suite(flux, math)
    failed = [(r.name, r.detail) for r in results if not r.passed]
    assert not failed, failed
    assert len(results) >= 13
