"""Exact-Riemann flux mode ("exact-10": BASELINE's exact Riemann solver with 10
Newton iterations).

* CPU: the oracle's exact-10 flux is pinned against the reference's own exact
  solver (proj/src/exact_riemann.cpp via oracle/_ref: std::pow, Newton to
  1e-14) -- floored relative <= 1e-12, the BASELINE bound.
* GPU: the CUDA path equals the oracle bitwise (both use the same portable
  log/exp in place of std::pow), including the vacuum error.
"""
import numpy as np
import pytest

import paper_2106_13465_b200 as P
from oracle import oracle as O

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built here")
MODEL = P.GasModel()


def floored_rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)))


def state_pairs(rng, n):
    out = []
    for _ in range(n):
        wl = [rng.uniform(0.05, 20), rng.uniform(-4, 4), rng.uniform(-3, 3), rng.uniform(1e-3, 50)]
        wr = [rng.uniform(0.05, 20), rng.uniform(-4, 4), rng.uniform(-3, 3), rng.uniform(1e-3, 50)]
        out.append((np.array(wl), np.array(wr)))
    # Sod, strong shocks, strong rarefactions, a blast front, equal states
    out += [(np.array([1.0, 0, 0, 1.0]), np.array([0.125, 0, 0, 0.1])),
            (np.array([1.0, 0, 0, 1000.0]), np.array([1.0, 0, 0, 0.01])),
            (np.array([1.0, -2.0, 0, 0.4]), np.array([1.0, 2.0, 0, 0.4])),
            (np.array([5.99924, 19.5975, 0, 460.894]), np.array([5.99242, -6.19633, 0, 46.095])),
            (np.array([1.0, 0.3, 0.1, 2.0]), np.array([1.0, 0.3, 0.1, 2.0]))]
    return out


@needs_ref
def test_oracle_exact10_matches_reference_exact_solver():
    rng = np.random.default_rng(2106)
    worst, checked = 0.0, 0
    for wl, wr in state_pairs(rng, 5000):
        try:
            ref, iters = O.ref_exact_flux(wl, wr)
        except O.CheckerError:  # vacuum: both must reject it
            with pytest.raises(O.CheckerError):
                O.exact10_flux(wl, wr)
            continue
        assert iters <= 10  # 10 fixed iterations cover the reference's convergence
        worst = max(worst, floored_rel(O.exact10_flux(wl, wr), ref))
        checked += 1
    assert checked > 4000
    assert worst <= 1e-12, worst


def test_exact10_reduces_to_physical_flux_for_equal_states():
    rng = np.random.default_rng(4)
    for _ in range(100):
        w = np.array([rng.uniform(0.1, 5), rng.uniform(-2, 2), rng.uniform(-2, 2), rng.uniform(0.1, 5)])
        e = w[3] / (1.4 - 1.0) + 0.5 * w[0] * (w[1] ** 2 + w[2] ** 2)
        exact = np.array([w[0] * w[1], w[0] * w[1] * w[1] + w[3], w[0] * w[1] * w[2], (e + w[3]) * w[1]])
        assert floored_rel(O.exact10_flux(w, w), exact) <= 1e-13


def test_oracle_exact10_run_is_close_to_hllc_run():
    """Sanity: the two fluxes solve the same PDE (Sod tube to t=0.2)."""
    a = O.make_case("sod", 4, 200)
    b = a.copy()
    O.run_until(a, 0.2)
    with O.flux_mode("exact10"):
        O.run_until(b, 0.2)
    rho_a, rho_b = a.interior()[0, 0], b.interior()[0, 0]
    assert np.mean(np.abs(rho_a - rho_b)) < 5e-3


def vacuum_grid(nx=32, ny=16):
    """Two cold halves rushing apart: the centre interface generates vacuum."""
    g = O.make_case("uniform", nx, ny)
    u = g.u
    rho, p = 1.0, 0.01
    for i in range(1, nx + 1):
        vel = -3.0 if i <= nx // 2 else 3.0
        u[0, i + 1, 2:ny + 2] = rho
        u[1, i + 1, 2:ny + 2] = rho * vel
        u[2, i + 1, 2:ny + 2] = 0.0
        u[3, i + 1, 2:ny + 2] = p / 0.3999999999999999 + 0.5 * rho * vel * vel
    return g


def test_oracle_reports_vacuum_as_validation_error():
    g = vacuum_grid()
    with O.flux_mode("exact10"), pytest.raises(O.CheckerError) as e:
        O.run_sequential(g, 3, "transmit")
    assert e.value.category == 7
    assert "vacuum-generating Riemann states are out of scope" in str(e.value)
    assert str(e.value).startswith("step 0: column sweep strip 1:")


# ---- GPU --------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("case,nx,ny,steps,bc,seed", [
    ("blast", 48, 48, 6, "reflect", 0), ("corner_blast", 64, 40, 10, "reflect", 0),
    ("sod_x", 64, 24, 20, "transmit", 0), ("random", 40, 33, 8, "transmit", 5),
    ("random", 33, 40, 8, "reflect", 6), ("random", 256, 192, 20, "transmit", 11),
    ("corner_blast", 160, 128, 40, "reflect", 0),
])
def test_gpu_exact10_bitwise_equals_oracle(gpu, case, nx, ny, steps, bc, seed):
    grid = P.make_case(case, nx, ny, MODEL, seed=seed)
    ref = O.make_case(case, nx, ny, seed=seed)
    dt = P.run_gpu(grid, MODEL, steps, bc, flux="exact10")
    with O.flux_mode("exact10"):
        dt_ref = O.run_sequential(ref, steps, bc)
    if not np.array_equal(grid.planes, ref.u):
        bad = np.argwhere(grid.planes != ref.u)
        pytest.fail(f"{len(bad)} values differ, first {bad[:4].tolist()}; "
                    f"floored rel {floored_rel(grid.planes, ref.u):.3g}")
    assert dt == dt_ref


@pytest.mark.gpu
def test_gpu_exact10_run_until_sod(gpu):
    grid = P.make_case("sod", 4, 200, MODEL)
    ref = O.make_case("sod", 4, 200)
    n = P.run_until_gpu(grid, MODEL, 0.2, "reflect", flux="exact10")
    with O.flux_mode("exact10"):
        n_ref = O.run_until(ref, 0.2)
    assert n == n_ref
    assert np.array_equal(grid.planes, ref.u)


@pytest.mark.gpu
def test_gpu_exact10_vacuum_error_matches_oracle(gpu):
    g = vacuum_grid()
    grid = P.Grid2D(g.nx, g.ny, g.dx, g.dy, g.u.copy())
    with O.flux_mode("exact10"), pytest.raises(O.CheckerError) as e_ref:
        O.run_sequential(g, 3, "transmit")
    with pytest.raises(P.ValidationError) as e_gpu:
        P.run_gpu(grid, MODEL, 3, "transmit", flux="exact10")
    assert str(e_gpu.value) == str(e_ref.value)
