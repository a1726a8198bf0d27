"""Tolerance math mode (hydro_gpu_set_math(HYDRO_GPU_MATH_TOLERANCE)).

Bar: the north-star contract, compare_tolerance (proj/src/audit.cpp:137-154)
max|a-b| / max(|a|,|b|,1) <= 1e-12 on the interior after N steps, against
the C oracle at oracle-sized grids and, at BASELINE's full sizes, against the
bitwise mode's result, whose digest is pinned to the reference's by
tests/golden/golden_full.json (so it is the reference's state).  The dt of
the last step is held to the same relative bound.  Errors keep the
reference's category and message (the fast pass redoes a failing item with
the exact arithmetic).
"""
import json
import os

import numpy as np
import pytest

import paper_2106_13465_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-12
HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN_FULL = json.load(open(os.path.join(HERE, "golden", "golden_full.json")))
MODEL = P.GasModel()


def max_rel(a: np.ndarray, b: np.ndarray) -> float:
    """compare_tolerance's floored relative difference (audit.cpp:146)."""
    return float((np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)).max())


def gpu_run(case, nx, ny, steps, bc, seed=0, flux="hllc", math="tolerance"):
    grid = P.make_case(case, nx, ny, MODEL, seed=seed)
    with P.GpuGrid(grid.nx, grid.ny, grid.dx, grid.dy, MODEL, bc, device=0, flux=flux,
                   math=math) as g:
        g.upload(grid.planes)
        dt = g.run(steps)
        g.download(grid.planes)
    return grid, dt


@pytest.mark.parametrize("flux", ["hllc", "exact10"])
@pytest.mark.parametrize("case,nx,ny,steps,bc,seed", [
    ("corner_blast", 256, 256, 100, "reflect", 0),   # BASELINE config 0
    ("sod_x", 192, 160, 60, "transmit", 0),
    ("random", 160, 224, 30, "transmit", 5),
    ("random", 97, 65, 20, "reflect", 6),
    ("blast", 37, 53, 9, "reflect", 0),
])
def test_tolerance_mode_within_1e12_of_oracle(gpu, flux, case, nx, ny, steps, bc, seed):
    grid, dt = gpu_run(case, nx, ny, steps, bc, seed, flux)
    ref = O.make_case(case, nx, ny, seed=seed)
    with O.flux_mode(flux):
        dt_ref = O.run_sequential(ref, steps, bc)
    got, want = grid.interior(), ref.u[:, 2:nx + 2, 2:ny + 2]
    mx, _ = O.compare_tolerance(O.Grid(nx, ny, grid.dx, grid.dy, grid.planes.copy()), ref)
    assert mx <= TOL and max_rel(got, want) <= TOL, (mx, max_rel(got, want))
    assert abs(dt - dt_ref) <= TOL * max(abs(dt), abs(dt_ref))


@pytest.mark.parametrize("name", ["cfg1_sod_x_2048_200", "cfg1_sod_x_2048_200_exact10",
                                  "random_1024_20_exact10"])
def test_tolerance_mode_full_size(gpu, name):
    """Full-size BASELINE workloads: the tolerance state against the bitwise
    state, itself checked against the reference's digest."""
    rec = GOLDEN_FULL[name]
    nx, ny = rec["nx"], rec["ny"]
    out = {}
    for math in ("bitwise", "tolerance"):
        planes = np.empty((4, nx + 4, ny + 4))
        with P.GpuGrid(nx, ny, 1.0 / nx, 1.0 / ny, MODEL, rec["bc"], device=0,
                       flux=rec.get("flux", "hllc"), math=math) as g:
            g.init_case(rec["case"], rec["seed"])
            dt = g.run(rec["steps"])
            g.download(planes)
        out[math] = (planes, dt)
    exact = P.Grid2D(nx, ny, 1.0 / nx, 1.0 / ny, out["bitwise"][0])
    assert f"{P.grid_digest(exact):016x}" == rec["digest"]
    a, b = out["bitwise"][0][:, 2:nx + 2, 2:ny + 2], out["tolerance"][0][:, 2:nx + 2, 2:ny + 2]
    assert max_rel(a, b) <= TOL
    assert not np.array_equal(a, b), "tolerance mode ran the bitwise kernels"
    assert abs(out["bitwise"][1] - out["tolerance"][1]) <= TOL * out["bitwise"][1]


def test_mode_switch_on_one_context(gpu):
    """set_math between runs re-captures the step graph: bitwise -> tolerance
    -> bitwise on one context, the last run bitwise the oracle's."""
    grid = P.make_case("random", 96, 80, MODEL, seed=12)
    ref = O.make_case("random", 96, 80, seed=12)
    with P.GpuGrid(96, 80, grid.dx, grid.dy, MODEL, "transmit", device=0) as g:
        g.upload(grid.planes)
        g.run(4)
        g.set_math("tolerance")
        g.run(4)
        g.set_math("bitwise")
        g.upload(grid.planes)
        g.run(8)
        g.download(grid.planes)
    O.run_sequential(ref, 8, "transmit")
    assert np.array_equal(grid.planes, ref.u)


def test_tolerance_mode_positivity_error_matches_reference(gpu):
    """The CFL=25 fault injection of test_schedulers.cpp:115-128 fails with the
    reference's category and exact message in tolerance mode too."""
    model = P.GasModel(cfl=25.0)
    grid = P.make_case("blast", 64, 64, model)
    ref = O.make_case("blast", 64, 64)
    with pytest.raises(O.CheckerError) as e_ref:
        O.run_sequential(ref, 5, "reflect", cfl=25.0)
    with pytest.raises(P.PositivityError) as e_gpu:
        P.run_gpu(grid, model, 5, "reflect", math="tolerance")
    assert e_gpu.value.category == P.ErrorCategory.POSITIVITY
    assert str(e_gpu.value) == str(e_ref.value)


def test_unknown_math_mode_is_a_config_error(gpu):
    with P.GpuGrid(16, 16, 1 / 16, 1 / 16, MODEL, "reflect", device=0) as g:
        with pytest.raises(P.ConfigError):
            g.set_math("fast")
        rc = g._lib.hydro_gpu_set_math(g._ctx, 7)
        assert rc == 1


@pytest.mark.parametrize("scale,bc", [(1e-310, "reflect"), (1e-300, "transmit"), (1e200, "transmit")])
def test_tolerance_mode_redo_items_are_decomposition_invariant(gpu, scale, bc):
    """Denormal / tiny / huge momenta send work items through the redo pass.
    In tolerance mode the redo pass repeats the fast pass's arithmetic (only
    the reference's branches differ), so the result is within 1e-12 of the
    oracle and bitwise independent of the segment lengths."""
    grid = P.make_case("random", 72, 40, MODEL, seed=17)
    grid.planes[1:3, 10:40, :] *= scale  # momenta of a band of rows
    ref = O.Grid(grid.nx, grid.ny, grid.dx, grid.dy, grid.planes.copy())
    msg_ref = None
    try:
        O.run_sequential(ref, 6, bc)
    except O.CheckerError as e:  # huge momenta: the reference's positivity error
        msg_ref = str(e)
    outs, msgs = [], []
    for seg in ((0, 0), (8, 4), (40, 72)):
        planes = grid.planes.copy()
        with P.GpuGrid(72, 40, grid.dx, grid.dy, MODEL, bc, device=0, math="tolerance") as g:
            g.tune(seg[0], seg[1], 0)
            g.upload(planes)
            try:
                g.run(6)
                msgs.append(None)
            except P.PositivityError as e:
                msgs.append(str(e))
            g.download(planes)
        outs.append(planes)
    assert msgs == [msg_ref] * 3
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    if msg_ref is None:
        assert max_rel(outs[0][:, 2:74, 2:42], ref.u[:, 2:74, 2:42]) <= TOL


@pytest.mark.parametrize("scale", [1e-310, 1e-200, 1e150])
def test_tolerance_mode_extreme_densities_match_the_oracle(gpu, scale):
    """The whole state scaled by `scale` (rho, momenta, E -- the same flow:
    the Euler equations are invariant under rho, p -> a rho, a p at fixed
    velocities): subnormal, tiny or huge densities and pressures, outside the
    fast pass's envelope, so every item takes the redo pass, which must use
    IEEE division and sqrt where the fast formulas cannot take the operands
    (a flushed reciprocal seed of a subnormal density gave NaN velocities and
    a false 'pres non-positive').  The reference accepts these states; the GPU
    must too, within 1e-12 of the oracle and independent of the
    segmentation."""
    grid = P.make_case("random", 64, 48, MODEL, seed=23)
    grid.planes *= scale
    ref = O.Grid(grid.nx, grid.ny, grid.dx, grid.dy, grid.planes.copy())
    dt_ref = O.run_sequential(ref, 3, "transmit")
    outs, dts = [], []
    for seg in ((0, 0), (8, 8), (64, 48)):
        planes = grid.planes.copy()
        with P.GpuGrid(64, 48, grid.dx, grid.dy, MODEL, "transmit", device=0, math="tolerance") as g:
            g.tune(seg[0], seg[1], 0)
            g.upload(planes)
            dts.append(g.run(3))
            g.download(planes)
        outs.append(planes)
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    got, want = outs[0][:, 2:66, 2:50], ref.u[:, 2:66, 2:50]
    assert np.isfinite(got).all()
    # relative to the scale (the floored metric would pass tiny states trivially)
    assert max_rel(got / scale, want / scale) <= 1e-10
    assert abs(dts[0] - dt_ref) <= 1e-10 * dt_ref  # subnormal states carry ~44 bits
