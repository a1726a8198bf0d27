"""The fused schedule (one sweep_xy launch per time step, csrc/hydro_fused.cuh)
against the oracle and against the split schedule (sweep_x + sweep_y).

Bar: bitwise.  Every cell update is a pure function of its 5-cell window
(sweep_strip, proj/src/euler_kernel.cpp:111-223), so keeping the column
sweep's output in shared memory must not change a bit: every plane including
ghosts, the last dt, and the first error in the reference's order
(schedulers.cpp:23-26,80-91) are compared exactly, in both arithmetics.
"""
import numpy as np
import pytest

import paper_2106_13465_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu
MODEL = P.GasModel()


def gpu_run(case, nx, ny, steps, bc, seed, schedule, math="bitwise", seg=0, splits=None):
    grid = P.make_case(case, nx, ny, MODEL, seed=seed)
    with P.GpuGrid(nx, ny, grid.dx, grid.dy, MODEL, bc, device=0, math=math) as g:
        g.set_schedule(schedule, seg)
        g.upload(grid.planes)
        dts = [g.run(k) for k in (splits or [steps])]
        g.download(grid.planes)
        fused_launches = None
        if schedule == "fused":
            g.set_timing(True)
            g.reset_counters()
            g.run(4)
            fused_launches = g.fused_times()[1]
    return grid.planes, dts, fused_launches


# band width is 120 output columns: one band, band edges, a ragged last band,
# short and ragged row segments, both boundary conditions
SHAPES = [
    ("corner_blast", 64, 64, 10, "reflect", 0),
    ("random", 96, 119, 7, "transmit", 5),
    ("random", 40, 120, 6, "reflect", 6),
    ("random", 40, 121, 6, "transmit", 7),
    ("random", 130, 250, 7, "reflect", 8),
    ("sod_x", 33, 241, 12, "transmit", 0),
    ("corner_blast", 257, 121, 6, "reflect", 0),
    ("random", 4, 40, 5, "transmit", 9),
    ("random", 7, 5, 5, "reflect", 10),
]


@pytest.mark.parametrize("case,nx,ny,steps,bc,seed", SHAPES)
@pytest.mark.parametrize("seg", [0, 16])
def test_fused_schedule_matches_the_oracle_bitwise(gpu, case, nx, ny, steps, bc, seed, seg):
    planes, dts, launches = gpu_run(case, nx, ny, steps, bc, seed, "fused", seg=seg)
    assert launches == 4, "the fused kernel did not run (an even step count is fused throughout)"
    ref = O.make_case(case, nx, ny, seed=seed)
    dt_ref = O.run_sequential(ref, steps, bc)
    if not np.array_equal(planes, ref.u):
        bad = np.argwhere(planes != ref.u)
        pytest.fail(f"{len(bad)} values differ from the oracle, first {bad[:4].tolist()}")
    assert dts[-1] == dt_ref


@pytest.mark.parametrize("math", ["bitwise", "tolerance"])
@pytest.mark.parametrize("case,nx,ny,steps,bc,seed", [
    ("random", 300, 97, 5, "transmit", 11),
    ("corner_blast", 512, 512, 20, "reflect", 0),
    ("random", 200, 363, 8, "reflect", 12),
])
def test_fused_equals_split_in_both_arithmetics(gpu, math, case, nx, ny, steps, bc, seed):
    ps, ds, _ = gpu_run(case, nx, ny, steps, bc, seed, "split", math)
    pf, df, _ = gpu_run(case, nx, ny, steps, bc, seed, "fused", math)
    assert np.array_equal(ps.view(np.uint64), pf.view(np.uint64))
    assert ds == df


@pytest.mark.parametrize("math", ["bitwise", "tolerance"])
def test_fused_run_splits_compose(gpu, math):
    """run(3) + run(4) == run(7): an odd run starts with a split step and
    every run's last fused step leaves the final ghost bands, so the
    fused/split pattern differs between the two."""
    p1, d1, _ = gpu_run("random", 200, 180, 7, "reflect", 3, "fused", math)
    p2, d2, _ = gpu_run("random", 200, 180, 7, "reflect", 3, "fused", math, splits=[3, 4])
    assert np.array_equal(p1.view(np.uint64), p2.view(np.uint64))
    assert d1[-1] == d2[-1]


@pytest.mark.parametrize("schedule", ["fused", "split"])
@pytest.mark.parametrize("cfl,case,bc", [(25.0, "corner_blast", "reflect"), (3.0, "random", "transmit"),
                                         (12.0, "random", "reflect")])
def test_fused_reports_the_reference_error(gpu, schedule, cfl, case, bc):
    """CFL fault injection (test_schedulers.cpp:115-128): the same message as
    the oracle (the reference's first throw), whichever schedule hits it."""
    nx, ny = 96, 130
    model = P.GasModel(cfl=cfl)
    ref = O.make_case(case, nx, ny, seed=1)
    ref_msg = gpu_msg = None
    try:
        O.run_sequential(ref, 14, bc, cfl=cfl)
    except O.CheckerError as e:
        ref_msg = str(e)
    grid = P.make_case(case, nx, ny, model, seed=1)
    with P.GpuGrid(nx, ny, grid.dx, grid.dy, model, bc, device=0) as g:
        g.set_schedule(schedule)
        g.upload(grid.planes)
        try:
            g.run(14)
        except P.PositivityError as e:
            gpu_msg = str(e)
        g.download(grid.planes)
    assert gpu_msg == ref_msg
    if ref_msg is None:
        assert np.array_equal(grid.planes, ref.u)


@pytest.mark.parametrize("case,seed,dense", [("random", 21, True), ("corner_blast", 0, False)])
def test_auto_schedule_follows_the_context_s_own_runs(gpu, case, seed, dense):
    """The default schedule: a context's first run is fused; later runs are
    chosen from the uniform-window share and the event-timed step time of the
    runs before (dense random flow goes to the split sweeps at once; a blast
    in quiescent gas stays fused or tries split once, whichever times faster)
    -- and the results are bitwise those of the split schedule either way."""
    nx = ny = 384
    grid = P.make_case(case, nx, ny, MODEL, seed=seed)
    ref = P.make_case(case, nx, ny, MODEL, seed=seed)
    with P.GpuGrid(nx, ny, grid.dx, grid.dy, MODEL, "reflect", device=0) as g:
        assert g.schedule_choice() == (True, -1.0)
        g.upload(grid.planes)
        g.run(6)
        g.run(6)  # decided from the first run
        fused, share = g.schedule_choice()
        if dense:
            assert not fused and share < 0.2
        else:
            assert share >= 0.6
        g.run(6)
        g.run(5)
        assert isinstance(g.schedule_choice()[0], bool)
        g.download(grid.planes)
    with P.GpuGrid(nx, ny, ref.dx, ref.dy, MODEL, "reflect", device=0) as g:
        g.set_schedule("split")
        g.upload(ref.planes)
        g.run(23)
        g.download(ref.planes)
    assert np.array_equal(grid.planes.view(np.uint64), ref.planes.view(np.uint64))


@pytest.mark.parametrize("n,case,bc,nx", [(2, "sod_x", "transmit", 77), (3, "random", "reflect", 77),
                                          (8, "corner_blast", "reflect", 77), (5, "random", "transmit", 11),
                                          (4, "corner_blast", "reflect", 300)])
@pytest.mark.parametrize("schedule", ["fused", "split"])
def test_group_slabs_take_fused_steps(gpu, monkeypatch, n, case, bc, nx, schedule):
    """Row slabs on the fused schedule (hydro_gpu_group, all slabs on cuda:0):
    the fused step's row phase stores the halo rows into the neighbours'
    inboxes and the exchange fills the ghost rows of whichever buffer holds the
    state.  Odd and even step counts, two calls; every plane and ghost and the
    last dt equal one context on the whole grid, in either schedule."""
    ny = 130
    one = P.make_case(case, nx, ny, MODEL, seed=19)
    grp = one.copy()
    dt_one = None
    with P.GpuGrid(nx, ny, one.dx, one.dy, MODEL, bc, device=0) as g:
        g.set_schedule("split")
        g.upload(one.planes)
        g.run(13)
        dt_one = g.run(18)
        g.download(one.planes)
    monkeypatch.setenv("HYDRO_GPU_SCHEDULE", schedule)
    with P.GpuGroup(nx, ny, grp.dx, grp.dy, MODEL, bc, devices=[0] * n) as g:
        g.upload(grp.planes)
        g.run(13)
        dt_grp = g.run(18)
        g.download(grp.planes)
    assert dt_grp == dt_one
    assert np.array_equal(grp.planes.view(np.uint64), one.planes.view(np.uint64))


# ---- exact-10 flux on the fused schedule ---------------------------------------

def exact_run(case, nx, ny, steps, bc, seed, schedule, math="bitwise"):
    grid = P.make_case(case, nx, ny, MODEL, seed=seed)
    with P.GpuGrid(nx, ny, grid.dx, grid.dy, MODEL, bc, device=0, flux="exact10", math=math) as g:
        g.set_schedule(schedule)
        g.upload(grid.planes)
        dt = g.run(steps)
        g.download(grid.planes)
        g.set_timing(True)
        g.reset_counters()
        g.run(2)
        n_xy = g.fused_times()[1]
    return grid.planes, dt, n_xy


@pytest.mark.parametrize("case,nx,ny,steps,bc,seed", [
    ("corner_blast", 64, 130, 10, "reflect", 0), ("random", 40, 121, 6, "transmit", 31),
    ("random", 96, 250, 8, "reflect", 32), ("sod_x", 33, 241, 12, "transmit", 0),
    ("blast", 150, 150, 9, "reflect", 0),
])
def test_fused_exact10_matches_the_oracle_bitwise(gpu, case, nx, ny, steps, bc, seed):
    planes, dt, n_xy = exact_run(case, nx, ny, steps, bc, seed, "fused")
    assert n_xy == 2, "the fused kernel did not run with the exact-10 flux"
    ref = O.make_case(case, nx, ny, seed=seed)
    with O.flux_mode("exact10"):
        dt_ref = O.run_sequential(ref, steps, bc)
    if not np.array_equal(planes, ref.u):
        bad = np.argwhere(planes != ref.u)
        pytest.fail(f"{len(bad)} values differ from the oracle, first {bad[:4].tolist()}")
    assert dt == dt_ref


def test_fused_exact10_equals_split_in_tolerance_mode(gpu):
    ps, ds, _ = exact_run("random", 200, 363, 8, "reflect", 12, "split", "tolerance")
    pf, df, n_xy = exact_run("random", 200, 363, 8, "reflect", 12, "fused", "tolerance")
    assert n_xy == 2
    assert np.array_equal(ps.view(np.uint64), pf.view(np.uint64)) and ds == df


@pytest.mark.parametrize("axis", ["column", "row"])
def test_fused_exact10_reports_vacuum_like_the_oracle(gpu, axis):
    """Two cold halves rushing apart generate vacuum at the centre interface
    (exact_riemann.cpp:55-57), along i (the column phase finds it) or along j
    (the row phase does): the reference's validation error, word for word."""
    nx, ny = (32, 130) if axis == "column" else (40, 128)
    g = O.make_case("uniform", nx, ny)
    u = g.u
    rho, p = 1.0, 0.01
    ii, jj = np.meshgrid(np.arange(1, nx + 1), np.arange(1, ny + 1), indexing="ij")
    vel = np.where((ii <= nx // 2) if axis == "column" else (jj <= ny // 2), -3.0, 3.0)
    u[0, 2:nx + 2, 2:ny + 2] = rho
    u[1 if axis == "column" else 2, 2:nx + 2, 2:ny + 2] = rho * vel
    u[2 if axis == "column" else 1, 2:nx + 2, 2:ny + 2] = 0.0
    u[3, 2:nx + 2, 2:ny + 2] = p / 0.3999999999999999 + 0.5 * rho * vel * vel
    grid = P.Grid2D(g.nx, g.ny, g.dx, g.dy, g.u.copy())
    with O.flux_mode("exact10"), pytest.raises(O.CheckerError) as e_ref:
        O.run_sequential(g, 4, "transmit")
    assert axis in str(e_ref.value)
    with P.GpuGrid(nx, ny, grid.dx, grid.dy, MODEL, "transmit", device=0, flux="exact10") as gg:
        gg.set_schedule("fused")
        gg.upload(grid.planes)
        with pytest.raises(P.ValidationError) as e_gpu:
            gg.run(4)
    assert str(e_gpu.value) == str(e_ref.value)
