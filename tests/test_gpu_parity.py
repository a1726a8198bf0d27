"""Parity of the CUDA path (through the C-ABI) with the reference.

Bar: bitwise.  Every comparison below is exact equality of binary64 values
(the FNV-1a digest of proj/src/audit.cpp:53-76, or np.array_equal on every
plane including ghosts).  The contractual bound stated in DESIGN.md is the
reference's floored metric compare_tolerance (audit.cpp:137-154)
max|a-b|/max(|a|,|b|,1) <= 1e-12; bitwise equality implies it, and
test_tolerance_metric_is_zero asserts it explicitly.
"""
import json
import os

import numpy as np
import pytest

import paper_2106_13465_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))
FULL_PATH = os.path.join(HERE, "golden", "golden_full.json")
GOLDEN_FULL = json.load(open(FULL_PATH)) if os.path.exists(FULL_PATH) else {}
MODEL = P.GasModel()


def gpu_run(case, nx, ny, steps, bc, seed=0, model=MODEL, tune=None):
    grid = P.make_case(case, nx, ny, model, seed=seed)
    with P.GpuGrid(grid.nx, grid.ny, grid.dx, grid.dy, model, bc, device=0) as g:
        if tune:
            g.tune(*tune)
        g.upload(grid.planes)
        dt = g.run(steps)
        g.download(grid.planes)
    return grid, dt


def oracle_run(case, nx, ny, steps, bc, seed=0, cfl=0.8):
    ref = O.make_case(case, nx, ny, seed=seed)
    dt = O.run_sequential(ref, steps, bc, cfl=cfl)
    return ref, dt


@pytest.mark.parametrize("name", sorted(GOLDEN))
def test_golden_digest(gpu, name):
    """Digest of the GPU result == digest the unmodified reference produced."""
    rec = GOLDEN[name]
    grid, _ = gpu_run(rec["case"], rec["nx"], rec["ny"], rec["steps"], rec["bc"], rec["seed"])
    assert f"{P.grid_digest(grid):016x}" == rec["digest"], rec["provenance"]


@pytest.mark.parametrize("case,nx,ny,steps,bc,seed", [
    ("corner_blast", 64, 64, 12, "reflect", 0),
    ("blast", 37, 53, 9, "reflect", 0),
    ("sod_x", 48, 40, 15, "transmit", 0),
    ("random", 70, 33, 8, "transmit", 3),
    ("random", 33, 70, 8, "reflect", 4),
    ("blast", 4, 4, 5, "reflect", 0),
    ("corner_blast", 4, 9, 6, "transmit", 0),
    ("random", 33, 33, 7, "reflect", 2),     # rows/cols nx-1, nx in different warp groups
    ("random", 65, 97, 6, "transmit", 8),
    ("corner_blast", 97, 65, 9, "reflect", 0),
])
def test_every_plane_and_ghost_matches_oracle(gpu, case, nx, ny, steps, bc, seed):
    grid, dt = gpu_run(case, nx, ny, steps, bc, seed)
    ref, dt_ref = oracle_run(case, nx, ny, steps, bc, seed)
    if not np.array_equal(grid.planes, ref.u):
        bad = np.argwhere(grid.planes != ref.u)
        pytest.fail(f"{len(bad)} values differ, first {bad[:4].tolist()}")
    assert dt == dt_ref


@pytest.mark.parametrize("ny", [35, 45, 63, 65])
@pytest.mark.parametrize("bc", ["transmit", "reflect"])
def test_odd_width_wall_ghosts(gpu, ny, bc):
    """Odd ny: the column sweep's last TMA store unit straddles the y-wall
    ghost column ny+1 (stores clip at 16-byte granularity), which must still
    carry the ghost value."""
    a, _ = gpu_run("random", 24, ny, 3, bc, 9)
    ref, _ = oracle_run("random", 24, ny, 3, bc, 9)
    assert np.array_equal(a.planes, ref.u)


@pytest.mark.parametrize("seg", [(1, 2, 0), (3, 4, 0), (7, 1000, 128), (1000, 6, 0), (5, 1, 0)])
def test_launch_geometry_does_not_change_bits(gpu, seg):
    """Strip segmentation is an execution detail: any split is bitwise equal
    (the GPU analogue of acceptance criterion 1, acceptance_tests.cpp:48-113)."""
    a, _ = gpu_run("random", 96, 80, 10, "transmit", 5, tune=seg)
    ref, _ = oracle_run("random", 96, 80, 10, "transmit", 5)
    assert np.array_equal(a.planes, ref.u)


def test_split_runs_equal_one_run(gpu):
    grid = P.make_case("corner_blast", 96, 64, MODEL)
    whole = grid.copy()
    with P.GpuGrid(96, 64, grid.dx, grid.dy, MODEL, "reflect", device=0) as g:
        g.upload(grid.planes)
        g.run(7)
        g.run(0)
        g.run(6)
        g.download(grid.planes)
        g.upload(whole.planes)
        g.run(13)
        g.download(whole.planes)
    ref, _ = oracle_run("corner_blast", 96, 64, 13, "reflect")
    assert np.array_equal(whole.planes, ref.u)
    assert np.array_equal(grid.interior(), whole.interior())


def test_zero_steps_is_identity(gpu):
    grid = P.make_case("random", 20, 30, MODEL, seed=9)
    before = grid.planes.copy()
    P.run_gpu(grid, MODEL, 0)
    assert np.array_equal(grid.planes, before)


def test_uniform_gas_is_a_fixed_point(gpu):
    """test_schedulers.cpp:49-61 / test_kernel.cpp:126-139 on the GPU."""
    grid = P.make_case("uniform", 40, 24, MODEL)
    before = grid.interior().copy()
    P.run_gpu(grid, MODEL, 6, "reflect")
    assert np.array_equal(grid.interior(), before)


def test_advance_matches_reference_advance(gpu):
    grid = P.make_case("random", 50, 44, MODEL, seed=21)
    ref = O.make_case("random", 50, 44, seed=21)
    P.advance_gpu(grid, MODEL, 3.25e-4, "transmit")
    O.advance(ref, 3.25e-4, "transmit")
    assert np.array_equal(grid.planes, ref.u)


def test_run_until_matches_reference(gpu):
    """run_until with its final-dt clamp (schedulers.cpp:118-138), on the
    reference's own Sod tube (cases.cpp:54-69) to t=0.2 as check_sod_profile."""
    grid = P.make_case("sod", 4, 200, MODEL)
    ref = O.make_case("sod", 4, 200)
    steps = P.run_until_gpu(grid, MODEL, 0.2, "reflect")
    steps_ref = O.run_until(ref, 0.2, "reflect")
    assert steps == steps_ref
    assert np.array_equal(grid.planes, ref.u)


def test_compute_dt_matches(gpu):
    grid = P.make_case("random", 31, 47, MODEL, seed=8)
    ref = O.make_case("random", 31, 47, seed=8)
    dt = P.compute_dt_gpu(grid, MODEL)
    assert dt == 0.8 * O.compute_limit(ref)


@pytest.mark.parametrize("case,seed", [("random", 77), ("corner_blast", 0), ("blast", 0),
                                       ("sod_x", 0), ("uniform", 0)])
def test_device_initialiser_equals_host(gpu, case, seed):
    host = P.make_case(case, 67, 45, MODEL, seed=seed)
    dev = P.Grid2D(67, 45, host.dx, host.dy)
    with P.GpuGrid(67, 45, host.dx, host.dy, MODEL, "reflect", device=0) as g:
        g.init_case(case, seed)
        g.download(dev.planes)
    assert np.array_equal(dev.planes, host.planes)


def test_positivity_error_matches_reference_message(gpu):
    """Fault injection of test_schedulers.cpp:115-128: CFL=25 must fail with a
    positivity error carrying the step and sweep -- here the exact message."""
    model = P.GasModel(cfl=25.0)
    grid = P.make_case("blast", 64, 64, model)
    ref = O.make_case("blast", 64, 64)
    with pytest.raises(O.CheckerError) as e_ref:
        O.run_sequential(ref, 5, "reflect", cfl=25.0)
    with pytest.raises(P.PositivityError) as e_gpu:
        P.run_gpu(grid, model, 5, "reflect")
    assert e_gpu.value.category == P.ErrorCategory.POSITIVITY
    assert str(e_gpu.value) == str(e_ref.value)
    assert "step" in str(e_gpu.value) and "sweep" in str(e_gpu.value)
    if O.ref_available():
        g2 = O.make_case("blast", 64, 64)
        with pytest.raises(O.CheckerError) as e_true:
            O.ref_run(g2, 5, "reflect", cfl=25.0)
        assert str(e_true.value) == str(e_gpu.value)


@pytest.mark.parametrize("cfl,case,bc", [(3.0, "random", "transmit"), (6.0, "corner_blast", "reflect"),
                                         (2.2, "sod_x", "transmit"), (12.0, "random", "reflect")])
def test_error_paths_match_oracle(gpu, cfl, case, bc):
    model = P.GasModel(cfl=cfl)
    grid = P.make_case(case, 48, 40, model, seed=1)
    ref = O.make_case(case, 48, 40, seed=1)
    ref_msg = gpu_msg = None
    try:
        O.run_sequential(ref, 30, bc, cfl=cfl)
    except O.CheckerError as e:
        ref_msg = str(e)
    try:
        P.run_gpu(grid, model, 30, bc)
    except P.PositivityError as e:
        gpu_msg = str(e)
    assert gpu_msg == ref_msg
    if ref_msg is None:
        assert np.array_equal(grid.planes, ref.u)


def test_tolerance_metric_is_zero(gpu):
    grid, _ = gpu_run("random", 80, 72, 20, "transmit", 13)
    ref, _ = oracle_run("random", 80, 72, 20, "transmit", 13)
    max_rel, l1 = O.compare_tolerance(O.Grid(grid.nx, grid.ny, grid.dx, grid.dy, grid.planes), ref)
    assert max_rel <= 1e-12 and max_rel == 0.0 and l1 == 0.0


@pytest.mark.parametrize("p2p", [False, True])
@pytest.mark.parametrize("world,case,bc", [(2, "corner_blast", "reflect"), (3, "random", "transmit"),
                                           (4, "sod_x", "transmit"), (5, "random", "reflect")])
def test_slab_decomposition_loopback(gpu, world, case, bc, p2p):
    """Row slabs with halo swaps and the dt min-reduction, all slabs on one
    device (the multi-GPU schedule without waiting kernels).  p2p: the row
    sweep stores the halo rows into the neighbours' inboxes itself
    (hydro_gpu_set_halo_peers), as over NVLink."""
    import torch

    from paper_2106_13465_b200 import slab as S
    nx, ny, steps = 53, 40, 17
    full = P.make_case(case, nx, ny, MODEL, seed=4)
    slabs = []
    stream = torch.cuda.current_stream()
    for r in range(world):
        geo = S.SlabGeometry(nx, ny, r, world)
        sl = S.GpuSlab(geo, full.dx, full.dy, MODEL, bc, 0)
        sl.bind_stream(stream)
        sl.grid.upload(S.slab_planes(full.planes, nx, world, r))
        slabs.append(sl)
    S.run_loopback(slabs, steps, p2p=p2p)
    torch.cuda.synchronize()
    parts = []
    for sl in slabs:
        p = np.zeros((4, sl.geo.nx + 4, ny + 4))
        sl.grid.download(p)
        parts.append(p)
    got = S.gather_planes(parts, nx, ny)
    ref, _ = oracle_run(case, nx, ny, steps, bc, 4)
    assert np.array_equal(got[:, 2:nx + 2, 2:ny + 2], ref.u[:, 2:nx + 2, 2:ny + 2])
    assert np.array_equal(got, ref.u)


@pytest.mark.parametrize("name", sorted(GOLDEN_FULL))
def test_full_size_golden(gpu, name):
    """BASELINE configs at full size against digests from the reference (HLLC)
    or, for the exact-10 flux, from the oracle's restatement."""
    rec = GOLDEN_FULL[name]
    nx, ny = rec["nx"], rec["ny"]
    dx, dy = 1.0 / nx, 1.0 / ny
    planes = np.empty((4, nx + 4, ny + 4))
    with P.GpuGrid(nx, ny, dx, dy, MODEL, rec["bc"], device=0, flux=rec.get("flux", "hllc")) as g:
        g.init_case(rec["case"], rec["seed"])
        g.run(rec["steps"])
        g.download(planes)
    grid = P.Grid2D(nx, ny, dx, dy, planes)
    assert f"{P.grid_digest(grid):016x}" == rec["digest"], rec["provenance"]


@pytest.mark.parametrize("scale,bc", [(1e-310, "reflect"), (1e-300, "transmit"), (1e200, "transmit")])
def test_exact_redo_path_is_bitwise(gpu, scale, bc):
    """Denormal / tiny / huge momenta push FastMath out of its proven range, so
    warps redo their work items with IEEE division -- still bitwise."""
    grid = P.make_case("random", 72, 40, MODEL, seed=17)
    grid.planes[1:3, 10:40, :] *= scale  # momenta of a band of rows
    ref = O.Grid(grid.nx, grid.ny, grid.dx, grid.dy, grid.planes.copy())
    msg_ref = msg_gpu = None
    try:
        O.run_sequential(ref, 6, bc)
    except O.CheckerError as e:
        msg_ref = str(e)
    try:
        P.run_gpu(grid, MODEL, 6, bc)
    except P.PositivityError as e:
        msg_gpu = str(e)
    assert msg_gpu == msg_ref
    if msg_ref is None:
        assert np.array_equal(grid.planes, ref.u)


@pytest.mark.parametrize("case,seed", [("random", 13465), ("sod_x", 0), ("corner_blast", 0), ("blast", 0)])
def test_slab_device_initialiser_matches_full_grid(gpu, case, seed):
    """hydro_gpu_init_case on a row slab (bench.py --gpus N) builds the slab's
    rows of the global case: global row indices, global Sod position, global
    random-field cell numbering."""
    from paper_2106_13465_b200 import slab as S
    nx, ny, world = 61, 37, 3
    full = P.make_case(case, nx, ny, MODEL, seed=seed)
    for r in range(world):
        geo = S.SlabGeometry(nx, ny, r, world)
        sl = S.GpuSlab(geo, full.dx, full.dy, MODEL, "reflect", 0)
        sl.grid.init_case(case, seed)
        got = np.zeros((4, geo.nx + 4, ny + 4))
        sl.grid.download(got)
        want = S.slab_planes(full.planes, nx, world, r)
        assert np.array_equal(got[:, 2:geo.nx + 2, 2:ny + 2], want[:, 2:geo.nx + 2, 2:ny + 2]), r
        sl.grid.close()


@pytest.mark.gpu
def test_one_cell_perturbation_stays_inside_the_stencil(gpu):
    """Stencil locality of the whole GPU step (the reference pins it per strip,
    proj/tests/test_kernel.cpp:153-179): with a fixed dt (advance_sequential)
    a one-ulp change of one interior cell can only reach cells within the
    two-cell stencil of the column sweep and then of the row sweep -- a 5x5
    box (plus the mirrored ghost copies) -- and leaves every other value bit
    for bit unchanged."""
    base = P.make_case("random", 48, 40, MODEL, seed=31)
    pert = base.copy()
    i0, j0 = 21, 17
    for v in range(4):
        k = (v, i0 + 1, j0 + 1)  # planes index = grid index + 1 (ghost offset -1 -> 0)
        pert.planes[k] = np.nextafter(pert.planes[k], np.inf)
    P.advance_gpu(base, MODEL, 2.5e-4, "transmit")
    P.advance_gpu(pert, MODEL, 2.5e-4, "transmit")
    diff = np.argwhere(base.planes != pert.planes)
    assert len(diff) > 0
    for v, ii, jj in diff:
        i, j = ii - 1, jj - 1
        assert abs(i - i0) <= 2 and abs(j - j0) <= 2, (v, i, j)


@pytest.mark.gpu
@pytest.mark.parametrize("n,case,bc,flux", [
    (2, "sod_x", "transmit", "hllc"), (3, "random", "transmit", "hllc"),
    (5, "corner_blast", "reflect", "hllc"), (4, "blast", "reflect", "hllc"),
    (3, "random", "reflect", "exact10"), (8, "random", "transmit", "hllc"),
    (8, "corner_blast", "reflect", "exact10"),
])
def test_single_process_group_equals_one_domain(gpu, n, case, bc, flux):
    """hydro_gpu_group (one host thread, n row slabs, peer-memory halo,
    on-device dt min): here all slabs share cuda:0, so the event joins and
    inbox parities run for real; every plane and ghost, the last dt and the
    digest equal a single context on the whole grid."""
    nx, ny, steps = 77, 52, 30
    one = P.make_case(case, nx, ny, MODEL, seed=9)
    grp = one.copy()
    dt_one = P.run_gpu(one, MODEL, steps, bc, flux=flux)
    with P.GpuGroup(nx, ny, grp.dx, grp.dy, MODEL, bc, devices=[0] * n, flux=flux) as g:
        assert [r for _, r, _ in g.slabs()] == [nx // n + (1 if k < nx % n else 0) for k in range(n)]
        g.upload(grp.planes)
        dt_grp = g.run(steps)
        g.download(grp.planes)
    assert dt_grp == dt_one
    assert np.array_equal(grp.planes, one.planes)


@pytest.mark.gpu
def test_single_process_group_device_init_and_error(gpu):
    """The group's device initialiser builds the global case slab by slab,
    and a positivity failure is the one the single domain reports."""
    nx, ny = 64, 40
    ref = P.make_case("sod_x", nx, ny, MODEL)
    P.run_gpu(ref, MODEL, 12, "transmit")
    got = np.zeros_like(ref.planes)
    with P.GpuGroup(nx, ny, 1.0 / nx, 1.0 / ny, MODEL, "transmit", devices=[0, 0, 0]) as g:
        g.init_case("sod_x")
        g.run(12)
        g.download(got)
    assert np.array_equal(got, ref.planes)
    # CFL 25 drives the blast to a positivity failure (test_schedulers.cpp:115-128)
    hot = P.GasModel(cfl=25.0)
    one = P.make_case("blast", 64, 64, hot)
    with pytest.raises(P.PositivityError) as e1:
        P.run_gpu(one, hot, 5, "reflect")
    two = P.make_case("blast", 64, 64, hot)
    with P.GpuGroup(64, 64, two.dx, two.dy, hot, "reflect", devices=[0, 0, 0]) as g:
        g.upload(two.planes)
        with pytest.raises(P.PositivityError) as e2:
            g.run(5)
    assert str(e1.value) == str(e2.value)
