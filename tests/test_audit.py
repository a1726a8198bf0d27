"""Device-side audit: the composable state hash and the
conservation totals computed without downloading the grid."""
import numpy as np
import pytest

import paper_2106_13465_b200 as P
from paper_2106_13465_b200 import hydro as H

MODEL = P.GasModel()


def test_host_state_hash_sensitivity_and_ghost_blindness():
    g = P.make_case("random", 24, 20, seed=4)
    h0 = H.grid_state_hash(g)
    g.planes[2, 10, 7] = np.nextafter(g.planes[2, 10, 7], 9.0)
    assert H.grid_state_hash(g) != h0
    g.planes[2, 10, 7] = np.nextafter(g.planes[2, 10, 7], -9.0)
    assert H.grid_state_hash(g) == h0
    g.planes[0, 0, 3] = 5.0  # ghost row: not part of the state
    assert H.grid_state_hash(g) == h0


def test_host_pairwise_sum_matches_audit_definition():
    from paper_2106_13465_b200 import _lib
    import ctypes as C
    rng = np.random.default_rng(0)
    for n in (1, 7, 8, 9, 100, 1001):
        v = rng.uniform(-1, 1, n)
        got = _lib.lib().hydro_pairwise_sum(v.ctypes.data_as(C.POINTER(C.c_double)), n)

        def pw(a):
            if a.size <= 8:
                s = 0.0
                for x in a:
                    s += float(x)
                return s
            h = a.size // 2
            return pw(a[:h]) + pw(a[h:])
        assert got == pw(v)


@pytest.mark.gpu
@pytest.mark.parametrize("case,nx,ny,steps,bc", [("random", 70, 45, 6, "transmit"),
                                                  ("corner_blast", 64, 64, 20, "reflect")])
def test_device_state_hash_equals_host_hash(gpu, case, nx, ny, steps, bc):
    grid = P.make_case(case, nx, ny, MODEL, seed=3)
    with P.GpuGrid(nx, ny, grid.dx, grid.dy, MODEL, bc) as g:
        g.upload(grid.planes)
        g.run(steps)
        dev = g.state_hash()
        tot = g.totals()
        g.download(grid.planes)
    assert dev == H.grid_state_hash(grid)
    host = [grid.dx * grid.dy * np.sum(grid.interior()[v]) for v in range(4)]
    for v in range(4):
        assert abs(tot[v] - host[v]) <= 1e-13 * max(1.0, abs(host[v]))


@pytest.mark.gpu
def test_slab_row_hashes_compose_to_the_full_grid_hash(gpu):
    import torch

    from paper_2106_13465_b200 import slab as S
    nx, ny, world = 61, 40, 3
    full = P.make_case("random", nx, ny, MODEL, seed=8)
    with P.GpuGrid(nx, ny, full.dx, full.dy, MODEL, "transmit") as g:
        g.upload(full.planes)
        g.run(5)
        want = g.state_hash()
    slabs = []
    for r in range(world):
        sl = S.GpuSlab(S.SlabGeometry(nx, ny, r, world), full.dx, full.dy, MODEL, "transmit", 0)
        sl.bind_stream(torch.cuda.current_stream())
        sl.grid.upload(S.slab_planes(full.planes, nx, world, r))
        slabs.append(sl)
    S.run_loopback(slabs, 5)
    torch.cuda.synchronize()
    rows = [sl.grid.row_audit()[0] for sl in slabs]  # (4, n_r) each
    combined = H.combine_row_hashes(np.concatenate(rows, axis=1).ravel())
    assert combined == want
