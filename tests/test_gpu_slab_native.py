"""The multi-rank schedule driven from C++ (hydro_gpu_comm_attach): per rank
one captured CUDA graph per run, with the NCCL min-allreduce of the dt limit
per step and the first error over all ranks at the end.

On a one-GPU box only a one-rank NCCL communicator can be formed (NCCL
refuses two ranks on one device), so these tests run the whole native path --
NCCL loaded at run time, the allreduces captured inside the graph, the error
allreduce, the exchange timing -- on a one-slab decomposition (both walls
physical) and compare it bitwise with the single-domain run; the multi-slab
halo logic of the same schedule is covered by the loopback / multi-process
tests (test_gpu_parity.py, test_gpu_slab_mp.py)."""
import os
import socket

import numpy as np
import pytest

import paper_2106_13465_b200 as P

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def nccl_world(gpu):
    import torch
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def _native_slab(case, n, bc, flux="hllc", math="bitwise", model=P.GasModel()):
    from paper_2106_13465_b200 import slab as S
    geo = S.SlabGeometry(n, n, 0, 1)
    sl = S.GpuSlab(geo, 1.0 / n, 1.0 / n, model, bc, 0, flux=flux, math=math)
    comm = S.TorchComm()
    assert comm.setup_native(sl), "NCCL native driver not available"
    return sl, comm


@pytest.mark.parametrize("case,n,bc,steps,flux,math", [
    ("corner_blast", 96, "reflect", 30, "hllc", "bitwise"),
    ("random", 80, "transmit", 20, "hllc", "bitwise"),
    ("sod_x", 64, "transmit", 25, "exact10", "bitwise"),
    ("random", 72, "transmit", 15, "hllc", "tolerance"),
])
def test_native_slab_run_equals_single_domain(nccl_world, case, n, bc, steps, flux, math):
    from paper_2106_13465_b200 import slab as S
    seed = 5 if case == "random" else 0
    ref = P.make_case(case, n, n, seed=seed)
    with P.GpuGrid(n, n, ref.dx, ref.dy, P.GasModel(), bc, device=0, flux=flux, math=math) as g:
        g.upload(ref.planes)
        dt_ref = g.run(steps)
        g.download(ref.planes)
    sl, comm = _native_slab(case, n, bc, flux, math)
    sl.grid.init_case(case, seed)
    S.run_slab(sl, comm, steps)  # the library's graph, not the per-step Python driver
    got = np.zeros_like(ref.planes)
    sl.grid.download(got)
    assert np.array_equal(got, ref.planes)
    # the graph is replayed for a second run of the same length: same bits
    sl.grid.init_case(case, seed)
    dt2 = sl.grid.run(steps)
    sl.grid.download(got)
    assert np.array_equal(got, ref.planes) and dt2 == dt_ref
    sl.grid.close()


def test_native_slab_error_is_the_references(nccl_world):
    """A CFL far above stability fails: the error slots are min-allreduced
    inside the graph, and the message is the single domain's."""
    bad = P.GasModel(cfl=25.0)
    ref = P.make_case("corner_blast", 64, 64, bad)
    with P.GpuGrid(64, 64, ref.dx, ref.dy, bad, "reflect", device=0) as g:
        g.upload(ref.planes)
        with pytest.raises(P.PositivityError) as want:
            g.run(10)
    sl, comm = _native_slab("corner_blast", 64, "reflect", model=bad)
    sl.grid.init_case("corner_blast", 0)
    with pytest.raises(P.PositivityError) as got:
        sl.grid.run(10)
    assert str(got.value) == str(want.value)
    sl.grid.close()


def test_native_slab_exchange_is_timed(nccl_world):
    sl, comm = _native_slab("sod_x", 128, "transmit")
    sl.grid.init_case("sod_x", 0)
    sl.grid.set_timing(True)
    sl.grid.run(8)
    ms, cnt = sl.grid.comm_times()
    kt = sl.grid.kernel_times()
    _, n_xy = sl.grid.fused_times()
    sl.grid.set_timing(False)
    assert cnt == 8 and ms > 0.0  # one exchange per step in either schedule
    assert n_xy == 8 or (kt["n_x"] == 8 and kt["n_y"] == 8)
    sl.grid.close()
