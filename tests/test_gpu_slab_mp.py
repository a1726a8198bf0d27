"""The multi-process slab driver on real kernels: 2 ranks (processes) on one
B200, gloo for the dt allreduce (host-side, so no kernel waits on another
process), the peer-memory halo through CUDA IPC between the processes -- the
bench.py --gpus N code path except NCCL and the second GPU.  The gathered
state must be bitwise the single-domain reference run."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

NX, NY, STEPS = 70, 48, 12


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, case, bc, outdir):
    import torch
    import torch.distributed as dist

    import paper_2106_13465_b200 as P
    from paper_2106_13465_b200 import slab as S
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    model = P.GasModel()
    full = P.make_case(case, NX, NY, model, seed=8)
    geo = S.SlabGeometry(NX, NY, rank, world)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sl = S.GpuSlab(geo, full.dx, full.dy, model, bc, 0)
    sl.bind_stream(stream)
    sl.grid.upload(S.slab_planes(full.planes, NX, world, rank))
    comm = S.TorchComm()
    assert comm.setup_p2p(sl)
    S.run_slab(sl, comm, STEPS)
    torch.cuda.synchronize()
    out = np.zeros((4, geo.nx + 4, NY + 4))
    sl.grid.download(out)
    np.save(os.path.join(outdir, f"slab{rank}.npy"), out)
    dist.barrier()
    sl.grid.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("case,bc", [("random", "transmit"), ("corner_blast", "reflect")])
def test_two_process_slabs_with_ipc_halo(gpu, case, bc):
    from oracle import oracle as O
    from paper_2106_13465_b200 import slab as S
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank, args=(world, _free_port(), case, bc, d), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"slab{r}.npy")) for r in range(world)]
    got = S.gather_planes(parts, NX, NY)
    ref = O.make_case(case, NX, NY, seed=8)
    O.run_sequential(ref, STEPS, bc)
    assert np.array_equal(got[:, 2:NX + 2, 2:NY + 2], ref.u[:, 2:NX + 2, 2:NY + 2])
