"""The CUDA-IPC plumbing of the peer-memory halo (hydro_gpu_inbox_ipc_handle /
hydro_gpu_ipc_open): two processes on one device -- one exports its slab
inbox, the other maps it and stores into it, the first reads the bytes back.
No kernel waits on another process (the handshake is a host queue)."""
import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _owner(q_handle, q_done, q_result):
    import torch

    import paper_2106_13465_b200 as P
    from paper_2106_13465_b200 import slab as S
    torch.cuda.set_device(0)
    with P.GpuGrid(8, 40, 1 / 8, 1 / 40, P.GasModel(), "reflect", device=0) as g:
        ptr, count = g.inbox()
        q_handle.put((g.inbox_ipc_handle(), count))
        q_done.get(timeout=120)
        box = S.device_tensor(ptr, 4 * count, device=torch.device("cuda", 0))
        q_result.put(box.cpu().numpy())


def _peer(q_handle, q_done):
    import torch

    import paper_2106_13465_b200 as P
    from paper_2106_13465_b200 import slab as S
    torch.cuda.set_device(0)
    handle, count = q_handle.get(timeout=120)
    with P.GpuGrid(8, 40, 1 / 8, 1 / 40, P.GasModel(), "reflect", device=0) as g:
        ptr = g.ipc_open(handle)
        peer = S.device_tensor(ptr, 4 * count, device=torch.device("cuda", 0))
        peer.copy_(torch.arange(4 * count, dtype=torch.float64, device="cuda"))
        torch.cuda.synchronize()
        q_done.put(True)


def test_inbox_ipc_roundtrip_between_processes(gpu):
    ctx = mp.get_context("spawn")
    q_handle, q_done, q_result = ctx.Queue(), ctx.Queue(), ctx.Queue()
    a = ctx.Process(target=_owner, args=(q_handle, q_done, q_result))
    b = ctx.Process(target=_peer, args=(q_handle, q_done))
    a.start()
    b.start()
    got = q_result.get(timeout=180)
    b.join(60)
    a.join(60)
    assert a.exitcode == 0 and b.exitcode == 0
    assert np.array_equal(got, np.arange(got.size, dtype=np.float64))
