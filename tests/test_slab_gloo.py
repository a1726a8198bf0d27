"""The multi-GPU slab driver (paper_2106_13465_b200/slab.py) over a real
2-rank torch.distributed gloo group on CPU.

The per-slab physics is supplied by the oracle (test infrastructure), so what
is under test is the driver itself: row split, which rows are exchanged with
which neighbour, the order of halo swap / dt min-allreduce / sweeps, and the
first-error gather.  The gathered result must be bitwise the single-domain
reference run.
"""
import os
import socket
import tempfile
import time

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2106_13465_b200 import slab as S

NX, NY, STEPS = 41, 26, 14


class OracleSlab:
    """Slab backend computing with the CPU oracle on numpy planes."""

    def __init__(self, geo, planes, dx, dy, bc, cfl=0.8):
        self.geo, self.bc, self.cfl = geo, bc, cfl
        self.g = O.Grid(geo.nx, NY, dx, dy, planes)
        self.lims = [torch.zeros(1, dtype=torch.float64) for _ in range(2)]
        self._recv = None
        self.err = torch.full((1,), -1, dtype=torch.int64)
        self.walls = (O.WALL_XLO if geo.wall_lo else 0) | (O.WALL_XHI if geo.wall_hi else 0)

    def prologue(self, step):
        O.apply_boundary(self.g, self.bc, self.walls)
        self.lims[step & 1][0] = O.compute_limit(self.g)

    def limit(self, step):
        return self.lims[step & 1]

    def halo_send(self):
        n = self.geo.nx
        u = self.g.u
        return (torch.from_numpy(np.ascontiguousarray(u[:, 2:4, :])).reshape(-1),
                torch.from_numpy(np.ascontiguousarray(u[:, n:n + 2, :])).reshape(-1))

    def halo_recv(self):
        size = 4 * 2 * (NY + 4)
        self._recv = (torch.zeros(size, dtype=torch.float64), torch.zeros(size, dtype=torch.float64))
        return self._recv

    def halo_done(self):
        n = self.geo.nx
        if not self.geo.wall_lo:
            self.g.u[:, 0:2, :] = self._recv[0].numpy().reshape(4, 2, NY + 4)
        if not self.geo.wall_hi:
            self.g.u[:, n + 2:n + 4, :] = self._recv[1].numpy().reshape(4, 2, NY + 4)

    def sweep_x(self, step):
        dt = self.cfl * float(self.lims[step & 1][0])
        O.sweep_axis(self.g, 0, dt)
        O.apply_boundary(self.g, self.bc, O.WALL_Y)

    def sweep_y(self, step):
        dt = self.cfl * float(self.lims[step & 1][0])
        O.sweep_axis(self.g, 1, dt)
        O.apply_boundary(self.g, self.bc, self.walls)
        self.lims[(step + 1) & 1][0] = O.compute_limit(self.g)

    def finish(self):
        pass

    def error_key(self):
        return self.err

    def raise_error(self, key):
        raise RuntimeError(f"error key {key:x}")


class PeerOracleSlab(OracleSlab):
    """OracleSlab with the peer-memory halo of GpuSlab: the inbox (2 parities
    x 2 sides x one 2-row block) is a shared file mapping, its "IPC handle"
    the file name, and the row sweep writes its rows 1..2 / n-1..n into the
    neighbours' inboxes of parity (s+1)&1 -- the same protocol as the row
    sweep kernel over NVLink, exercised by real concurrent processes."""

    def __init__(self, geo, planes, dx, dy, bc, outdir, fail_handle=False, jitter=0.0):
        super().__init__(geo, planes, dx, dy, bc)
        self.rng = np.random.default_rng(geo.rank)
        self.jitter = jitter
        self.path = os.path.join(outdir, f"inbox{geo.rank}.bin")
        self.inbox = np.memmap(self.path, dtype=np.float64, mode="w+", shape=(2, 2, 4, 2, NY + 4))
        self.fail_handle = fail_handle
        self.up = self.dn = None
        self.p2p = False

    def ipc_handle(self):
        if self.fail_handle:
            raise RuntimeError("no peer access")
        return self.path.encode()

    def open_peer(self, handle):
        return np.memmap(handle.decode(), dtype=np.float64, mode="r+", shape=(2, 2, 4, 2, NY + 4))

    def set_peers(self, upper, lower):
        self.up, self.dn = upper, lower
        self.p2p = True

    def halo_out(self, step):
        par, n, u = step & 1, self.geo.nx, self.g.u
        if self.up is not None:
            self.up[par, 1] = u[:, 2:4, :]      # rows 1..2 -> its ghost rows n'+1..n'+2
            self.up.flush()
        if self.dn is not None:
            self.dn[par, 0] = u[:, n:n + 2, :]  # rows n-1..n -> its ghost rows -1..0
            self.dn.flush()

    def _wait(self):
        if self.jitter:  # random per-rank delays: perturb the interleaving of ranks
            time.sleep(self.rng.uniform(0, self.jitter))

    def sweep_x(self, step):
        self._wait()
        super().sweep_x(step)

    def inbox_in(self, step):
        self._wait()
        if self.jitter and self.geo.rank % 2:  # a slow reader: neighbours race ahead
            time.sleep(0.03)
        par, n = step & 1, self.geo.nx
        if not self.geo.wall_lo:
            self.g.u[:, 0:2, :] = self.inbox[par, 0]
        if not self.geo.wall_hi:
            self.g.u[:, n + 2:n + 4, :] = self.inbox[par, 1]

    def sweep_y(self, step):
        super().sweep_y(step)
        self._wait()
        if self.p2p:
            self.halo_out(step + 1)


def _worker(rank, world, port, case, bc, outdir, mode="nccl"):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                           world_size=world)
    full = O.make_case(case, NX, NY, seed=6)
    geo = S.SlabGeometry(NX, NY, rank, world)
    planes = S.slab_planes(full.u, NX, world, rank)
    comm = S.TorchComm()
    if mode == "nccl":
        sl = OracleSlab(geo, planes, full.dx, full.dy, bc)
    else:
        sl = PeerOracleSlab(geo, planes, full.dx, full.dy, bc, outdir,
                            fail_handle=(mode == "p2p_fail" and rank == 1),
                            jitter=0.01 if mode == "p2p_jitter" else 0.0)
        used = comm.setup_p2p(sl)
        assert used == (mode != "p2p_fail")  # every rank agrees on the transport
    S.run_slab(sl, comm, STEPS)
    np.save(os.path.join(outdir, f"slab{rank}.npy"), sl.g.u)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,case,bc", [(2, "corner_blast", "reflect"), (2, "random", "transmit"),
                                           (3, "sod_x", "transmit")])
def test_slab_driver_over_gloo_matches_single_domain(world, case, bc):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), case, bc, d), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"slab{r}.npy")) for r in range(world)]
    got = S.gather_planes(parts, NX, NY)
    ref = O.make_case(case, NX, NY, seed=6)
    O.run_sequential(ref, STEPS, bc)
    assert np.array_equal(got[:, 2:NX + 2, 2:NY + 2], ref.u[:, 2:NX + 2, 2:NY + 2])


@pytest.mark.parametrize("mode", ["p2p", "p2p_fail", "p2p_jitter"])
@pytest.mark.parametrize("world,case,bc", [(2, "random", "transmit"), (3, "corner_blast", "reflect")])
def test_peer_memory_halo_schedule_over_gloo(world, case, bc, mode):
    """The peer-memory halo protocol (row sweep writes the neighbours' inbox
    of parity (s+1)&1, the reader copies parity s&1 after the dt allreduce)
    with truly concurrent ranks; p2p_fail: one rank cannot export its inbox,
    so all ranks fall back to send/recv together."""
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), case, bc, d, mode), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"slab{r}.npy")) for r in range(world)]
    got = S.gather_planes(parts, NX, NY)
    ref = O.make_case(case, NX, NY, seed=6)
    O.run_sequential(ref, STEPS, bc)
    assert np.array_equal(got[:, 2:NX + 2, 2:NY + 2], ref.u[:, 2:NX + 2, 2:NY + 2])


@pytest.mark.parametrize("nx,parts", [(10, 3), (41, 2), (16384 * 8, 8), (7, 7)])
def test_split_rows_is_split_range(nx, parts):
    rows = [S.split_rows(nx, parts, p) for p in range(parts)]
    assert sum(n for _, n in rows) == nx
    assert rows[0][0] == 0
    for (r0, n), (r1, _) in zip(rows, rows[1:]):
        assert r1 == r0 + n
    assert max(n for _, n in rows) - min(n for _, n in rows) <= 1
    assert rows[0][1] >= rows[-1][1]  # extra rows go to the first slabs


def test_gather_of_cut_slabs_is_identity():
    full = O.make_case("random", NX, NY, seed=2).u
    for world in (1, 2, 5):
        parts = [S.slab_planes(full, NX, world, r) for r in range(world)]
        assert np.array_equal(S.gather_planes(parts, NX, NY), full)


def _digest_worker(rank, world, port, case, bc, outdir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = O.make_case(case, NX, NY, seed=6)
    geo = S.SlabGeometry(NX, NY, rank, world)
    sl = OracleSlab(geo, S.slab_planes(full.u, NX, world, rank), full.dx, full.dy, bc)
    comm = S.TorchComm()
    # the C++ schedule needs NCCL: over gloo every rank stays on the Python one
    assert comm.setup_native(sl) is False and not comm.native
    S.run_slab(sl, comm, STEPS)

    def send(h, to):
        dist.send(torch.tensor([h - (1 << 64) if h >= (1 << 63) else h], dtype=torch.int64), to)

    def recv(frm):
        t = torch.zeros(1, dtype=torch.int64)
        dist.recv(t, frm)
        return int(t.item()) & ((1 << 64) - 1)

    planes = np.ascontiguousarray(sl.g.u)
    h = S.chained_digest(planes, geo.nx, NY, rank, world, send, recv)
    if rank == world - 1:
        with open(os.path.join(outdir, "digest"), "w") as f:
            f.write(f"{h:016x}")
    dist.destroy_process_group()


@pytest.mark.parametrize("world,case,bc", [(2, "random", "transmit"), (3, "corner_blast", "reflect")])
def test_chained_slab_digest_is_the_grid_digest(world, case, bc):
    """The reference's byte-serial FNV-1a digest (audit.cpp:53-76) of a grid
    held as row slabs, chained over the ranks plane by plane without gathering
    the grid (bench.py gates multi-rank runs on it), equals the digest of the
    single-domain run."""
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_digest_worker, args=(world, _free_port(), case, bc, d), nprocs=world, join=True)
        got = open(os.path.join(d, "digest")).read()
    ref = O.make_case(case, NX, NY, seed=6)
    O.run_sequential(ref, STEPS, bc)
    assert got == f"{O.digest(ref):016x}"
