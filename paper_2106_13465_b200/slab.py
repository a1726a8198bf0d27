"""Row-slab decomposition of one HYDRO grid over several GPUs.

The grid's i axis (the slow memory axis, grid.hpp:54-57) is split into
near-equal slabs, one per rank, exactly like split_range
(proj/src/decomposition.cpp:9-16).  Per step the only exchanges are

  * the dt min-allreduce: every slab's min of cell_dt_limit, folded into one
    value, the distributed twin of compute_dt_parallel's slot-min
    (proj/src/schedulers.cpp:47-65) -- min is exact and order-free, so the
    result is bitwise the sequential dt;
  * one 2-row halo swap before the column sweep: rows 1..2 go to the rank
    above, rows n-1..n to the rank below -- the column-sweep InterfaceBuffer of
    the reference (decomposition.hpp:58-79).  The row sweep is slab-local.

The driver is written against two small protocols so the same code path runs
over NCCL on B200s (GpuSlab + TorchComm(nccl)) and over gloo on CPU in the
tests (an oracle-backed slab + TorchComm(gloo)).

Halo transport.  With peer memory (NVLink; CUDA IPC between the rank
processes) the halo needs no communication call at all: the row sweep of
step s stores its rows 1..2 / n-1..n straight into the neighbours' inboxes
(parity (s+1)&1) and each rank copies its own inbox into its ghost rows
before the column sweep of step s+1 (include/hydro_gpu.h,
hydro_gpu_set_halo_peers).  The dt min-allreduce that sits between the two on
every rank's stream is the synchronisation: a neighbour's allreduce of step
s+1 cannot complete before this rank's row sweep of step s has, and the
inbox parity keeps the neighbour's next write off the block being read.  All
ranks agree on the transport collectively (TorchComm.setup_p2p); otherwise
(or with HYDRO_HALO=nccl) the halo is one batched send/recv per neighbour.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

from .hydro import GasModel, GpuGrid

NO_ERROR = (1 << 64) - 1


def split_rows(nx: int, parts: int, part: int) -> tuple[int, int]:
    """(row0, rows) of slab `part`: the first nx % parts slabs get one extra row
    (split_range, decomposition.cpp:9-16).  row0 is the global row of local
    row 1, minus 1."""
    base, extra = divmod(nx, parts)
    rows = base + (1 if part < extra else 0)
    row0 = part * base + min(part, extra)
    return row0, rows


@dataclass
class SlabGeometry:
    global_nx: int
    ny: int
    rank: int
    world: int

    @property
    def row0(self) -> int:
        return split_rows(self.global_nx, self.world, self.rank)[0]

    @property
    def nx(self) -> int:
        return split_rows(self.global_nx, self.world, self.rank)[1]

    @property
    def wall_lo(self) -> bool:
        return self.rank == 0

    @property
    def wall_hi(self) -> bool:
        return self.rank == self.world - 1


class _DeviceView:
    """__cuda_array_interface__ over library-owned device memory, so torch can
    alias it without a copy."""

    def __init__(self, ptr: int, count: int, typestr: str = "<f8"):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def device_tensor(ptr: int, count: int, dtype=torch.float64, device=None) -> torch.Tensor:
    typestr = {torch.float64: "<f8", torch.int64: "<i8"}[dtype]
    return torch.as_tensor(_DeviceView(ptr, count, typestr), device=device)


class GpuSlab:
    """One rank's slab, resident on one GPU (a hydro_gpu_ctx in slab mode)."""

    def __init__(self, geo: SlabGeometry, dx: float, dy: float, model: GasModel, bc: str,
                 device: int, flux: str = "hllc", math: str = "bitwise"):
        self.geo = geo
        self.device = torch.device("cuda", device)
        self.grid = GpuGrid(geo.nx, geo.ny, dx, dy, model, bc, device=device, row0=geo.row0,
                            global_nx=geo.global_nx, wall_lo=geo.wall_lo, wall_hi=geo.wall_hi,
                            flux=flux, math=math)
        h = self.grid.halo()
        n = h["count"]
        self._halo = {k: device_tensor(h[k], n, device=self.device)
                      for k in ("send_lo", "send_hi", "recv_lo", "recv_hi")}
        self._limits = [device_tensor(self.grid.limit_slot(s), 1, device=self.device)
                        for s in (0, 1)]
        self._err = device_tensor(self.grid.error_slot(), 1, torch.int64, device=self.device)
        self.p2p = False

    def bind_stream(self, stream: torch.cuda.Stream):
        self.grid.set_stream(stream.cuda_stream)

    # peer-memory halo --------------------------------------------------------
    def inbox_ptr(self) -> int:
        return self.grid.inbox()[0]

    def ipc_handle(self) -> bytes:
        return self.grid.inbox_ipc_handle()

    def open_peer(self, handle: bytes) -> int:
        return self.grid.ipc_open(handle)

    def set_peers(self, upper: int | None, lower: int | None):
        self.grid.set_halo_peers(upper, lower)
        self.p2p = True

    def halo_out(self, step: int):
        self.grid.slab_halo_out(step)

    def inbox_in(self, step: int):
        self.grid.slab_inbox_in(step)

    # phases ------------------------------------------------------------------
    def prologue(self, step: int):
        self.grid.slab_prologue(step)

    def sweep_x(self, step: int):
        self.grid.slab_sweep_x(step)

    def sweep_y(self, step: int):
        self.grid.slab_sweep_y(step)

    def finish(self):
        self.grid.slab_finish()

    # exchange buffers ----------------------------------------------------------
    def limit(self, step: int) -> torch.Tensor:
        return self._limits[step & 1]

    def halo_send(self) -> tuple[torch.Tensor, torch.Tensor]:
        self.grid.slab_halo_pack()  # rows 1..2 / n-1..n of the tiled state -> the send blocks
        return self._halo["send_lo"], self._halo["send_hi"]

    def halo_recv(self) -> tuple[torch.Tensor, torch.Tensor]:
        return self._halo["recv_lo"], self._halo["recv_hi"]

    def halo_done(self):
        self.grid.slab_halo_unpack()  # the received blocks -> ghost rows

    def error_key(self) -> torch.Tensor:
        return self._err

    def raise_error(self, key: int):
        self.grid.raise_error_key(key)


class TorchComm:
    """Exchange steps over a torch.distributed process group (nccl on GPUs,
    gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def min_limit(self, t: torch.Tensor):
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)

    def swap_halos(self, slab):
        if self.world == 1:
            return
        send_lo, send_hi = slab.halo_send()
        recv_lo, recv_hi = slab.halo_recv()
        ops = []
        P2POp = self.dist.P2POp
        if self.rank > 0:
            ops.append(P2POp(self.dist.isend, send_lo, self.rank - 1, self.group))
            ops.append(P2POp(self.dist.irecv, recv_lo, self.rank - 1, self.group))
        if self.rank < self.world - 1:
            ops.append(P2POp(self.dist.isend, send_hi, self.rank + 1, self.group))
            ops.append(P2POp(self.dist.irecv, recv_hi, self.rank + 1, self.group))
        for req in self.dist.batch_isend_irecv(ops):
            req.wait()
        slab.halo_done()

    def _all_true(self, ok: bool) -> bool:
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return bool(t.item())

    def setup_p2p(self, slab) -> bool:
        """Collective: maps the neighbours' inboxes into this rank (CUDA IPC)
        and switches every rank to the peer-memory halo -- only if all ranks
        succeeded, so the ranks never disagree on the transport."""
        self.p2p = False
        if self.world == 1:
            return False
        want = os.environ.get("HYDRO_HALO", "p2p") == "p2p"
        ok, handle = want, None
        if ok:
            try:
                handle = slab.ipc_handle()
            except Exception:  # noqa: BLE001 -- any failure means: use NCCL
                ok = False
        handles = [None] * self.world
        self.dist.all_gather_object(handles, handle, group=self.group)
        up = dn = None
        if ok:
            try:
                if self.rank > 0:
                    up = slab.open_peer(handles[self.rank - 1])
                if self.rank < self.world - 1:
                    dn = slab.open_peer(handles[self.rank + 1])
            except Exception:  # noqa: BLE001
                ok = False
        if self._all_true(ok):
            slab.set_peers(up, dn)
            self.p2p = True
        return self.p2p

    def setup_native(self, slab) -> bool:
        """Collective: hands the whole step schedule to the library
        (hydro_gpu_comm_attach): per rank ONE captured CUDA graph per run with
        an NCCL min-allreduce of the dt limit per step, the peer-memory halo
        and the first error over all ranks -- no per-step host calls.  Only
        over NCCL (one GPU per rank) with the peer-memory halo in place, and
        only if every rank can load NCCL; otherwise the Python schedule
        (run_slab) stays.  HYDRO_SLAB_DRIVER=python forces the latter."""
        from .hydro import comm_unique_id
        self.native = False
        want = (os.environ.get("HYDRO_SLAB_DRIVER", "native") == "native"
                and self.dist.get_backend(self.group) == "nccl"
                and (self.world == 1 or getattr(self, "p2p", False)))
        uid = None
        if want and self.rank == 0:
            try:
                uid = comm_unique_id()
            except Exception:  # noqa: BLE001 -- no NCCL: stay on the Python schedule
                uid = None
        box = [uid]
        self.dist.broadcast_object_list(box, src=0, group=self.group)
        uid = box[0]
        if not self._all_true(want and uid is not None):
            return False
        slab.grid.comm_attach(uid, self.world, self.rank)
        self.native = True
        return True

    def first_error(self, key: torch.Tensor) -> int:
        if self.world == 1:
            keys = [key.clone()]
        else:
            keys = [torch.empty_like(key) for _ in range(self.world)]
            self.dist.all_gather(keys, key, group=self.group)
        vals = [int(k.cpu().item()) & NO_ERROR for k in keys]
        return min(vals)


class LoopbackComm:
    """All slabs in one process (tests on a single device): exchanges are
    plain copies, phases run slab after slab in stream order."""

    def __init__(self, slabs):
        self.slabs = slabs
        self.p2p = False

    def setup_p2p(self) -> bool:
        """Peer-memory halo between slabs of one process: the neighbours'
        inboxes are plain device pointers (no IPC needed)."""
        ptrs = [s.inbox_ptr() for s in self.slabs]
        n = len(self.slabs)
        for k, s in enumerate(self.slabs):
            s.set_peers(ptrs[k - 1] if k > 0 else None, ptrs[k + 1] if k < n - 1 else None)
        self.p2p = n > 1
        return self.p2p

    def min_limit_all(self, step: int):
        lims = torch.stack([s.limit(step) for s in self.slabs])
        m = lims.min(dim=0).values
        for s in self.slabs:
            s.limit(step).copy_(m)

    def swap_halos_all(self):
        for a, b in zip(self.slabs[:-1], self.slabs[1:]):
            a_lo, a_hi = a.halo_send()
            b_lo, b_hi = b.halo_send()
            a.halo_recv()[1].copy_(b_lo)
            b.halo_recv()[0].copy_(a_hi)
        for s in self.slabs:
            s.halo_done()

    def first_error(self) -> int:
        return min(int(s.error_key().cpu().item()) & NO_ERROR for s in self.slabs)


def run_slab(slab, comm: TorchComm, steps: int) -> None:
    """run_sequential's step order on one rank's slab.  All device work is
    enqueued on the current stream; the only host synchronisation is the
    final error gather."""
    if steps <= 0:
        return
    if getattr(comm, "native", False):  # the library runs the whole schedule
        slab.grid.run(steps)
        return
    p2p = getattr(comm, "p2p", False)
    slab.prologue(0)
    if p2p:
        slab.halo_out(0)
    for s in range(steps):
        comm.min_limit(slab.limit(s))  # also orders the peer-memory halo
        if p2p:
            slab.inbox_in(s)
        else:
            comm.swap_halos(slab)
        slab.sweep_x(s)
        slab.sweep_y(s)
    slab.finish()
    key = comm.first_error(slab.error_key())
    if key != NO_ERROR:
        slab.raise_error(key)


def run_loopback(slabs, steps: int, p2p: bool = False) -> None:
    """Same schedule as run_slab for several slabs held by one process."""
    if steps <= 0:
        return
    comm = LoopbackComm(slabs)
    if p2p:
        comm.setup_p2p()
    for sl in slabs:
        sl.prologue(0)
    if comm.p2p:
        for sl in slabs:
            sl.halo_out(0)
    for s in range(steps):
        comm.min_limit_all(s)
        if comm.p2p:
            for sl in slabs:
                sl.inbox_in(s)
        else:
            comm.swap_halos_all()
        for sl in slabs:
            sl.sweep_x(s)
        for sl in slabs:
            sl.sweep_y(s)
    for sl in slabs:
        sl.finish()
    key = comm.first_error()
    if key != NO_ERROR:
        slabs[0].raise_error(key)


def chained_digest(planes, nx: int, ny: int, rank: int, world: int, send, recv) -> int | None:
    """The reference's grid digest (audit.cpp:53-76) of a grid held as row
    slabs, without gathering it: FNV-1a is a byte-serial chain, so each rank
    continues the state of the rank above over its own rows, plane by plane
    (send(h, to_rank) / recv(from_rank) -> h carry the 64-bit state).
    Returns the digest on rank world-1, None elsewhere."""
    from .hydro import FNV_BASIS, fnv1a_rows
    h = FNV_BASIS
    if world == 1:
        for v in range(4):
            h = fnv1a_rows(h, planes[v], nx, ny)
        return h
    for v in range(4):
        if not (v == 0 and rank == 0):
            h = recv(rank - 1 if rank > 0 else world - 1)
        h = fnv1a_rows(h, planes[v], nx, ny)
        if not (v == 3 and rank == world - 1):
            send(h, rank + 1 if rank < world - 1 else 0)
    return h if rank == world - 1 else None


def gather_planes(slabs_or_planes, global_nx: int, ny: int):
    """Assembles full Grid2D planes from per-slab planes (rank order).  Ghost
    rows of the global grid come from the outer slabs."""
    import numpy as np
    out = np.zeros((4, global_nx + 4, ny + 4))
    parts = list(slabs_or_planes)
    world = len(parts)
    for r, planes in enumerate(parts):
        row0, n = split_rows(global_nx, world, r)
        lo = 0 if r == 0 else 2
        hi = n + 4 if r == world - 1 else n + 2
        out[:, row0 + lo: row0 + hi, :] = planes[:, lo:hi, :]
    return out


def slab_planes(full, global_nx: int, world: int, rank: int):
    """The (4, n+4, ny+4) planes of slab `rank` cut from full-grid planes,
    including the 2 neighbour rows on each side."""
    row0, n = split_rows(global_nx, world, rank)
    return full[:, row0: row0 + n + 4, :].copy()
