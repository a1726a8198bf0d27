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
"""
from __future__ import annotations

import ctypes as C
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
                 device: int, flux: str = "hllc"):
        self.geo = geo
        self.device = torch.device("cuda", device)
        self.grid = GpuGrid(geo.nx, geo.ny, dx, dy, model, bc, device=device, row0=geo.row0,
                            global_nx=geo.global_nx, wall_lo=geo.wall_lo, wall_hi=geo.wall_hi,
                            flux=flux)
        h = self.grid.halo()
        n = h["count"]
        self._halo = {k: device_tensor(h[k], n, device=self.device)
                      for k in ("send_lo", "send_hi", "recv_lo", "recv_hi")}
        self._limits = [device_tensor(self.grid.limit_slot(s), 1, device=self.device)
                        for s in (0, 1)]
        self._err = device_tensor(self.grid.error_slot(), 1, torch.int64, device=self.device)

    def bind_stream(self, stream: torch.cuda.Stream):
        self.grid.set_stream(stream.cuda_stream)

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
        return self._halo["send_lo"], self._halo["send_hi"]

    def halo_recv(self) -> tuple[torch.Tensor, torch.Tensor]:
        return self._halo["recv_lo"], self._halo["recv_hi"]

    def halo_done(self):
        pass  # received straight into the ghost rows

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
    slab.prologue(0)
    for s in range(steps):
        comm.min_limit(slab.limit(s))
        comm.swap_halos(slab)
        slab.sweep_x(s)
        slab.sweep_y(s)
    slab.finish()
    key = comm.first_error(slab.error_key())
    if key != NO_ERROR:
        slab.raise_error(key)


def run_loopback(slabs, steps: int) -> None:
    """Same schedule as run_slab for several slabs held by one process."""
    if steps <= 0:
        return
    comm = LoopbackComm(slabs)
    for sl in slabs:
        sl.prologue(0)
    for s in range(steps):
        comm.min_limit_all(s)
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
