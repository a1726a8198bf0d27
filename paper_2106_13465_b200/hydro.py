"""Host-side mirror of the reference hydro2d interface for the GPU path.

Names, argument meaning and error behaviour follow the reference (paths
relative to /root/reference/):

===========================================  =================================
reference                                    here
===========================================  =================================
``GasModel`` (include/hydro/types.hpp:38-41)  :class:`GasModel`
``Grid2D`` (include/hydro/grid.hpp:26-64)     :class:`Grid2D` (numpy planes)
``make_case`` (src/bench.cpp:24-37)           :func:`make_case` (+ BASELINE cases)
``run_sequential`` (schedulers.hpp:24)        :func:`run_gpu`
``advance_sequential`` (schedulers.hpp:21)    :func:`advance_gpu`
``run_until`` (schedulers.hpp:28)             :func:`run_until_gpu`
``compute_dt`` (euler_kernel.hpp:75)          :func:`compute_dt_gpu`
``grid_checksum().digest`` (audit.hpp:34)     :func:`grid_digest`
``hydro::Error`` + categories (errors.hpp)    :class:`HydroError` & subclasses
===========================================  =================================

All stepping runs in libhydro_b200.so on the GPU; nothing here computes
physics.  Errors carry the reference's category and message text, e.g.
``step 3: column sweep strip 17: rho non-positive at strip cell -2``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from . import _lib as L


class ErrorCategory(IntEnum):
    """hydro::ErrorCategory (errors.hpp:10-18), numbered +1; CUDA = device failure."""
    CONFIG = 1
    POSITIVITY = 2
    PROTOCOL = 3
    TASK_GRAPH = 4
    EQUIVALENCE = 5
    IO = 6
    VALIDATION = 7
    CUDA = 8


_CATEGORY_NAME = {1: "config", 2: "positivity", 3: "protocol", 4: "task-graph",
                  5: "equivalence", 6: "io", 7: "validation", 8: "cuda"}


class HydroError(RuntimeError):
    """hydro::Error: a message plus an ErrorCategory (errors.hpp:20-29)."""

    def __init__(self, category: int, message: str, info: dict | None = None):
        super().__init__(message)
        self.category = ErrorCategory(category)
        self.info = info or {}

    def cli_line(self) -> str:
        """The CLI's one-line rendering (tools/hydrobench.cpp:153-159)."""
        return f"error: {_CATEGORY_NAME[int(self.category)]}: {self}"


class ConfigError(HydroError):
    def __init__(self, message: str):
        super().__init__(ErrorCategory.CONFIG, message)


class PositivityError(HydroError):
    """Carries the non-positive field like PositivityError (errors.hpp:40-49)."""

    @property
    def field(self) -> str:
        return ("rho", "pres", "internal energy")[self.info.get("field", 0)]


class DeviceError(HydroError):
    pass


class ValidationError(HydroError):
    """ErrorCategory::Validation, e.g. a vacuum-generating Riemann problem in
    the exact-10 flux mode (exact_riemann.cpp:55-57)."""


def _raise_for(status: int, info: L.ErrorInfo | None = None, message: str | None = None):
    if status == 0:
        return
    msg = message if message is not None else (info.message.decode() if info else "")
    details = {}
    if info is not None:
        details = {k: getattr(info, k) for k in ("step", "phase", "strip", "loop", "cell", "field")}
    if status == ErrorCategory.POSITIVITY:
        raise PositivityError(status, msg, details)
    if status == ErrorCategory.VALIDATION:
        raise ValidationError(status, msg, details)
    if status == ErrorCategory.CONFIG:
        raise ConfigError(msg or "invalid configuration")
    if status == ErrorCategory.CUDA:
        raise DeviceError(status, msg or "CUDA failure")
    raise HydroError(status, msg, details)


@dataclass(frozen=True)
class GasModel:
    gamma: float = 1.4
    cfl: float = 0.8


BC = {"reflect": 0, "transmit": 1}
FLUX = {"hllc": 0, "exact10": 1}
# Sweep arithmetic (include/hydro_gpu.h, enum hydro_gpu_math): "bitwise" is the
# reference's bits; "tolerance" holds compare_tolerance max_rel <= 1e-12.
MATH = {"bitwise": 0, "tolerance": 1}
SCHEDULE = {"split": 0, "fused": 1, "auto": 2}
CASES = {"uniform": 0, "blast": 1, "sod": 2, "corner_blast": 3, "sod_x": 4, "random": 5}
RHO, MOM_X, MOM_Y, ENER = 0, 1, 2, 3


class Grid2D:
    """Four (nx+4) x (ny+4) fp64 planes, row-major, j fastest (grid.hpp:15-19)."""

    def __init__(self, nx: int, ny: int, dx: float, dy: float, planes: np.ndarray | None = None):
        if nx < 4 or ny < 4:
            raise ConfigError(f"grid interior must be at least 4x4, got {nx}x{ny}")
        if not (dx > 0.0) or not (dy > 0.0):
            raise ConfigError("cell sizes must be positive")
        self.nx, self.ny, self.dx, self.dy = nx, ny, dx, dy
        if planes is None:
            planes = np.zeros((4, nx + 4, ny + 4))
        if planes.shape != (4, nx + 4, ny + 4) or planes.dtype != np.float64:
            raise ConfigError("planes must be float64 of shape (4, nx+4, ny+4)")
        self.planes = np.ascontiguousarray(planes)

    def at(self, var: int, i: int, j: int) -> float:
        return float(self.planes[var, i + 1, j + 1])

    def cell(self, i: int, j: int) -> tuple:
        return tuple(float(self.planes[v, i + 1, j + 1]) for v in range(4))

    def interior(self) -> np.ndarray:
        return self.planes[:, 2:self.nx + 2, 2:self.ny + 2]

    def copy(self) -> "Grid2D":
        return Grid2D(self.nx, self.ny, self.dx, self.dy, self.planes.copy())


def make_case(case: str, nx: int, ny: int, model: GasModel = GasModel(), seed: int = 0) -> Grid2D:
    """Initial conditions: the reference's uniform/blast/sod (cases.cpp:11-69)
    plus the BASELINE configs' corner_blast, sod_x and random."""
    if case not in CASES:
        raise ConfigError(f"unknown case '{case}' (expected one of {', '.join(CASES)})")
    if case == "sod":
        nx = 4
    planes = np.zeros((4, nx + 4, ny + 4))
    dx, dy = C.c_double(), C.c_double()
    rc = L.lib().hydro_init_case_host(CASES[case], nx, ny, model.gamma, seed,
                                      L.planes_of(planes), ny + 4, C.byref(dx), C.byref(dy))
    if rc:
        raise ConfigError(f"cannot build case '{case}' on a {nx}x{ny} grid")
    return Grid2D(nx, ny, dx.value, dy.value, planes)


def grid_digest(grid: Grid2D) -> int:
    """FNV-1a over the interior bytes (audit.cpp:53-76)."""
    return int(L.lib().hydro_grid_digest(L.planes_of(grid.planes), grid.ny + 4, grid.nx, grid.ny))


FNV_BASIS = 14695981039346656037


def fnv1a_rows(h: int, plane: np.ndarray, nx: int, ny: int) -> int:
    """FNV-1a of grid_digest continued from state h over interior rows 1..nx of
    one (nx+4, ny+4) plane; chaining it over (plane, row slab) in plane-major,
    slab order from FNV_BASIS gives the whole grid's digest."""
    assert plane.dtype == np.float64 and plane.flags.c_contiguous
    return int(L.lib().hydro_fnv1a_rows(h, plane.ctypes.data_as(L._dp), plane.shape[1], nx, ny))


def comm_unique_id() -> bytes:
    """An NCCL unique id for hydro_gpu_comm_attach (made on one rank)."""
    buf = C.create_string_buffer(128)
    rc = L.lib().hydro_gpu_comm_unique_id(buf)
    if rc:
        raise DeviceError(rc, "NCCL unavailable (libnccl.so.2)")
    return buf.raw


def grid_state_hash(grid: Grid2D) -> int:
    """Composable state hash (FNV-1a over per-row FNV-1a hashes) of host planes;
    equals GpuGrid.state_hash() of the same state."""
    return int(L.lib().hydro_grid_state_hash(L.planes_of(grid.planes), grid.ny + 4, grid.nx, grid.ny))


def combine_row_hashes(rows) -> int:
    arr = np.ascontiguousarray(rows, dtype=np.uint64)
    return int(L.lib().hydro_combine_row_hashes(arr.ctypes.data_as(C.POINTER(C.c_uint64)), arr.size))


class GpuGrid:
    """One device-resident grid (or row slab): a hydro_gpu_ctx."""

    def __init__(self, nx: int, ny: int, dx: float, dy: float, model: GasModel = GasModel(),
                 bc: str = "reflect", device: int = -1, row0: int = 0, global_nx: int | None = None,
                 wall_lo: bool = True, wall_hi: bool = True, flux: str = "hllc",
                 math: str = "bitwise"):
        if bc not in BC:
            raise ConfigError(f"unknown boundary '{bc}' (expected reflect or transmit)")
        if flux not in FLUX:
            raise ConfigError(f"unknown flux '{flux}' (expected hllc or exact10)")
        self.flux = flux
        self.nx, self.ny, self.dx, self.dy = nx, ny, dx, dy
        self.model, self.bc = model, bc
        self.row0 = row0
        self.global_nx = global_nx if global_nx is not None else nx
        cfg = L.Cfg(nx, ny, dx, dy, model.gamma, model.cfl, BC[bc], FLUX[flux], device, row0,
                    self.global_nx, int(wall_lo), int(wall_hi))
        self._lib = L.lib()
        self._ctx = C.c_void_p()
        rc = self._lib.hydro_gpu_create(C.byref(cfg), C.byref(self._ctx))
        if rc:
            _raise_for(rc, message=f"hydro_gpu_create failed ({self._lib.hydro_gpu_status_string(rc).decode()}) "
                                   f"for a {nx}x{ny} grid")
        self.math = "bitwise"
        if math != "bitwise":
            self.set_math(math)

    # -- lifetime ---------------------------------------------------------
    def close(self):
        if self._ctx:
            self._lib.hydro_gpu_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._ctx

    def _check(self, rc: int):
        if rc:
            info = L.ErrorInfo()
            self._lib.hydro_gpu_last_error(self._ctx, C.byref(info))
            _raise_for(rc, info)

    # -- transfer ---------------------------------------------------------
    def upload(self, planes: np.ndarray):
        self._check(self._lib.hydro_gpu_upload(self._ctx, L.planes_of(planes), planes.shape[2]))

    def download(self, planes: np.ndarray):
        self._check(self._lib.hydro_gpu_download(self._ctx, L.planes_of(planes), planes.shape[2]))

    def upload_ptr(self, plane_ptrs, row_stride: int):
        arr = L._planes(*[C.cast(C.c_void_p(p), L._dp) for p in plane_ptrs])
        self._check(self._lib.hydro_gpu_upload(self._ctx, arr, row_stride))

    def download_ptr(self, plane_ptrs, row_stride: int):
        arr = L._planes(*[C.cast(C.c_void_p(p), L._dp) for p in plane_ptrs])
        self._check(self._lib.hydro_gpu_download(self._ctx, arr, row_stride))

    def upload_ptr_async(self, plane_ptrs, row_stride: int):
        """hydro_gpu_upload_async: enqueued on the context's stream (pinned
        host planes that stay alive until sync)."""
        arr = L._planes(*[C.cast(C.c_void_p(p), L._dp) for p in plane_ptrs])
        self._check(self._lib.hydro_gpu_upload_async(self._ctx, arr, row_stride))

    def download_ptr_async(self, plane_ptrs, row_stride: int):
        arr = L._planes(*[C.cast(C.c_void_p(p), L._dp) for p in plane_ptrs])
        self._check(self._lib.hydro_gpu_download_async(self._ctx, arr, row_stride))

    def init_case(self, case: str, seed: int = 0):
        self._check(self._lib.hydro_gpu_init_case(self._ctx, CASES[case], seed))

    # -- stepping ---------------------------------------------------------
    def run(self, steps: int) -> float:
        last = C.c_double(0.0)
        self._check(self._lib.hydro_gpu_run(self._ctx, steps, C.byref(last)))
        return last.value

    def advance(self, dt: float):
        self._check(self._lib.hydro_gpu_advance(self._ctx, dt))

    def run_until(self, t_end: float) -> int:
        steps = C.c_int(0)
        self._check(self._lib.hydro_gpu_run_until(self._ctx, t_end, C.byref(steps)))
        return steps.value

    def compute_dt(self) -> float:
        dt = C.c_double(0.0)
        self._check(self._lib.hydro_gpu_compute_dt(self._ctx, C.byref(dt)))
        return dt.value

    def set_stream(self, stream_ptr: int | None):
        """Issue all work on this cudaStream_t (0 = the CUDA default stream);
        None restores the context's own stream."""
        if stream_ptr is None:
            self._check(self._lib.hydro_gpu_use_own_stream(self._ctx))
        else:
            self._check(self._lib.hydro_gpu_set_stream(self._ctx, C.c_void_p(stream_ptr)))

    def run_async(self, steps: int):
        self._check(self._lib.hydro_gpu_run_async(self._ctx, steps))

    def sync(self):
        self._check(self._lib.hydro_gpu_sync(self._ctx))

    # -- slab phases --------------------------------------------------------
    def slab_prologue(self, step: int = 0):
        self._check(self._lib.hydro_gpu_slab_prologue(self._ctx, step))

    def slab_sweep_x(self, step: int):
        self._check(self._lib.hydro_gpu_slab_sweep_x(self._ctx, step))

    def slab_sweep_y(self, step: int):
        self._check(self._lib.hydro_gpu_slab_sweep_y(self._ctx, step))

    def slab_finish(self):
        self._check(self._lib.hydro_gpu_slab_finish(self._ctx))

    def limit_slot(self, step: int) -> int:
        p = L._dp()
        self._check(self._lib.hydro_gpu_limit_slot(self._ctx, step, C.byref(p)))
        return C.cast(p, C.c_void_p).value

    def error_slot(self) -> int:
        p = C.POINTER(C.c_uint64)()
        self._check(self._lib.hydro_gpu_error_slot(self._ctx, C.byref(p)))
        return C.cast(p, C.c_void_p).value

    # peer-memory halo (include/hydro_gpu.h: hydro_gpu_inbox ...) -------------
    def inbox(self) -> tuple[int, int]:
        p = L._dp()
        count = C.c_size_t()
        self._check(self._lib.hydro_gpu_inbox(self._ctx, C.byref(p), C.byref(count)))
        return C.cast(p, C.c_void_p).value, count.value

    def inbox_ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(64)
        self._check(self._lib.hydro_gpu_inbox_ipc_handle(self._ctx, buf))
        return buf.raw

    def ipc_open(self, handle: bytes) -> int:
        buf = C.create_string_buffer(bytes(handle), 64)
        p = L._dp()
        self._check(self._lib.hydro_gpu_ipc_open(self._ctx, buf, C.byref(p)))
        return C.cast(p, C.c_void_p).value

    def set_halo_peers(self, upper: int | None, lower: int | None):
        self._check(self._lib.hydro_gpu_set_halo_peers(self._ctx, upper or None, lower or None))

    def slab_halo_pack(self):
        self._check(self._lib.hydro_gpu_slab_halo_pack(self._ctx))

    def slab_halo_unpack(self):
        self._check(self._lib.hydro_gpu_slab_halo_unpack(self._ctx))

    def compare(self, other: "GpuGrid") -> float:
        """compare_tolerance max_rel against another context of the same
        geometry (hydro_gpu_compare, on the device)."""
        out = C.c_double()
        self._check(self._lib.hydro_gpu_compare(self._ctx, other._ctx, C.byref(out)))
        return out.value

    def slab_halo_out(self, step: int):
        self._check(self._lib.hydro_gpu_slab_halo_out(self._ctx, step))

    def slab_inbox_in(self, step: int):
        self._check(self._lib.hydro_gpu_slab_inbox_in(self._ctx, step))

    def halo(self) -> dict:
        ptrs = [L._dp() for _ in range(4)]
        count = C.c_size_t()
        self._check(self._lib.hydro_gpu_halo(self._ctx, *[C.byref(p) for p in ptrs], C.byref(count)))
        names = ("send_lo", "send_hi", "recv_lo", "recv_hi")
        out = {n: C.cast(p, C.c_void_p).value for n, p in zip(names, ptrs)}
        out["count"] = count.value
        return out

    def raise_error_key(self, key: int):
        info = L.ErrorInfo()
        rc = self._lib.hydro_gpu_decode_error(self._ctx, key, C.byref(info))
        _raise_for(rc, info)

    # -- device-side audit -------------------------------------------------
    def row_audit(self) -> tuple[np.ndarray, np.ndarray]:
        """(row hashes, row sums), shape (4, nx) each, without downloading the grid."""
        h = np.zeros(4 * self.nx, dtype=np.uint64)
        s = np.zeros(4 * self.nx)
        self._check(self._lib.hydro_gpu_row_audit(self._ctx, h.ctypes.data_as(C.POINTER(C.c_uint64)),
                                                  s.ctypes.data_as(L._dp)))
        return h.reshape(4, self.nx), s.reshape(4, self.nx)

    def state_hash(self) -> int:
        out = C.c_uint64()
        self._check(self._lib.hydro_gpu_state_hash(self._ctx, C.byref(out)))
        return out.value

    def totals(self) -> np.ndarray:
        out = np.zeros(4)
        self._check(self._lib.hydro_gpu_totals(self._ctx, out.ctypes.data_as(L._dp)))
        return out

    # -- instrumentation ----------------------------------------------------
    def set_timing(self, on: bool):
        self._check(self._lib.hydro_gpu_set_timing(self._ctx, int(on)))

    def kernel_times(self) -> dict:
        ms = [C.c_double() for _ in range(3)]
        n = [C.c_longlong() for _ in range(3)]
        self._check(self._lib.hydro_gpu_kernel_times(self._ctx, *[C.byref(x) for x in ms],
                                                     *[C.byref(x) for x in n]))
        return {"ms_x": ms[0].value, "ms_y": ms[1].value, "ms_other": ms[2].value,
                "n_x": n[0].value, "n_y": n[1].value, "n_other": n[2].value}

    def skipped(self) -> tuple[int, int]:
        """Cell updates of the (column, row) sweeps since reset_counters() taken
        by the uniform-window identity (hydro_gpu_skipped)."""
        x, y = C.c_uint64(), C.c_uint64()
        self._check(self._lib.hydro_gpu_skipped(self._ctx, C.byref(x), C.byref(y)))
        return x.value, y.value

    def reset_counters(self):
        self._check(self._lib.hydro_gpu_reset_counters(self._ctx))

    def tune(self, seg_x: int = 0, seg_y: int = 0, block: int = 0):
        self._check(self._lib.hydro_gpu_tune(self._ctx, seg_x, seg_y, block))

    def tune_order(self, band_x: int = 0, band_y: int = 0):
        """hydro_gpu_tune_order: claim-order bands of the sweeps (0 = automatic)."""
        self._check(self._lib.hydro_gpu_tune_order(self._ctx, band_x, band_y))

    def set_math(self, math: str):
        """hydro_gpu_set_math: "bitwise" (default) or "tolerance"."""
        if math not in MATH:
            raise ConfigError(f"unknown math mode '{math}' (expected bitwise or tolerance)")
        self._check(self._lib.hydro_gpu_set_math(self._ctx, MATH[math]))
        self.math = math

    def set_schedule(self, schedule: str, seg: int = 0):
        """hydro_gpu_set_schedule: "fused" (one launch per step before the
        last, both sweeps), "split" (a column- and a row-sweep launch per
        step) or "auto" (default: fused where the last runs' updates were
        mostly uniform-window identities, split on dense flow); seg = rows
        per fused work item (0 = automatic).  Bitwise the same results."""
        if schedule not in SCHEDULE:
            raise ConfigError(f"unknown schedule '{schedule}' (expected split, fused or auto)")
        self._check(self._lib.hydro_gpu_set_schedule(self._ctx, SCHEDULE[schedule], seg))

    def schedule_choice(self) -> tuple[bool, float]:
        """hydro_gpu_schedule_choice: (the next run takes fused steps, the
        uniform-window share behind an automatic choice or -1)."""
        f, sh = C.c_int(), C.c_double()
        self._check(self._lib.hydro_gpu_schedule_choice(self._ctx, C.byref(f), C.byref(sh)))
        return bool(f.value), sh.value

    def fused_times(self) -> tuple[float, int]:
        """(device ms, count) of the fused steps timed with set_timing(True)."""
        ms = C.c_double()
        n = C.c_longlong()
        self._check(self._lib.hydro_gpu_fused_times(self._ctx, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    # multi-rank slabs driven from C++ (hydro_gpu_comm_attach) -----------------
    def comm_attach(self, unique_id: bytes, nranks: int, rank: int):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        self._check(self._lib.hydro_gpu_comm_attach(self._ctx, buf, nranks, rank))

    def comm_times(self) -> tuple[float, int]:
        """(device ms, count) of the per-step exchanges timed with set_timing(True)."""
        ms = C.c_double()
        n = C.c_longlong()
        self._check(self._lib.hydro_gpu_comm_times(self._ctx, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def col_offset(self) -> int:
        """Column offset of the device layout (state(); tiled in blocks of 32
        rows x 8 columns x 4 variables, include/hydro_gpu.h hydro_gpu_state)."""
        return int(self._lib.hydro_gpu_col_offset())

    def state(self) -> tuple[int, int]:
        p = L._dp()
        pitch = C.c_size_t()
        self._check(self._lib.hydro_gpu_state(self._ctx, C.byref(p), C.byref(pitch)))
        return C.cast(p, C.c_void_p).value, pitch.value


class GpuGroup:
    """One grid as row slabs over several devices, driven by this thread
    (hydro_gpu_group, include/hydro_gpu.h): peer-memory halo and an on-device
    dt min across slabs; bitwise equal to one GpuGrid on the whole grid.
    devices: one ordinal per slab (repeats allowed, e.g. [0, 0, 0])."""

    def __init__(self, nx: int, ny: int, dx: float, dy: float, model: GasModel = GasModel(),
                 bc: str = "reflect", devices=(0,), flux: str = "hllc"):
        if bc not in BC:
            raise ConfigError(f"unknown boundary '{bc}' (expected reflect or transmit)")
        if flux not in FLUX:
            raise ConfigError(f"unknown flux '{flux}' (expected hllc or exact10)")
        self.nx, self.ny, self.dx, self.dy = nx, ny, dx, dy
        cfg = L.Cfg(nx, ny, dx, dy, model.gamma, model.cfl, BC[bc], FLUX[flux], -1, 0, nx, 1, 1)
        n = len(devices)
        devs = (C.c_int * n)(*devices)
        self._lib = L.lib()
        self._g = C.c_void_p()
        rc = self._lib.hydro_gpu_group_create(C.byref(cfg), n, devs, C.byref(self._g))
        if rc:
            _raise_for(rc, message=f"hydro_gpu_group_create failed "
                                   f"({self._lib.hydro_gpu_status_string(rc).decode()}) "
                                   f"for {n} slabs of a {nx}x{ny} grid")

    def close(self):
        if self._g:
            self._lib.hydro_gpu_group_destroy(self._g)
            self._g = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, rc: int):
        if rc:
            info = L.ErrorInfo()
            self._lib.hydro_gpu_group_last_error(self._g, C.byref(info))
            _raise_for(rc, info)

    def slabs(self) -> list[tuple[int, int, int]]:
        """(row0, rows, device) per slab."""
        n = C.c_int(0)
        self._check(self._lib.hydro_gpu_group_slabs(self._g, C.byref(n), None, None, None))
        r0, rows, dev = (C.c_int * n.value)(), (C.c_int * n.value)(), (C.c_int * n.value)()
        self._check(self._lib.hydro_gpu_group_slabs(self._g, C.byref(n), r0, rows, dev))
        return list(zip(r0, rows, dev))

    def upload(self, planes: np.ndarray):
        self._check(self._lib.hydro_gpu_group_upload(self._g, L.planes_of(planes), planes.shape[2]))

    def download(self, planes: np.ndarray):
        self._check(self._lib.hydro_gpu_group_download(self._g, L.planes_of(planes),
                                                       planes.shape[2]))

    def init_case(self, case: str, seed: int = 0):
        self._check(self._lib.hydro_gpu_group_init_case(self._g, CASES[case], seed))

    def run(self, steps: int) -> float:
        last = C.c_double(0.0)
        self._check(self._lib.hydro_gpu_group_run(self._g, steps, C.byref(last)))
        return last.value


def _context_for(grid: Grid2D, model: GasModel, bc: str, flux: str = "hllc",
                 math: str = "bitwise") -> GpuGrid:
    g = GpuGrid(grid.nx, grid.ny, grid.dx, grid.dy, model, bc, flux=flux, math=math)
    g.upload(grid.planes)
    return g


def run_gpu(grid: Grid2D, model: GasModel = GasModel(), steps: int = 1, bc: str = "reflect",
            flux: str = "hllc", math: str = "bitwise") -> float:
    """run_sequential(grid, model, steps) on the GPU, in place; returns the last dt."""
    with _context_for(grid, model, bc, flux, math) as g:
        try:
            last = g.run(steps)
        finally:
            g.download(grid.planes)
    return last


def advance_gpu(grid: Grid2D, model: GasModel, dt: float, bc: str = "reflect") -> None:
    """advance_sequential(grid, model, dt) on the GPU, in place."""
    with _context_for(grid, model, bc) as g:
        try:
            g.advance(dt)
        finally:
            g.download(grid.planes)


def run_until_gpu(grid: Grid2D, model: GasModel, t_end: float, bc: str = "reflect",
                  flux: str = "hllc", math: str = "bitwise") -> int:
    """run_until(grid, model, t_end) on the GPU, in place; returns steps taken."""
    with _context_for(grid, model, bc, flux, math) as g:
        try:
            steps = g.run_until(t_end)
        finally:
            g.download(grid.planes)
    return steps


def compute_dt_gpu(grid: Grid2D, model: GasModel = GasModel()) -> float:
    """compute_dt(grid, model): cfl * min cell_dt_limit over the interior."""
    with _context_for(grid, model, "reflect") as g:
        return g.compute_dt()
