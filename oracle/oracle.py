"""ctypes front-end to the CPU checker -- TEST INFRASTRUCTURE ONLY.

Loaded only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs.  Two libraries:

* ``liboracle.so``: the plain-C restatement of the reference step
  (hydro_oracle.c), always built by ``oracle/Makefile``;
* ``_ref/libhydro_ref.so``: the unmodified reference library compiled from
  /root/reference sources plus ref_shim.cpp (present when the reference was
  available at build time; prebuilt files travel to the GPU box).

Grids are numpy float64 arrays of shape (4, nx+4, ny+4): the Grid2D plane
layout of proj/include/hydro/grid.hpp:15-19,54-57.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhydro_ref.so")

CASES = {"uniform": 0, "blast": 1, "sod": 2, "corner_blast": 3, "sod_x": 4, "random": 5}
BCS = {"reflect": 0, "transmit": 1}
STRATEGIES = {"sequential": 0, "fine_grain": 1, "coarse_grain": 2, "task_graph": 3}
WALL_XLO, WALL_XHI, WALL_Y, WALL_ALL = 1, 2, 4, 7

_dp = C.POINTER(C.c_double)


class OracleError(C.Structure):
    _fields_ = [("category", C.c_int), ("step", C.c_int), ("phase", C.c_int),
                ("strip", C.c_int), ("loop", C.c_int), ("cell", C.c_int),
                ("field", C.c_int), ("message", C.c_char * 256)]


class CheckerError(RuntimeError):
    def __init__(self, category: int, message: str, info=None):
        super().__init__(message)
        self.category = category
        self.info = info


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = C.CDLL(ORACLE_SO)
        i, d, u64 = C.c_int, C.c_double, C.c_uint64
        perr = C.POINTER(OracleError)
        L.oracle_init_case.argtypes = [_dp, i, i, i, d, u64, _dp, _dp, perr]
        L.oracle_init_random_rows.argtypes = [_dp, i, i, i, i, d, u64, perr]
        L.oracle_apply_boundary.argtypes = [_dp, i, i, i, i]
        L.oracle_apply_boundary.restype = None
        L.oracle_compute_limit.argtypes = [_dp, i, i, d, d, d, _dp, perr]
        L.oracle_sweep_axis.argtypes = [_dp, i, i, d, d, d, i, d, perr]
        L.oracle_run_sequential.argtypes = [_dp, i, i, d, d, d, d, i, i, _dp, perr]
        L.oracle_advance.argtypes = [_dp, i, i, d, d, d, i, d, perr]
        L.oracle_run_until.argtypes = [_dp, i, i, d, d, d, d, i, d, C.POINTER(C.c_int), perr]
        L.oracle_sweep_strip.argtypes = [_dp, i, d, d, d, _dp, _dp, perr]
        L.oracle_riemann_flux.argtypes = [_dp, _dp, d, _dp, perr]
        L.oracle_digest.argtypes = [_dp, i, i]
        L.oracle_digest.restype = u64
        L.oracle_sums.argtypes = [_dp, i, i, _dp]
        L.oracle_sums.restype = None
        L.oracle_compare_tolerance.argtypes = [_dp, _dp, i, i, _dp, _dp]
        L.oracle_compare_tolerance.restype = None
        L.oracle_set_flux.argtypes = [i]
        L.oracle_set_flux.restype = None
        L.oracle_set_threads.argtypes = [i]
        L.oracle_set_threads.restype = None
        L.oracle_exact10_flux.argtypes = [_dp, _dp, d, _dp]
        L.oracle_splitmix64.argtypes = [u64]
        L.oracle_splitmix64.restype = u64
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"{REF_SO} missing: run `make -C oracle ref` "
                               "where /root/reference exists")
        R = C.CDLL(REF_SO)
        i, d, u64 = C.c_int, C.c_double, C.c_uint64
        R.ref_run.argtypes = [_dp, i, i, d, d, d, d, i, i, i, i, _dp, C.c_char_p, i]
        R.ref_run_windows.argtypes = [_dp, i, i, d, d, d, d, i, i, C.POINTER(C.c_int), i, i,
                                      _dp, C.c_char_p, i]
        R.ref_advance.argtypes = [_dp, i, i, d, d, d, i, d, C.c_char_p, i]
        R.ref_run_until.argtypes = [_dp, i, i, d, d, d, d, i, d, C.POINTER(C.c_int), C.c_char_p, i]
        R.ref_compute_dt.argtypes = [_dp, i, i, d, d, d, d]
        R.ref_compute_dt.restype = d
        R.ref_make_case.argtypes = [i, i, i, d, d, _dp, _dp, _dp]
        R.ref_digest.argtypes = [_dp, i, i]
        R.ref_digest.restype = u64
        R.ref_checksum_line.argtypes = [_dp, i, i, C.c_char_p, i]
        R.ref_sweep_strip.argtypes = [_dp, i, d, d, d, _dp, _dp, C.c_char_p, i]
        R.ref_riemann_flux.argtypes = [_dp, _dp, d, _dp]
        R.ref_hardware_concurrency.restype = i
        R.ref_exact_flux.argtypes = [_dp, _dp, d, _dp]
        _ref = R
    return _ref


@dataclass
class Grid:
    """Grid2D twin: u has shape (4, nx+4, ny+4)."""
    nx: int
    ny: int
    dx: float
    dy: float
    u: np.ndarray

    def copy(self) -> "Grid":
        return Grid(self.nx, self.ny, self.dx, self.dy, self.u.copy())

    def interior(self) -> np.ndarray:
        return self.u[:, 2:self.nx + 2, 2:self.ny + 2]


def _raise(rc: int, err: OracleError):
    if rc != 0:
        raise CheckerError(rc, err.message.decode(), {
            "step": err.step, "phase": err.phase, "strip": err.strip,
            "loop": err.loop, "cell": err.cell, "field": err.field})


def make_case(case: str, nx: int, ny: int, gamma: float = 1.4, seed: int = 0) -> Grid:
    u = np.zeros((4, nx + 4, ny + 4))
    dx, dy = C.c_double(), C.c_double()
    err = OracleError()
    rc = lib().oracle_init_case(_ptr(u), nx, ny, CASES[case], gamma, seed,
                                C.byref(dx), C.byref(dy), C.byref(err))
    _raise(rc, err)
    return Grid(nx, ny, dx.value, dy.value, u)


def run_sequential(g: Grid, steps: int, bc: str = "reflect", gamma=1.4, cfl=0.8) -> float:
    err = OracleError()
    last = C.c_double(0.0)
    rc = lib().oracle_run_sequential(_ptr(g.u), g.nx, g.ny, g.dx, g.dy, gamma, cfl,
                                     BCS[bc], steps, C.byref(last), C.byref(err))
    _raise(rc, err)
    return last.value


def advance(g: Grid, dt: float, bc: str = "reflect", gamma=1.4) -> None:
    err = OracleError()
    rc = lib().oracle_advance(_ptr(g.u), g.nx, g.ny, g.dx, g.dy, gamma, BCS[bc], dt,
                              C.byref(err))
    _raise(rc, err)


def run_until(g: Grid, t_end: float, bc: str = "reflect", gamma=1.4, cfl=0.8) -> int:
    err = OracleError()
    steps = C.c_int(0)
    rc = lib().oracle_run_until(_ptr(g.u), g.nx, g.ny, g.dx, g.dy, gamma, cfl, BCS[bc],
                                t_end, C.byref(steps), C.byref(err))
    _raise(rc, err)
    return steps.value


def apply_boundary(g: Grid, bc: str = "reflect", walls: int = WALL_ALL) -> None:
    lib().oracle_apply_boundary(_ptr(g.u), g.nx, g.ny, BCS[bc], walls)


def compute_limit(g: Grid, gamma=1.4) -> float:
    err = OracleError()
    lim = C.c_double()
    rc = lib().oracle_compute_limit(_ptr(g.u), g.nx, g.ny, g.dx, g.dy, gamma,
                                    C.byref(lim), C.byref(err))
    _raise(rc, err)
    return lim.value


def sweep_axis(g: Grid, axis: int, dt: float, gamma=1.4) -> None:
    err = OracleError()
    rc = lib().oracle_sweep_axis(_ptr(g.u), g.nx, g.ny, g.dx, g.dy, gamma, axis, dt,
                                 C.byref(err))
    _raise(rc, err)


def sweep_strip(cells: np.ndarray, n: int, dx: float, dt: float, gamma=1.4):
    err = OracleError()
    first = np.zeros(4)
    last = np.zeros(4)
    rc = lib().oracle_sweep_strip(_ptr(cells), n, dx, dt, gamma, _ptr(first), _ptr(last),
                                  C.byref(err))
    _raise(rc, err)
    return first, last


def riemann_flux(wl, wr, gamma=1.4) -> np.ndarray:
    a = np.ascontiguousarray(wl, dtype=np.float64)
    b = np.ascontiguousarray(wr, dtype=np.float64)
    f = np.zeros(4)
    err = OracleError()
    rc = lib().oracle_riemann_flux(_ptr(a), _ptr(b), gamma, _ptr(f), C.byref(err))
    _raise(rc, err)
    return f


FLUXES = {"hllc": 0, "exact10": 1}


def set_flux(flux: str) -> None:
    """Interface flux of every oracle sweep: "hllc" (the reference hot path) or
    "exact10" (exact Riemann solver, 10 Newton iterations)."""
    lib().oracle_set_flux(FLUXES[flux])


class flux_mode:
    """Context manager: run oracle calls with the given flux, restore HLLC."""

    def __init__(self, flux: str):
        self.flux = flux

    def __enter__(self):
        set_flux(self.flux)

    def __exit__(self, *exc):
        set_flux("hllc")


def set_threads(n: int) -> None:
    """Strip-parallel sweeps (long golden runs; results equal one thread's)."""
    lib().oracle_set_threads(n)


def exact10_flux(wl, wr, gamma=1.4) -> np.ndarray:
    a = np.ascontiguousarray(wl, dtype=np.float64)
    b = np.ascontiguousarray(wr, dtype=np.float64)
    f = np.zeros(4)
    rc = lib().oracle_exact10_flux(_ptr(a), _ptr(b), gamma, _ptr(f))
    if rc:
        raise CheckerError(rc, "vacuum-generating Riemann states are out of scope")
    return f


def digest(g: Grid) -> int:
    return int(lib().oracle_digest(_ptr(g.u), g.nx, g.ny))


def sums(g: Grid) -> np.ndarray:
    s = np.zeros(4)
    lib().oracle_sums(_ptr(g.u), g.nx, g.ny, _ptr(s))
    return s


def compare_tolerance(a: Grid, b: Grid):
    mx, l1 = C.c_double(), C.c_double()
    lib().oracle_compare_tolerance(_ptr(a.u), _ptr(b.u), a.nx, a.ny, C.byref(mx), C.byref(l1))
    return mx.value, l1.value


# ---- the compiled reference -------------------------------------------------

def ref_make_case(case: str, nx: int, ny: int, gamma=1.4, cfl=0.8) -> Grid:
    ids = {"uniform": 0, "blast": 1, "sod": 2}
    dx, dy = C.c_double(), C.c_double()
    if case == "sod":
        nx = 4
    u = np.zeros((4, nx + 4, ny + 4))
    rc = ref().ref_make_case(ids[case], nx, ny, gamma, cfl, _ptr(u), C.byref(dx), C.byref(dy))
    if rc:
        raise CheckerError(rc, "ref_make_case failed")
    return Grid(nx, ny, dx.value, dy.value, u)


def ref_run(g: Grid, steps: int, bc="reflect", strategy="sequential", workers=1,
            gamma=1.4, cfl=0.8) -> float:
    secs = C.c_double(0.0)
    msg = C.create_string_buffer(512)
    rc = ref().ref_run(_ptr(g.u), g.nx, g.ny, g.dx, g.dy, gamma, cfl, BCS[bc], steps,
                       STRATEGIES[strategy], workers, C.byref(secs), msg, 512)
    if rc:
        raise CheckerError(rc, msg.value.decode())
    return secs.value


def ref_run_windows(g: Grid, steps_per, bc="reflect", strategy="sequential", workers=1,
                    gamma=1.4, cfl=0.8) -> list:
    """ref_run over consecutive windows of one flow (grid loaded once);
    returns the stepping seconds of each window."""
    n = len(steps_per)
    arr = (C.c_int * n)(*steps_per)
    secs = (C.c_double * n)()
    msg = C.create_string_buffer(512)
    rc = ref().ref_run_windows(_ptr(g.u), g.nx, g.ny, g.dx, g.dy, gamma, cfl, BCS[bc], n, arr,
                               STRATEGIES[strategy], workers, secs, msg, 512)
    if rc:
        raise CheckerError(rc, msg.value.decode())
    return list(secs)


def ref_advance(g: Grid, dt: float, bc="reflect", gamma=1.4) -> None:
    msg = C.create_string_buffer(512)
    rc = ref().ref_advance(_ptr(g.u), g.nx, g.ny, g.dx, g.dy, gamma, BCS[bc], dt, msg, 512)
    if rc:
        raise CheckerError(rc, msg.value.decode())


def ref_run_until(g: Grid, t_end: float, bc="reflect", gamma=1.4, cfl=0.8) -> int:
    msg = C.create_string_buffer(512)
    steps = C.c_int(0)
    rc = ref().ref_run_until(_ptr(g.u), g.nx, g.ny, g.dx, g.dy, gamma, cfl, BCS[bc], t_end,
                             C.byref(steps), msg, 512)
    if rc:
        raise CheckerError(rc, msg.value.decode())
    return steps.value


def ref_digest(g: Grid) -> int:
    return int(ref().ref_digest(_ptr(g.u), g.nx, g.ny))


def ref_checksum_line(g: Grid) -> str:
    out = C.create_string_buffer(256)
    ref().ref_checksum_line(_ptr(g.u), g.nx, g.ny, out, 256)
    return out.value.decode()


def ref_sweep_strip(cells: np.ndarray, n: int, dx: float, dt: float, gamma=1.4):
    first = np.zeros(4)
    last = np.zeros(4)
    msg = C.create_string_buffer(512)
    rc = ref().ref_sweep_strip(_ptr(cells), n, dx, dt, gamma, _ptr(first), _ptr(last), msg, 512)
    if rc:
        raise CheckerError(rc, msg.value.decode())
    return first, last


def ref_exact_flux(wl, wr, gamma=1.4):
    """(flux, newton iterations) of the reference's exact solver at x/t = 0."""
    a = np.ascontiguousarray(wl, dtype=np.float64)
    b = np.ascontiguousarray(wr, dtype=np.float64)
    f = np.zeros(4)
    rc = ref().ref_exact_flux(_ptr(a), _ptr(b), gamma, _ptr(f))
    if rc >= 100:
        raise CheckerError(rc - 100, "reference exact solver error")
    return f, rc


def ref_riemann_flux(wl, wr, gamma=1.4) -> np.ndarray:
    a = np.ascontiguousarray(wl, dtype=np.float64)
    b = np.ascontiguousarray(wr, dtype=np.float64)
    f = np.zeros(4)
    rc = ref().ref_riemann_flux(_ptr(a), _ptr(b), gamma, _ptr(f))
    if rc:
        raise CheckerError(rc, "riemann positivity")
    return f
