"""ctypes binding of libhydro_b200.so (the C-ABI declared in include/hydro_gpu.h).

The library is built in-tree by ``make -C paper_2106_13465_b200/csrc`` (or
``__graft_entry__.build()``).  There is no fallback: if the shared object is
missing or cannot be loaded, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
# HYDRO_B200_LIB selects an alternative build (tools/variants.sh); default in-tree.
LIB_PATH = os.environ.get("HYDRO_B200_LIB") or os.path.join(HERE, "libhydro_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "hydro_gpu.h")


class Cfg(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("dx", C.c_double), ("dy", C.c_double),
                ("gamma", C.c_double), ("cfl", C.c_double), ("bc", C.c_int), ("flux", C.c_int),
                ("device", C.c_int), ("row0", C.c_int), ("global_nx", C.c_int),
                ("wall_lo", C.c_int), ("wall_hi", C.c_int)]


class ErrorInfo(C.Structure):
    _fields_ = [("category", C.c_int), ("step", C.c_int), ("phase", C.c_int),
                ("strip", C.c_int), ("loop", C.c_int), ("cell", C.c_int), ("field", C.c_int),
                ("message", C.c_char * 256)]


_dp = C.POINTER(C.c_double)
_planes = _dp * 4
_ctx = C.c_void_p

_lib = None


def declared_symbols() -> list[str]:
    """Every function name include/hydro_gpu.h declares."""
    text = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(hydro_[a-z0-9_]+)\s*\(",
                                 text, re.M)))


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with "
                           "`make -C paper_2106_13465_b200/csrc` (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    i, d, u64, sz = C.c_int, C.c_double, C.c_uint64, C.c_size_t
    P = C.POINTER
    sig = {
        "hydro_gpu_abi_version": ([], i),
        "hydro_gpu_create": ([P(Cfg), P(_ctx)], i),
        "hydro_gpu_destroy": ([_ctx], i),
        "hydro_gpu_status_string": ([i], C.c_char_p),
        "hydro_gpu_last_error": ([_ctx, P(ErrorInfo)], i),
        "hydro_gpu_upload": ([_ctx, _planes, sz], i),
        "hydro_gpu_download": ([_ctx, _planes, sz], i),
        "hydro_gpu_upload_async": ([_ctx, _planes, sz], i),
        "hydro_gpu_download_async": ([_ctx, _planes, sz], i),
        "hydro_gpu_init_case": ([_ctx, i, u64], i),
        "hydro_gpu_run": ([_ctx, i, _dp], i),
        "hydro_gpu_advance": ([_ctx, d], i),
        "hydro_gpu_run_until": ([_ctx, d, P(i)], i),
        "hydro_gpu_compute_dt": ([_ctx, _dp], i),
        "hydro_gpu_set_stream": ([_ctx, C.c_void_p], i),
        "hydro_gpu_use_own_stream": ([_ctx], i),
        "hydro_gpu_run_async": ([_ctx, i], i),
        "hydro_gpu_sync": ([_ctx], i),
        "hydro_gpu_slab_prologue": ([_ctx, i], i),
        "hydro_gpu_limit_slot": ([_ctx, i, P(_dp)], i),
        "hydro_gpu_error_slot": ([_ctx, P(P(u64))], i),
        "hydro_gpu_halo": ([_ctx, P(_dp), P(_dp), P(_dp), P(_dp), P(sz)], i),
        "hydro_gpu_slab_sweep_x": ([_ctx, i], i),
        "hydro_gpu_slab_sweep_y": ([_ctx, i], i),
        "hydro_gpu_inbox": ([_ctx, P(_dp), P(sz)], i),
        "hydro_gpu_inbox_ipc_handle": ([_ctx, C.c_void_p], i),
        "hydro_gpu_ipc_open": ([_ctx, C.c_void_p, P(_dp)], i),
        "hydro_gpu_set_halo_peers": ([_ctx, C.c_void_p, C.c_void_p], i),
        "hydro_gpu_slab_halo_out": ([_ctx, i], i),
        "hydro_gpu_slab_inbox_in": ([_ctx, i], i),
        "hydro_gpu_slab_finish": ([_ctx], i),
        "hydro_gpu_slab_run_begin": ([_ctx, i, P(C.c_int)], i),
        "hydro_gpu_slab_step_xy": ([_ctx, i, i, i, i, i], i),
        "hydro_gpu_slab_run_end": ([_ctx, i], i),
        "hydro_gpu_decode_error": ([_ctx, u64, P(ErrorInfo)], i),
        "hydro_gpu_set_timing": ([_ctx, i], i),
        "hydro_gpu_kernel_times": ([_ctx, _dp, _dp, _dp, P(C.c_longlong), P(C.c_longlong),
                                    P(C.c_longlong)], i),
        "hydro_gpu_reset_counters": ([_ctx], i),
        "hydro_gpu_tune": ([_ctx, i, i, i], i),
        "hydro_gpu_tune_order": ([_ctx, i, i], i),
        "hydro_gpu_set_math": ([_ctx, i], i),
        "hydro_gpu_set_schedule": ([_ctx, i, i], i),
        "hydro_gpu_fused_times": ([_ctx, _dp, P(C.c_longlong)], i),
        "hydro_gpu_schedule_choice": ([_ctx, P(C.c_int), _dp], i),
        "hydro_gpu_state": ([_ctx, P(_dp), P(sz)], i),
        "hydro_gpu_col_offset": ([], i),
        "hydro_gpu_comm_unique_id": ([C.c_void_p], i),
        "hydro_gpu_comm_attach": ([_ctx, C.c_void_p, i, i], i),
        "hydro_gpu_comm_times": ([_ctx, _dp, P(C.c_longlong)], i),
        "hydro_gpu_skipped": ([_ctx, P(u64), P(u64)], i),
        "hydro_gpu_download_rows": ([_ctx, _planes, sz, i, i], i),
        "hydro_gpu_compare": ([_ctx, _ctx, _dp], i),
        "hydro_gpu_slab_halo_pack": ([_ctx], i),
        "hydro_gpu_slab_halo_unpack": ([_ctx], i),
        "hydro_gpu_math_selftest": ([i, _dp, _dp, _dp, _dp, P(i), sz], i),
        "hydro_grid_digest": ([_planes, sz, i, i], u64),
        "hydro_grid_state_hash": ([_planes, sz, i, i], u64),
        "hydro_fnv1a_rows": ([u64, _dp, sz, i, i], u64),
        "hydro_combine_row_hashes": ([P(u64), sz], u64),
        "hydro_pairwise_sum": ([_dp, sz], d),
        "hydro_gpu_row_audit": ([_ctx, P(u64), _dp], i),
        "hydro_gpu_state_hash": ([_ctx, P(u64)], i),
        "hydro_gpu_totals": ([_ctx, _dp], i),
        "hydro_init_case_host": ([i, i, i, d, u64, _planes, sz, _dp, _dp], i),
        "hydro_gpu_group_create": ([P(Cfg), i, P(i), P(_ctx)], i),
        "hydro_gpu_group_destroy": ([_ctx], i),
        "hydro_gpu_group_last_error": ([_ctx, P(ErrorInfo)], i),
        "hydro_gpu_group_slabs": ([_ctx, P(i), P(i), P(i), P(i)], i),
        "hydro_gpu_group_upload": ([_ctx, _planes, sz], i),
        "hydro_gpu_group_download": ([_ctx, _planes, sz], i),
        "hydro_gpu_group_init_case": ([_ctx, i, u64], i),
        "hydro_gpu_group_run": ([_ctx, i, _dp], i),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def planes_of(u) -> "C.Array":
    """4 plane pointers (address of cell (-1,-1)) of a (4, nx+4, ny+4) float64 array."""
    arr = _planes()
    for v in range(4):
        arr[v] = u[v].ctypes.data_as(_dp)
    return arr
