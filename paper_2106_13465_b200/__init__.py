"""B200-native HYDRO time step (arxiv 2106.13465 reference: hydro2d).

The hot path -- the directionally split MUSCL-Hancock/HLLC Godunov step -- runs
in hand-written sm_100a CUDA (csrc/, built into libhydro_b200.so) behind the
C-ABI in include/hydro_gpu.h.  This package is the host-side mirror of the
reference's stepping interface (hydro.py) and the multi-GPU slab driver
(slab.py).
"""
from .hydro import (  # noqa: F401
    BC, CASES, FLUX, MATH, ConfigError, DeviceError, ErrorCategory, GasModel, GpuGrid, GpuGroup, Grid2D, HydroError,
    PositivityError, ValidationError, advance_gpu, compute_dt_gpu, grid_digest, make_case, run_gpu,
    run_until_gpu,
)
