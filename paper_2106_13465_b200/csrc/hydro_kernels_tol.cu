// hydro_kernels_tol.cu -- the sweep kernels in tolerance math mode.
//
// The same source as hydro_kernels.cu, compiled with HB_TOLERANCE (and, like
// it, without contraction: Makefile NUMERICS_TOL): quotients are a * (1/b)
// with the reciprocal refined by one Newton step per denominator (no
// per-quotient correction, no range tests), square roots skip the final
// correction, and the exact-10 Newton loop stops at a 2^-26 step.  The dt
// speeds keep the bitwise arithmetic (hydro_physics.cuh dt_speed).  The result is no longer
// bitwise the reference's; tests/test_gpu_tolerance.py holds it to the
// north-star bound, compare_tolerance max_rel <= 1e-12 with scale
// max(|a|,|b|,1) (proj/src/audit.cpp:146), against the C oracle.  Every
// reference branch (positivity fallbacks, the HLLC equal-state shortcut, the
// error checks) is unchanged, and a work item whose fast pass meets a
// fallback or leaves the envelope is still redone through ExactMath.
#define HB_TOLERANCE 1
#include "hydro_kernels.cu"
