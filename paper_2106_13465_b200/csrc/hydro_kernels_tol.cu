// hydro_kernels_tol.cu -- the sweep kernels in tolerance math mode.
//
// The same source as hydro_kernels.cu, compiled with HB_TOLERANCE and FMA
// contraction (Makefile NUMERICS_TOL): quotients are a * (1/b) with the
// reciprocal refined once per denominator (no per-quotient correction, no
// range tests), and a*b+c may contract to one DFMA.  The result is no longer
// bitwise the reference's; tests/test_gpu_tolerance.py holds it to the
// north-star bound, compare_tolerance max_rel <= 1e-12 with scale
// max(|a|,|b|,1) (proj/src/audit.cpp:146), against the C oracle.  Every
// reference branch (positivity fallbacks, the HLLC equal-state shortcut, the
// error checks) is unchanged, and a work item whose fast pass meets a
// fallback or leaves the envelope is still redone through ExactMath.
#define HB_TOLERANCE 1
#include "hydro_kernels.cu"
