// hydro_kernels.cu -- the fused sweep kernels of the HYDRO step (sm_100a).
//
// One step of the reference (proj/src/schedulers.cpp:103-116) is
//   apply_boundary -> compute_dt -> column sweep -> apply_boundary -> row sweep.
// Here it is two launches per step:
//   sweep_x  (Column axis, strips along i): reads U_a, writes U_b, and writes
//            the j-ghost columns of U_b (the y-wall half of the second
//            apply_boundary, grid.cpp:44-59) from its own outputs;
//   sweep_y  (Row axis, strips along j): reads U_b, writes U_a, writes the
//            i-ghost rows of U_a for the next step (the x-wall half of
//            apply_boundary, grid.cpp:26-42), and folds cell_dt_limit of the
//            new state into the next step's dt (compute_dt, :233-242).
// Every thread owns one strip segment and walks it with a register sliding
// window: primitive conversion, minmod slopes, Hancock predictor, evolved
// faces, HLLC flux and the conservative update of the reference's four strip
// loops (euler_kernel.cpp:111-223) are fused, no per-strip scratch touches
// HBM.  Segments overlap by the 2-cell stencil halo only.
#include <cuda_runtime.h>

#include "hydro_kernels.cuh"

namespace hb {

namespace {

constexpr unsigned long long kEmptyLimit = ~0ull;  // sentinel above every positive double

__device__ __forceinline__ void record(unsigned long long* err, unsigned long long key) {
  atomicMin(err, key);
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = (w < v) ? w : v;
  }
  return v;
}

// Walks strip cells [ka, kb] (local strip coordinates: cell k holds grid
// index k-1).  load(k) returns the conserved state of cell k in sweep
// orientation; sink(k, u, rr) receives the updated cell and 1/rho.
// kg converts a local strip cell to the global one used in error keys.
template <class Load, class Sink>
__device__ __forceinline__ void walk_strip(int ka, int kb, const Load& load, Sink& sink,
                                           const Gas& g, double dtdx, unsigned long long* err,
                                           unsigned long long key_base, int kg) {
  const double half = 0.5 * dtdx;
  Recip rr;
  Prim wA, wB, wC;
  Cons uA, uB, uC;
  int f;
  uA = load(ka - 2);
  if ((f = to_prim(uA, g, wA, rr)) >= 0)
    record(err, key_base | ((unsigned long long)(ka - 2 + kg) << 2) | (unsigned)f);
  uB = load(ka - 1);
  if ((f = to_prim(uB, g, wB, rr)) >= 0)
    record(err, key_base | ((unsigned long long)(ka - 1 + kg) << 2) | (unsigned)f);
  Face frPrev;
  Flux fluxPrev;
#pragma unroll 1
  for (int c = ka - 1; c <= kb + 1; ++c) {
    uC = load(c + 1);
    if ((f = to_prim(uC, g, wC, rr)) >= 0)
      record(err, key_base | ((unsigned long long)(c + 1 + kg) << 2) | (unsigned)f);
    Face fl, fr;
    predict_faces(wA, wB, wC, half, g, fl, fr);
    if (c >= ka) {
      const Flux F = hllc(frPrev, fl, g);
      if (c > ka) {
        Cons u = uA;
        Recip rn;
        if ((f = update_cell(u, fluxPrev, F, dtdx, rn)) >= 0)
          record(err, key_base | (1ull << 20) |
                          ((unsigned long long)(c - 1 + kg) << 2) | (unsigned)f);
        sink(c - 1, u, rn);
      }
      fluxPrev = F;
    }
    frPrev = fr;
    wA = wB;
    wB = wC;
    uA = uB;
    uB = uC;
  }
}

__device__ __forceinline__ bool latched(const SweepArgs& a) {
  return *(volatile unsigned long long*)a.err != kNoError;
}

__device__ __forceinline__ double step_dt(const SweepArgs& a) {
  return a.explicit_dt ? a.dt_value : a.cfl * __longlong_as_double((long long)*a.limit_in);
}

// ---------------------------------------------------------------------------
// Column sweep: thread = column j, segment of rows.  Loads of one row by a
// warp are 32 consecutive doubles per variable (coalesced).
__global__ void __launch_bounds__(128) sweep_x_kernel(SweepArgs a) {
  const int j = 1 + blockIdx.x * blockDim.x + threadIdx.x;
  if (j > a.ny) return;
  if (latched(a)) return;
  if (*(volatile unsigned long long*)a.dt_err != kNoError) {
    // compute_dt of this step failed (detected by the previous row sweep).
    record(a.err, *(volatile unsigned long long*)a.dt_err);
    return;
  }
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && a.limit_out)
    *a.limit_out = kEmptyLimit;
  const Gas g = make_gas(a.gamma);
  const double dt = step_dt(a);
  const double dtdx = dt / a.dx;
  const int i_lo = 1 + blockIdx.y * a.seg;
  const int i_hi = min(a.nx, i_lo + a.seg - 1);
  const double* __restrict__ src = a.src;
  double* __restrict__ dst = a.dst;
  const size_t pitch = a.pitch;
  auto load = [&](int k) -> Cons {
    const int i = k - 1;
    return {__ldg(src + cell_index(pitch, 0, i, j)), __ldg(src + cell_index(pitch, 1, i, j)),
            __ldg(src + cell_index(pitch, 2, i, j)), __ldg(src + cell_index(pitch, 3, i, j))};
  };
  const int ny = a.ny;
  const bool refl = a.bc == 0;
  auto put = [&](int i, int jj, const Cons& u, bool neg) {
    dst[cell_index(pitch, 0, i, jj)] = u.r;
    dst[cell_index(pitch, 1, i, jj)] = u.ma;
    dst[cell_index(pitch, 2, i, jj)] = neg ? -u.mb : u.mb;
    dst[cell_index(pitch, 3, i, jj)] = u.e;
  };
  auto sink = [&](int k, const Cons& u, const Recip&) {
    const int i = k - 1;
    put(i, j, u, false);
    // y-wall ghosts of the column-sweep output (grid.cpp:44-59).
    if (refl) {
      if (j <= 2) put(i, 1 - j, u, true);
      if (j >= ny - 1) put(i, 2 * ny + 1 - j, u, true);
    } else {
      if (j == 1) { put(i, 0, u, false); put(i, -1, u, false); }
      if (j == ny) { put(i, ny + 1, u, false); put(i, ny + 2, u, false); }
    }
  };
  const unsigned long long base = error_key(a.step, 1, j, 0, 0, 0);
  walk_strip(i_lo + 1, i_hi + 1, load, sink, g, dtdx, a.err, base, a.row0);
}

// ---------------------------------------------------------------------------
// Row sweep: thread = row i, segment of columns.  Also produces the next
// step's dt limit and the i-wall ghost rows.
__global__ void __launch_bounds__(128) sweep_y_kernel(SweepArgs a) {
  const int i = 1 + blockIdx.x * blockDim.x + threadIdx.x;
  if (latched(a)) return;
  const bool active = i <= a.nx;
  const Gas g = make_gas(a.gamma);
  const double dt = step_dt(a);
  const double dtdx = dt / a.dx;
  const int j_lo = 1 + blockIdx.y * a.seg;
  const int j_hi = min(a.ny, j_lo + a.seg - 1);
  const double* __restrict__ src = a.src;
  double* __restrict__ dst = a.dst;
  const size_t pitch = a.pitch;
  const int nx = a.nx;
  const bool refl = a.bc == 0;
  const bool mirror_lo = a.wall_lo && i <= 2;
  const bool mirror_hi = a.wall_hi && i >= nx - 1;
  double lim_min = __longlong_as_double(0x7ff0000000000000ll);
  unsigned long long dt_key = kNoError;
  auto load = [&](int k) -> Cons {
    const int j = k - 1;
    return {__ldg(src + cell_index(pitch, 0, i, j)), __ldg(src + cell_index(pitch, 2, i, j)),
            __ldg(src + cell_index(pitch, 1, i, j)), __ldg(src + cell_index(pitch, 3, i, j))};
  };
  auto put = [&](int ii, int j, const Cons& u, bool neg) {
    dst[cell_index(pitch, 0, ii, j)] = u.r;
    dst[cell_index(pitch, 2, ii, j)] = u.ma;
    dst[cell_index(pitch, 1, ii, j)] = neg ? -u.mb : u.mb;
    dst[cell_index(pitch, 3, ii, j)] = u.e;
  };
  const int gi = a.row0 + i;
  auto sink = [&](int k, const Cons& u, const Recip& rn) {
    const int j = k - 1;
    put(i, j, u, false);
    if (mirror_lo) {  // x-wall ghosts for the next column sweep (grid.cpp:26-42)
      if (refl) put(1 - i, j, u, true);
      else if (i == 1) { put(0, j, u, false); put(-1, j, u, false); }
    }
    if (mirror_hi) {
      if (refl) put(2 * nx + 1 - i, j, u, true);
      else if (i == nx) { put(nx + 1, j, u, false); put(nx + 2, j, u, false); }
    }
    if (a.want_limit) {
      double lim;
      const int f = dt_limit(u, rn, a.spacing, g, lim);
      if (f >= 0) {
        const unsigned long long key = error_key(a.step + 1, 0, gi, 0, j, f);
        dt_key = key < dt_key ? key : dt_key;
      } else {
        lim_min = smin(lim_min, lim);
      }
    }
  };
  if (active) {
    const unsigned long long base = error_key(a.step, 2, gi, 0, 0, 0);
    walk_strip(j_lo + 1, j_hi + 1, load, sink, g, dtdx, a.err, base, 0);
  }
  if (a.want_limit) {
    const unsigned long long m = warp_min_u64((unsigned long long)__double_as_longlong(lim_min));
    const unsigned long long e = warp_min_u64(dt_key);
    if ((threadIdx.x & 31) == 0) {
      atomicMin(a.limit_out, m);
      if (e != kNoError) atomicMin(a.dt_err, e);
    }
  }
}

// ---------------------------------------------------------------------------
// Start-of-run pass: apply_boundary on the physical walls of the current
// state and compute_dt's min-reduction for the first step.
__global__ void __launch_bounds__(256) prologue_kernel(PrologueArgs a) {
  const int j = 1 + blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = j <= a.ny;
  const size_t pitch = a.pitch;
  double* u = a.u;
  const bool refl = a.bc == 0;
  const Gas g = make_gas(a.gamma);
  double lim = __longlong_as_double(0x7ff0000000000000ll);
  unsigned long long key = kNoError;
  const int nx = a.nx, ny = a.ny;
  for (int i = 1 + blockIdx.y; active && i <= nx; i += gridDim.y) {
    Cons c = {u[cell_index(pitch, 0, i, j)], u[cell_index(pitch, 1, i, j)],
              u[cell_index(pitch, 2, i, j)], u[cell_index(pitch, 3, i, j)]};
    auto put = [&](int ii, int jj, int negv) {
      u[cell_index(pitch, 0, ii, jj)] = c.r;
      u[cell_index(pitch, 1, ii, jj)] = negv == 1 ? -c.ma : c.ma;
      u[cell_index(pitch, 2, ii, jj)] = negv == 2 ? -c.mb : c.mb;
      u[cell_index(pitch, 3, ii, jj)] = c.e;
    };
    if (a.wall_lo && i <= 2) {
      if (refl) put(1 - i, j, 1);
      else if (i == 1) { put(0, j, 0); put(-1, j, 0); }
    }
    if (a.wall_hi && i >= nx - 1) {
      if (refl) put(2 * nx + 1 - i, j, 1);
      else if (i == nx) { put(nx + 1, j, 0); put(nx + 2, j, 0); }
    }
    if (a.full_bc) {
      if (refl) {
        if (j <= 2) put(i, 1 - j, 2);
        if (j >= ny - 1) put(i, 2 * ny + 1 - j, 2);
      } else {
        if (j == 1) { put(i, 0, 0); put(i, -1, 0); }
        if (j == ny) { put(i, ny + 1, 0); put(i, ny + 2, 0); }
      }
    }
    if (a.want_limit) {
      const Recip rr = make_recip(c.r);
      double l;
      const int f = dt_limit(c, rr, a.spacing, g, l);
      if (f >= 0) {
        const unsigned long long k = error_key(a.step, 0, a.row0 + i, 0, j, f);
        key = k < key ? k : key;
      } else {
        lim = smin(lim, l);
      }
    }
  }
  if (a.want_limit) {
    const unsigned long long m = warp_min_u64((unsigned long long)__double_as_longlong(lim));
    const unsigned long long e = warp_min_u64(key);
    if ((threadIdx.x & 31) == 0) {
      atomicMin(a.limit_out, m);
      if (e != kNoError) atomicMin(a.err, e);
    }
  }
}

// End-of-run ghosts: the reference's last apply_boundary ran on the column
// sweep output, so every ghost band mirrors U_b (grid.cpp:23-60).
__global__ void finish_kernel(FinishArgs a) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const size_t pitch = a.pitch;
  const bool refl = a.bc == 0;
  if (t < a.ny) {  // i-wall ghost rows from U_b interior rows
    const int j = t + 1;
    for (int layer = 1; layer <= 2; ++layer) {
      const int srcs[2] = {refl ? layer : 1, refl ? a.nx + 1 - layer : a.nx};
      const int gh[2] = {1 - layer, a.nx + layer};
      const int on[2] = {a.wall_lo, a.wall_hi};
      for (int s = 0; s < 2; ++s) {
        if (!on[s]) continue;
        for (int v = 0; v < 4; ++v) {
          const double x = a.post_x[cell_index(pitch, v, srcs[s], j)];
          a.u[cell_index(pitch, v, gh[s], j)] = (refl && v == 1) ? -x : x;
        }
      }
    }
  } else if (t < a.ny + a.nx) {  // j-wall ghost columns, already mirrored in U_b
    const int i = t - a.ny + 1;
    const int cols[4] = {-1, 0, a.ny + 1, a.ny + 2};
    for (int c = 0; c < 4; ++c)
      for (int v = 0; v < 4; ++v)
        a.u[cell_index(pitch, v, i, cols[c])] = a.post_x[cell_index(pitch, v, i, cols[c])];
  }
}

// ---------------------------------------------------------------------------
// Case initialisers (cases.cpp:11-69 and the BASELINE configs), bitwise equal
// to the host versions in hydro_host.cpp.
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double rnd_sym(unsigned long long seed, unsigned long long cell,
                                          int var) {
  const unsigned long long h = splitmix64(seed ^ (4ull * cell + (unsigned long long)var));
  const double unit = (double)(h >> 11) * 0x1.0p-53;
  return 2.0 * unit - 1.0;
}

__global__ void init_kernel(InitArgs a) {
  const int j = 1 + blockIdx.x * blockDim.x + threadIdx.x;
  if (j > a.ny) return;
  for (int i = 1 + blockIdx.y; i <= a.nx; i += gridDim.y) {
  const int gi = a.row0 + i;
  Prim w = {1.0, 0.0, 0.0, 1.0};
  switch (a.case_id) {
    case 1: w.p = 1e-5 * (a.gamma - 1.0); break;
    case 3: w.p = 1e-5; break;
    case 2:
      if (!(j <= a.ny / 2)) w = {0.125, 0.0, 0.0, 0.1};
      break;
    case 4:
      if (!(gi <= a.global_nx / 2)) w = {0.125, 0.0, 0.0, 0.1};
      break;
    case 5: {
      const unsigned long long cell =
          (unsigned long long)(gi - 1) * (unsigned long long)a.ny + (unsigned long long)(j - 1);
      w.r = 1.0 + 0.1 * rnd_sym(a.seed, cell, 0);
      w.p = 1.0 + 0.1 * rnd_sym(a.seed, cell, 1);
      w.va = 0.1 * rnd_sym(a.seed, cell, 2);
      w.vb = 0.1 * rnd_sym(a.seed, cell, 3);
      break;
    }
    default: break;
  }
  // prim_to_cons (euler_kernel.cpp:22-28)
  double e = w.p / (a.gamma - 1.0) + 0.5 * w.r * (w.va * w.va + w.vb * w.vb);
  if (a.case_id == 3 && gi == 1 && j == 1) e = 1.0 / (a.dx * a.dy);
  if (a.case_id == 1) {
    const int gnx = a.global_nx, ny = a.ny;
    const bool ci = (gnx % 2) ? (gi == (gnx + 1) / 2) : (gi == gnx / 2 || gi == gnx / 2 + 1);
    const bool cj = (ny % 2) ? (j == (ny + 1) / 2) : (j == ny / 2 || j == ny / 2 + 1);
    if (ci && cj) {
      const double share = 1.0 / ((double)((gnx % 2) ? 1 : 2) * (double)((ny % 2) ? 1 : 2));
      e = share / (a.dx * a.dy);
    }
  }
  const size_t p = a.pitch;
  a.u[cell_index(p, 0, i, j)] = w.r;
  a.u[cell_index(p, 1, i, j)] = w.r * w.va;
  a.u[cell_index(p, 2, i, j)] = w.r * w.vb;
  a.u[cell_index(p, 3, i, j)] = e;
  }
}

int segments(int n, int strips, int want_seg) {
  if (want_seg > 0) return (n + want_seg - 1) / want_seg;
  // Enough threads for ~2 waves of 148 SMs x 16 warps, segments >= 24 cells.
  const long long target = 148LL * 512 * 2;
  long long nseg = (target + strips - 1) / strips;
  const long long max_seg = (n + 23) / 24;
  if (nseg > max_seg) nseg = max_seg;
  if (nseg < 1) nseg = 1;
  return (int)nseg;
}

}  // namespace

void launch_sweep_x(const SweepArgs& a0, int block, cudaStream_t s) {
  SweepArgs a = a0;
  const int nseg = segments(a.nx, a.ny, a.seg);
  a.seg = (a.nx + nseg - 1) / nseg;
  dim3 grid((a.ny + block - 1) / block, nseg);
  sweep_x_kernel<<<grid, block, 0, s>>>(a);
}

void launch_sweep_y(const SweepArgs& a0, int block, cudaStream_t s) {
  SweepArgs a = a0;
  const int nseg = segments(a.ny, a.nx, a.seg);
  a.seg = (a.ny + nseg - 1) / nseg;
  dim3 grid((a.nx + block - 1) / block, nseg);
  sweep_y_kernel<<<grid, block, 0, s>>>(a);
}

void launch_prologue(const PrologueArgs& a, cudaStream_t s) {
  dim3 grid((a.ny + 255) / 256, a.nx < 4096 ? a.nx : 4096);
  prologue_kernel<<<grid, 256, 0, s>>>(a);
}

void launch_finish(const FinishArgs& a, cudaStream_t s) {
  const int n = a.nx + a.ny;
  finish_kernel<<<(n + 255) / 256, 256, 0, s>>>(a);
}

void launch_init(const InitArgs& a, cudaStream_t s) {
  dim3 grid((a.ny + 255) / 256, a.nx < 4096 ? a.nx : 4096);
  init_kernel<<<grid, 256, 0, s>>>(a);
}

}  // namespace hb
