// hydro_kernels.cuh -- device-side state layout and kernel parameter blocks.
#pragma once

#include <cuda.h>

#include <cstddef>
#include <cstdint>

#include "hydro_physics.cuh"

namespace hb {

// HBM layout ("row-interleaved planes"): for each grid row i in [-1, nx+2]
// the four variable rows rho, mom_x, mom_y, ener are stored back to back,
// each `pitch` doubles long; column j in [-1, ny+2] sits at offset j + kColOff,
// so interior column 1 starts a 64-byte DRAM access unit (the granule TMA
// fetches: column-sweep box rows of 32 columns are then exactly four units,
// row-sweep chunks of 8 columns one).  Two consecutive grid rows (all four
// variables) are one contiguous block of 8*pitch doubles -- a slab halo is a
// single contiguous send/recv.
constexpr int kColOff = 7;

// Staging (both sweeps): every warp stages chunks of all four variables for
// its 32 strips into its own ring of buffers (4 warps per CTA).
//   column sweep: kChunkX grid rows x 32 columns per chunk, kNBufX buffers;
//   row sweep:    kChunkY columns x 32 grid rows per chunk, kNBufY buffers.
#ifndef HB_NBUF
#define HB_NBUF 3
#endif
// The HLLC row sweep: 8-cell chunks in two buffers (64 KB per CTA, 3 CTAs
// per SM) for the bitwise TU; the tolerance TU's lighter walker fits 128
// registers, and 4-cell chunks in three buffers give it 4 CTAs per SM
// (gpurun_out r2fi: config 3 -4%, config 2 -3%, config 4 -8% per row sweep).
#ifndef HB_YCHUNK
#ifdef HB_TOLERANCE
#define HB_YCHUNK 4
#else
#define HB_YCHUNK 8
#endif
#endif
#ifndef HB_YNBUF
#ifdef HB_TOLERANCE
#define HB_YNBUF 3
#else
#define HB_YNBUF 2
#endif
#endif
// The exact-10 row sweep keeps 4-cell chunks in three buffers: with its
// interface memo an 8-cell ring would cost it a resident CTA per SM.
template <int AXIS, int FLUX = 0>
struct Staging {
  static constexpr bool kWide = AXIS == 1 && FLUX == 0;
  static constexpr int C = kWide ? HB_YCHUNK : 4;          // cells per strip per chunk
  static constexpr int NBUF = kWide ? HB_YNBUF : HB_NBUF;  // ring buffers per warp
  static constexpr int kChunkBytes = 32 * 4 * C * 8;
  static constexpr int kSmem = 4 * NBUF * kChunkBytes + 1024 + 4 * NBUF * 8;  // + align, mbarriers
};
constexpr int kXSmemBytes = Staging<0>::kSmem;
constexpr int kYSmemBytes = Staging<1>::kSmem;
// exact-10 sweeps: + one 13-double interface memo per thread
constexpr int kMemoBytes = 13 * 128 * 8;
constexpr int kExXSmemBytes = Staging<0, 1>::kSmem + kMemoBytes;
constexpr int kExYSmemBytes = Staging<1, 1>::kSmem + kMemoBytes;

// Both state buffers are stored TILED (r2): blocks of 32 grid rows x 8
// columns x 4 variables (8 KB), block (ti, tj) at ((ti + 1) * (pitch / 8) + tj)
// * 1024 doubles, element [v][ri][rj] inside, with ti = floor((i - 1) / 32),
// ri = i - 1 - 32 ti, tj = (j + kColOff) / 8, rj = (j + kColOff) % 8 (grid
// rows -1 .. nx+2, i.e. block rows -1 .. tile_rows - 2; `pitch` = 8 x the
// block columns).  A row-sweep chunk (32 rows of one row group x 8 columns x
// 4 variables) is then one contiguous 8 KB block, and a column-sweep chunk
// (4 rows x 32 columns) sixteen 256-byte pieces: tools/tma_pattern.cu
// streams the row sweep's pattern at 6.6 TB/s on this layout against 4.4 TB/s
// with 64-byte pieces of row-interleaved planes.
__host__ __device__ __forceinline__ size_t cell_index(size_t pitch, int v, int i, int j) {
  const int ti = (i + 31) / 32 - 1;  // floor((i - 1) / 32) for i >= -31
  const int ri = i - 1 - 32 * ti;
  const int c = j + kColOff;
  return (((size_t)(ti + 1) * (pitch / 8) + (size_t)(c >> 3)) * 4 + (size_t)v) * 256 +
         (size_t)ri * 8 + (size_t)(c & 7);
}
// distance between the variables of one cell
constexpr size_t kVarStep = 256;
// Block rows of a state buffer: grid rows -1 .. nx+2.
__host__ __device__ __forceinline__ int tile_rows(int nx) { return (nx + 1) / 32 + 2; }
__host__ __device__ __forceinline__ size_t state_doubles(int nx, size_t pitch) {
  return (size_t)tile_rows(nx) * (pitch / 8) * 1024;
}

inline size_t pitch_for(int ny) {
  const size_t need = (size_t)ny + 3 + kColOff;  // offsets 0..ny+2+kColOff
  return (need + 15) / 16 * 16;        // 128-byte rows
}

// The FUSED schedule (hydro_fused.cuh): bands of kFW output columns; the
// column phase loads kFLoadBlocks column blocks (one either side).
constexpr int kFW = 120;
constexpr int kFLoadBlocks = kFW / 8 + 2;

struct SweepArgs {
  const double* __restrict__ src;
  double* __restrict__ dst;
  size_t pitch;
  int nx, ny;                 // local interior extent
  int seg;                    // strip segment length per thread
  int nseg;                   // segments per strip
  int band;                   // strip groups per band of the claim order (item_coords)
  double dx;                  // spacing along the sweep
  double spacing;             // min(dx, dy) for the dt limit
  double gamma, cfl;
  int bc;                     // 0 reflect, 1 transmit
  int flux;                   // 0 HLLC, 1 exact Riemann (10 Newton iterations)
  int wall_lo, wall_hi;       // physical walls on the i sides of this slab
  int row0;                   // global row of local row 1, minus 1
  unsigned long long* limit_in;   // dt limit consumed by this step
  unsigned long long* limit_out;  // dt limit produced for the next step
  unsigned long long* err;        // latched error key
  unsigned long long* dt_err;     // dt failure for the next step
  int step;
  int explicit_dt;            // 1: use dt_value instead of cfl*limit_in
  double dt_value;
  int want_limit;             // row sweep: produce limit_out
  unsigned* counter;          // work-item counter of this sweep (starts at 0)
  unsigned* counter_next;     // the other sweep's counter, reset for its launch
  double* halo_up;            // row sweep: upper neighbour's inbox block for rows 1..2
  double* halo_dn;            // row sweep: lower neighbour's inbox block for rows nx-1..nx
  unsigned long long* skipped;  // cell updates taken by the uniform-window identity (counter)
  double dx2;                 // fused step: the row sweep's spacing (dy)
  unsigned* done;             // fused step: CTAs finished (the last one resets limit_in, counter)
  int last_step;              // fused step: the run's last -- leaves the final ghost bands behind
};

// All maps view a tiled buffer as dims {column in block, column block, row in
// block, var, block row} (strides not increasing).
struct TmaMaps {
  CUtensorMap y_load;         // U_b: one block {8 cols, 32 rows, 4 vars}
  CUtensorMap y_store;        // U_a: the same
  CUtensorMap x_load;         // U_a: {8 cols, 4 blocks, 4 rows, 4 vars} -> smem [var][row][col]
  CUtensorMap x_store;        // U_b: the same
  CUtensorMap ey_load;        // the exact-10 row sweep: {4 cols, 32 rows, 4 vars} of U_b
  CUtensorMap ey_store;       // ... and of U_a
  int y_cols, ey_cols;        // box widths (columns) of the y / ey maps
  // fused step (hydro_fused.cuh): loads {8 cols, kFLoadBlocks blocks, 4 rows,
  // 4 vars} -> smem [var][row][col], row stores {8 cols, kFW/8 blocks, 1 row,
  // 1 var}, of either buffer
  CUtensorMap fa_load, fb_load, fa_store, fb_store;
};

struct PrologueArgs {
  double* u;
  size_t pitch;
  int nx, ny;
  double spacing, gamma;
  int bc, wall_lo, wall_hi, row0;
  int want_limit, full_bc;
  unsigned long long* limit_out;
  unsigned long long* err;
  unsigned long long* dt_err;
  int step;
};

struct FinishArgs {
  const double* post_x;       // column-sweep output of the last step
  double* u;                  // final state
  size_t pitch;
  int nx, ny, bc, wall_lo, wall_hi;
};

struct InitArgs {
  double* u;
  size_t pitch;
  int nx, ny, global_nx, row0;
  int case_id;
  double gamma, dx, dy;
  unsigned long long seed;
};

struct Geometry {
  int ctas_x_per_sm;          // resident CTAs per SM (from the occupancy API)
  int ctas_y_per_sm;
  int ctas_x_exact;           // the same for the exact-10 flux instantiations
  int ctas_y_exact;
  int ctas_xy_per_sm;         // the fused step
  int sms;
};

bool make_tma_maps(TmaMaps* maps, double* A, double* B, size_t pitch, int nx, int ny);
int query_geometry(Geometry* g);
void launch_sweep_x(const SweepArgs& a, const TmaMaps& maps, const Geometry& geo, cudaStream_t s);
void launch_sweep_y(const SweepArgs& a, const TmaMaps& maps, const Geometry& geo, cudaStream_t s);
// Tolerance math mode (hydro_kernels_tol.cu): the same sweeps
// built with FMA contraction and uncorrected reciprocal quotients.
int query_geometry_tol(Geometry* g);
void launch_sweep_x_tol(const SweepArgs& a, const TmaMaps& maps, const Geometry& geo, cudaStream_t s);
void launch_sweep_y_tol(const SweepArgs& a, const TmaMaps& maps, const Geometry& geo, cudaStream_t s);
// The fused step (one launch per time step; hydro_fused.cuh): a.src -> a.dst
// with the maps of those buffers.  HLLC only.
void launch_sweep_xy(const SweepArgs& a, const CUtensorMap& load, const CUtensorMap& store,
                     const Geometry& geo, cudaStream_t s);
void launch_sweep_xy_tol(const SweepArgs& a, const CUtensorMap& load, const CUtensorMap& store,
                         const Geometry& geo, cudaStream_t s);
void launch_prologue(const PrologueArgs& a, cudaStream_t s);
void launch_prologue_tol(const PrologueArgs& a, cudaStream_t s);  // the tolerance mode's dt
void launch_finish(const FinishArgs& a, cudaStream_t s);
// The tiled U_b's ghost column ny+2 for reflecting walls with ny % 32 == 1
// (no-op otherwise); after every column sweep.
void launch_ghost_fix(double* b, size_t pitch, int nx, int ny, int bc, cudaStream_t s);
// ... and U_a's ghost row nx+2 (lower wall, nx % 32 == 1); after every row sweep.
void launch_ghost_row_fix(double* a, size_t pitch, int nx, int ny, int bc, int wall_hi,
                          cudaStream_t s);
// Row-layout <-> tiled transfers of plane rows (host transfer staging, the
// slab halo): rows[r][j + kColOff'] <-> cell (row0 + r, j) of variable v
// (or of all 4 variables, row-interleaved, for the halo blocks).
void launch_rows_to_tiles(const double* rows, size_t row_stride, double* u, size_t pitch, int v,
                          int i0, int n, int ny, cudaStream_t s);
void launch_tiles_to_rows(const double* u, size_t pitch, double* rows, size_t row_stride, int v,
                          int i0, int n, int ny, cudaStream_t s);
void launch_compare(const double* a, const double* b, size_t pitch, int nx, int ny,
                    unsigned long long* out, cudaStream_t s);
void launch_init(const InitArgs& a, cudaStream_t s);
void launch_row_audit(const double* u, size_t pitch, int nx, int ny, unsigned long long* hashes,
                      double* sums, cudaStream_t s);
void launch_math_selftest(int op, const double* a, const double* b, double* fast, double* ref,
                          int* ok, size_t n, cudaStream_t s);

}  // namespace hb
