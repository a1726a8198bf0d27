/*
 * hydro_gpu.h -- C-ABI of the B200-native HYDRO time step (libhydro_b200.so).
 *
 * This is the drop-in boundary for the reference hydro2d's stepping entry
 * points (all paths relative to /root/reference/):
 *
 *   reference (proj/include/hydro/schedulers.hpp)       replaced by
 *   -------------------------------------------------  ---------------------
 *   run_sequential(Grid2D&, const GasModel&, int)   :24  hydro_gpu_run
 *   advance_sequential(Grid2D&, const GasModel&, dt):21  hydro_gpu_advance
 *   run_until(Grid2D&, const GasModel&, double)     :28  hydro_gpu_run_until
 *   compute_dt(const Grid2D&, const GasModel&)  euler_kernel.hpp:75
 *                                                        hydro_gpu_compute_dt
 *   grid_checksum(...).digest          audit.hpp:34      hydro_grid_digest
 *   Grid2D storage (4 planes, grid.hpp:26-64)            hydro_gpu_upload /
 *                                                        hydro_gpu_download
 *   run_strategy dispatch (proj/src/bench.cpp:53-90)     a "gpu" strategy
 *
 *
 * Conventions: plain C types only, no exceptions cross the boundary, every
 * call returns an int status: 0 = OK, 1..7 = hydro::ErrorCategory + 1
 * (proj/include/hydro/errors.hpp:10-18), 8 = CUDA / device failure.  A
 * positivity failure carries the same step / sweep / strip / cell context the
 * reference prints (proj/src/schedulers.cpp:23-26,80-91): fetch it with
 * hydro_gpu_last_error.  A context is single-caller and its calls are
 * synchronous unless stated otherwise (the reference's callers are
 * single-threaded).
 *
 * Host plane layout accepted by upload/download: the reference Grid2D plane
 * layout -- (nx+4) rows of `row_stride` doubles, interior cell (i,j) at
 * row i+1, column j+1 (grid.hpp:54-57).  Pass the address of cell (-1,-1) of
 * each plane (&grid.at(Var(v), -1, -1)) and row_stride = ny+4.
 */
#ifndef HYDRO_GPU_H
#define HYDRO_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HYDRO_GPU_ABI_VERSION 1

enum hydro_gpu_status {
  HYDRO_GPU_OK = 0,
  HYDRO_GPU_ERR_CONFIG = 1,      /* ErrorCategory::Config */
  HYDRO_GPU_ERR_POSITIVITY = 2,  /* ErrorCategory::Positivity */
  HYDRO_GPU_ERR_PROTOCOL = 3,
  HYDRO_GPU_ERR_TASKGRAPH = 4,
  HYDRO_GPU_ERR_EQUIVALENCE = 5,
  HYDRO_GPU_ERR_IO = 6,
  HYDRO_GPU_ERR_VALIDATION = 7,
  HYDRO_GPU_ERR_CUDA = 8         /* no reference equivalent: device failure */
};

/* Boundary kind: REFLECT is the reference's apply_boundary
 * (proj/src/grid.cpp:23-60); TRANSMIT is zero-gradient (both ghost layers
 * copy the adjacent interior cell), needed by BASELINE configs 1, 2, 4. */
enum hydro_gpu_bc { HYDRO_GPU_BC_REFLECT = 0, HYDRO_GPU_BC_TRANSMIT = 1 };

/* Riemann flux: HLLC is the reference hot path (euler_kernel.cpp:59-109);
 * EXACT10 is BASELINE's "exact Riemann solver with 10 Newton iterations": the
 * reference's exact solver (exact_riemann.cpp) sampled at x/t = 0, with a
 * portable log/exp in place of std::pow (bitwise equal to the C oracle,
 * floored-relative 1e-12 against std::pow).  A vacuum-generating state pair
 * is a Validation error, as in exact_riemann.cpp:55-57. */
enum hydro_gpu_flux { HYDRO_GPU_FLUX_HLLC = 0, HYDRO_GPU_FLUX_EXACT10 = 1 };

/* Arithmetic of the sweeps.  BITWISE (the default) reproduces the reference's
 * -ffp-contract=off IEEE arithmetic bit for bit.  TOLERANCE is the
 * north-star contract instead: compare_tolerance max_rel <= 1e-12 against the
 * reference (proj/src/audit.cpp:146) -- quotients as a * (1/b) with one
 * Newton-refined reciprocal per denominator, square roots without the final
 * correction.  Every branch, fallback and error check of the
 * reference is kept, and the results do not depend on the launch geometry,
 * the slab split or how a run is divided into calls. */
enum hydro_gpu_math { HYDRO_GPU_MATH_BITWISE = 0, HYDRO_GPU_MATH_TOLERANCE = 1 };
/* Step schedule (hydro_gpu_set_schedule): SPLIT = a column-sweep and a
 * row-sweep launch per step; FUSED = one launch per step doing both sweeps
 * (the column sweep's output stays in shared memory), used with the HLLC
 * flux for every step of a run (after one split step when the step count is
 * odd), on whole domains and row slabs -- bitwise the same results.  AUTO
 * (the default) picks between them per run from the context's own completed
 * runs: the share of cell updates taken by the
 * uniform-window identity (fused above 0.6: memory-bound flow) and the
 * event-timed device time per step of each schedule (an untimed schedule is
 * tried once); a context's first run is fused. */
enum hydro_gpu_schedule {
  HYDRO_GPU_SCHEDULE_SPLIT = 0,
  HYDRO_GPU_SCHEDULE_FUSED = 1,
  HYDRO_GPU_SCHEDULE_AUTO = 2
};

/* Case ids for the initialisers (cases.cpp:11-69 + BASELINE configs). */
enum hydro_gpu_case {
  HYDRO_GPU_CASE_UNIFORM = 0,
  HYDRO_GPU_CASE_BLAST = 1,
  HYDRO_GPU_CASE_SOD_J = 2,
  HYDRO_GPU_CASE_CORNER_BLAST = 3,
  HYDRO_GPU_CASE_SOD_X = 4,
  HYDRO_GPU_CASE_RANDOM = 5
};

typedef struct hydro_gpu_cfg {
  int nx, ny;          /* interior extent held by this context (a slab for P>1) */
  double dx, dy;       /* cell sizes (Grid2D::dx/dy) */
  double gamma, cfl;   /* GasModel (types.hpp:38-41) */
  int bc;              /* enum hydro_gpu_bc */
  int flux;            /* enum hydro_gpu_flux */
  int device;          /* CUDA device ordinal; -1 = the calling thread's current */
  /* Row-slab decomposition along i.  A full grid is
   * row0 = 0, global_nx = nx, wall_lo = wall_hi = 1. */
  int row0;            /* global row index of this slab's first interior row, minus 1 */
  int global_nx;       /* interior rows of the whole grid */
  int wall_lo;         /* 1: rows 0,-1 are a physical wall; 0: filled by a halo exchange */
  int wall_hi;         /* 1: rows nx+1,nx+2 are a physical wall */
} hydro_gpu_cfg;

typedef struct hydro_gpu_error {
  int category;        /* enum hydro_gpu_status */
  int step;            /* step index within the failing call */
  int phase;           /* 0 = compute_dt, 1 = column sweep, 2 = row sweep */
  int strip;           /* 1-based strip (column j or row i); grid row for phase 0 */
  int loop;            /* 0 = primitive conversion, 1 = Riemann, 2 = conservative update */
  int cell;            /* strip-local index k - kGhost as printed by the reference */
  int field;           /* 0 = rho, 1 = pres, 2 = internal energy, 3 = vacuum */
  char message[256];   /* the reference's what() text, context included */
} hydro_gpu_error;

typedef struct hydro_gpu_ctx hydro_gpu_ctx;

/* ---- lifetime ---------------------------------------------------------- */
int hydro_gpu_abi_version(void);
int hydro_gpu_create(const hydro_gpu_cfg* cfg, hydro_gpu_ctx** out);
int hydro_gpu_destroy(hydro_gpu_ctx* ctx);
const char* hydro_gpu_status_string(int status);
int hydro_gpu_last_error(const hydro_gpu_ctx* ctx, hydro_gpu_error* out);

/* ---- state transfer (host <-> HBM) ------------------------------------- */
int hydro_gpu_upload(hydro_gpu_ctx* ctx, const double* const planes[4],
                     size_t row_stride);
/* Grid rows i_lo .. i_lo+nrows-1 (within -1 .. nx+2) of the 4 planes only;
 * planes[v] points at grid row i_lo's column -1. */
int hydro_gpu_download_rows(hydro_gpu_ctx* ctx, double* const planes[4], size_t row_stride,
                            int i_lo, int nrows);
/* compare_tolerance's max |a-b| / max(|a|,|b|,1) over the interior
 * (proj/src/audit.cpp:137-154) of two contexts of one geometry on one
 * device, computed on the device. */
int hydro_gpu_compare(hydro_gpu_ctx* a, hydro_gpu_ctx* b, double* max_rel);
int hydro_gpu_download(hydro_gpu_ctx* ctx, double* const planes[4],
                       size_t row_stride);
/* The same transfers enqueued on the context's stream without waiting (see
 * hydro_gpu_set_stream): with pinned host planes they overlap kernels of
 * other streams, so independent problems on two contexts pipeline copies
 * with compute.  The host planes must stay valid until hydro_gpu_sync. */
int hydro_gpu_upload_async(hydro_gpu_ctx* ctx, const double* const planes[4],
                           size_t row_stride);
int hydro_gpu_download_async(hydro_gpu_ctx* ctx, double* const planes[4],
                             size_t row_stride);
/* Device-side initialiser, bitwise equal to hydro_init_case_host. */
int hydro_gpu_init_case(hydro_gpu_ctx* ctx, int case_id, uint64_t seed);

/* ---- the reference's stepping entry points ----------------------------- */
/* Step counts of one run / run_until call are bounded (the device error
 * record orders failures by a 22-bit step field): more is a config error,
 * and run_until stops there with one. */
#define HYDRO_GPU_MAX_STEPS 4194302

/* run_sequential: `steps` steps of BC -> dt -> column sweep -> BC -> row
 * sweep.  *last_dt (may be NULL) receives the dt of the final step. */
int hydro_gpu_run(hydro_gpu_ctx* ctx, int steps, double* last_dt);
/* advance_sequential: one step with a caller-chosen dt. */
int hydro_gpu_advance(hydro_gpu_ctx* ctx, double dt);
/* run_until: advance to t_end, clamping the last dt; *steps = steps taken. */
int hydro_gpu_run_until(hydro_gpu_ctx* ctx, double t_end, int* steps);
/* compute_dt after apply_boundary: cfl * min cell_dt_limit. */
int hydro_gpu_compute_dt(hydro_gpu_ctx* ctx, double* dt);

/* ---- asynchronous, device-resident interface --------------------------- */
/* Stream all work of this context is issued on (a cudaStream_t; NULL is the
 * CUDA default stream, as everywhere in CUDA).  A new context uses its own
 * non-blocking stream; hydro_gpu_use_own_stream restores it. */
int hydro_gpu_set_stream(hydro_gpu_ctx* ctx, void* cuda_stream);
int hydro_gpu_use_own_stream(hydro_gpu_ctx* ctx);
/* Enqueues `steps` steps without synchronising; errors are latched on the
 * device and reported by the next hydro_gpu_sync. */
int hydro_gpu_run_async(hydro_gpu_ctx* ctx, int steps);
int hydro_gpu_sync(hydro_gpu_ctx* ctx);

/* ---- slab phases for multi-GPU drivers (one context per GPU) ----------- */
/* Physical-wall BC on the current state + local dt limit into the slot
 * step `step` reads.  Enqueued, not synchronised. */
int hydro_gpu_slab_prologue(hydro_gpu_ctx* ctx, int step);
/* Device address of the (pre-cfl) dt limit consumed by `step`: a driver
 * min-allreduces it across slabs between the previous row sweep and the
 * column sweep of `step`. */
int hydro_gpu_limit_slot(hydro_gpu_ctx* ctx, int step, double** dev_ptr);
/* Device address of the latched error key (uint64, min-combinable). */
int hydro_gpu_error_slot(hydro_gpu_ctx* ctx, uint64_t** dev_ptr);
/* Halo rows in the current state: send_lo = interior rows 1..2,
 * send_hi = rows nx-1..nx, recv_lo = ghost rows -1..0, recv_hi = ghost rows
 * nx+1..nx+2.  Each is one contiguous block of `count` doubles (2 rows x 4
 * variables x pitch), so a halo swap is one send/recv per neighbour. */
int hydro_gpu_halo(hydro_gpu_ctx* ctx, double** send_lo, double** send_hi,
                   double** recv_lo, double** recv_hi, size_t* count);
/* The collective halo transport: hydro_gpu_halo's four blocks (2 rows x 4
 * variables, `count` doubles each, the inbox format) are a staging buffer of
 * the tiled state: pack rows 1..2 / nx-1..nx into the send blocks before the
 * sends, unpack the received blocks into ghost rows -1..0 / nx+1..nx+2
 * after the receives (both on the context's stream). */
int hydro_gpu_slab_halo_pack(hydro_gpu_ctx* ctx);
int hydro_gpu_slab_halo_unpack(hydro_gpu_ctx* ctx);
int hydro_gpu_slab_sweep_x(hydro_gpu_ctx* ctx, int step);
int hydro_gpu_slab_sweep_y(hydro_gpu_ctx* ctx, int step);
/* Peer-memory halo (row slabs on NVLink-connected GPUs; replaces the per-step
 * send/recv of hydro_gpu_halo's blocks).  Each slab owns an inbox of 2 step
 * parities x 2 sides (side 0 = its ghost rows -1..0, side 1 = nx+1..nx+2),
 * each one block of `count` doubles laid out like hydro_gpu_halo's.  With
 * peers set, the row sweep of step s also stores the slab's updated rows 1..2
 * into the upper neighbour's side-1 inbox of parity (s+1)&1 and rows
 * nx-1..nx into the lower neighbour's side-0 inbox (the decomposition's
 * InterfaceBuffer, proj/include/hydro/decomposition.hpp:58-79, written by
 * the producing kernel); hydro_gpu_slab_inbox_in(step) copies the parity
 * step&1 inbox into the ghost rows before the column sweep.  Writer and
 * reader are ordered by the per-step dt min-allreduce between them, and the
 * parity keeps a neighbour's next write off the block being read. */
int hydro_gpu_inbox(hydro_gpu_ctx* ctx, double** inbox, size_t* count);
/* cudaIpcMemHandle_t of the inbox allocation (64 bytes) for another process. */
int hydro_gpu_inbox_ipc_handle(hydro_gpu_ctx* ctx, void* handle64);
/* Maps a neighbour's inbox from its IPC handle (closed by hydro_gpu_destroy). */
int hydro_gpu_ipc_open(hydro_gpu_ctx* ctx, const void* handle64, double** peer_inbox);
/* Neighbour inboxes (NULL: physical wall / NCCL halo); upper = slab above
 * (row0 smaller), lower = slab below. */
int hydro_gpu_set_halo_peers(hydro_gpu_ctx* ctx, double* upper_inbox, double* lower_inbox);
/* Copies the current rows 1..2 / nx-1..nx into the neighbours' inboxes of
 * parity step&1 (the initial exchange, after hydro_gpu_slab_prologue). */
int hydro_gpu_slab_halo_out(hydro_gpu_ctx* ctx, int step);
/* Ghost rows of the non-wall sides from this slab's inbox of parity step&1. */
int hydro_gpu_slab_inbox_in(hydro_gpu_ctx* ctx, int step);
/* Writes the reference's end-of-run ghost state (mirrors of the last
 * column-sweep output, grid.cpp:23-60 as applied before the last row sweep). */
int hydro_gpu_slab_finish(hydro_gpu_ctx* ctx);
/* The fused schedule for a caller that drives the slab's steps itself
 * (hydro_gpu_group): run_begin remakes the AUTO choice, counts the run and
 * says whether it takes fused steps; step_xy is one fused step (phase 0:
 * U_a -> U_b, 1: U_b -> U_a; first = the run's first fused step, last = the
 * run's last step, halo != 0: the inbox of parity step&1 is first copied into
 * the ghost rows of the step's input buffer); run_end enqueues
 * hydro_gpu_slab_finish's work unless the last step was fused, and the
 * counters the next AUTO choice reads. */
int hydro_gpu_slab_run_begin(hydro_gpu_ctx* ctx, int steps, int* fused);
int hydro_gpu_slab_step_xy(hydro_gpu_ctx* ctx, int step, int phase, int first, int last, int halo);
int hydro_gpu_slab_run_end(hydro_gpu_ctx* ctx, int fused_last);

/* ---- multi-rank slabs driven from C++ (one process per GPU) ------------ */
/* An NCCL unique id (128 bytes) made on one rank and shared with the others
 * by the caller (the reference has no multi-process layer). */
int hydro_gpu_comm_unique_id(void* id128);
/* Attaches this slab context to the ranks' NCCL communicator (NCCL is loaded
 * at run time).  With more than one rank the slab's halo neighbours must be
 * mapped first (hydro_gpu_set_halo_peers).  From then on hydro_gpu_run /
 * hydro_gpu_run_async run this rank's part of run_sequential
 * (schedulers.cpp:103-116) as ONE captured CUDA graph per step count: per
 * step the dt limit ncclMin-allreduced (compute_dt_parallel,
 * schedulers.cpp:47-65), the inbox copied into the ghost rows (the halo the
 * neighbours' row sweeps stored over NVLink), both sweeps; at the end the
 * error slots min-allreduced, so every rank reports the first error of the
 * whole grid.  All ranks must call the same runs. */
int hydro_gpu_comm_attach(hydro_gpu_ctx* ctx, const void* id128, int nranks, int rank);
/* Device milliseconds and count of the per-step exchanges (allreduce +
 * inbox copy) timed while timing is on (hydro_gpu_set_timing). */
int hydro_gpu_comm_times(hydro_gpu_ctx* ctx, double* ms, long long* n);
/* Synchronises and decodes a (possibly all-reduced) error key. */
int hydro_gpu_decode_error(hydro_gpu_ctx* ctx, uint64_t key, hydro_gpu_error* out);

/* ---- one process, several GPUs (n_gpus > 1) -------------- */
/* A row-slab decomposition of one grid driven by the calling host thread:
 * slab k (rows split like split_range, proj/src/decomposition.cpp:9-16) is a
 * hydro_gpu_ctx on devices[k] (NULL: device k mod the device count; repeated
 * ordinals are allowed, e.g. all slabs on one GPU).  Peer access is enabled
 * between all slab devices; the halo is the peer-memory inbox path above
 * with plain device pointers, and the dt of every step is the minimum of the
 * slabs' limits, read over NVLink by a one-warp kernel on each device after
 * an event join (the single-process twin of the NCCL min-allreduce,
 * compute_dt_parallel, proj/src/schedulers.cpp:47-65).  cfg describes the
 * whole grid (row0 / global_nx / wall_* are ignored).  Results are bitwise
 * those of one context on the whole grid.  Returns HYDRO_GPU_ERR_CUDA if two
 * distinct devices cannot access each other's memory. */
typedef struct hydro_gpu_group hydro_gpu_group;
int hydro_gpu_group_create(const hydro_gpu_cfg* cfg, int n_gpus, const int* devices,
                           hydro_gpu_group** out);
int hydro_gpu_group_destroy(hydro_gpu_group* group);
int hydro_gpu_group_last_error(const hydro_gpu_group* group, hydro_gpu_error* out);
/* Slab count and, per slab (arrays of n entries, any may be NULL), its first
 * global row minus 1, its rows and its device. */
int hydro_gpu_group_slabs(const hydro_gpu_group* group, int* n, int* row0, int* rows,
                          int* devices);
/* Whole-grid planes in the reference layout (as hydro_gpu_upload/download). */
int hydro_gpu_group_upload(hydro_gpu_group* group, const double* const planes[4],
                           size_t row_stride);
int hydro_gpu_group_download(hydro_gpu_group* group, double* const planes[4],
                             size_t row_stride);
int hydro_gpu_group_init_case(hydro_gpu_group* group, int case_id, uint64_t seed);
/* hydro_gpu_set_math on every slab. */
int hydro_gpu_group_set_math(hydro_gpu_group* group, int math);
/* run_sequential over all slabs; *last_dt as hydro_gpu_run. */
int hydro_gpu_group_run(hydro_gpu_group* group, int steps, double* last_dt);

/* ---- instrumentation ---------------------------------------------------- */
/* When on, every sweep launch is bracketed by CUDA events on the launch
 * stream; hydro_gpu_kernel_times returns the summed device milliseconds and
 * launch counts since the last reset. */
int hydro_gpu_set_timing(hydro_gpu_ctx* ctx, int on);
int hydro_gpu_kernel_times(hydro_gpu_ctx* ctx, double* ms_x, double* ms_y,
                           double* ms_other, long long* n_x, long long* n_y,
                           long long* n_other);
int hydro_gpu_reset_counters(hydro_gpu_ctx* ctx);
/* Cell updates of the column / row sweeps since the last reset_counters that
 * took the uniform-window identity (a cell whose 5-cell
 * stencil window equals its predecessor's, whose update was the identity,
 * gets the identical result without re-evaluating it). */
int hydro_gpu_skipped(hydro_gpu_ctx* ctx, uint64_t* x, uint64_t* y);
/* Launch-geometry override (0 = default): strip segment length along the
 * column and row sweeps; block must be 0 or 128. */
int hydro_gpu_tune(hydro_gpu_ctx* ctx, int seg_x, int seg_y, int block);
/* Claim-order override of the column / row sweep: work items run in bands of
 * `band` strip groups (32 strips each) x all segments; 0 = automatic, a value
 * >= the number of strip groups = segment-major over the whole grid. */
int hydro_gpu_tune_order(hydro_gpu_ctx* ctx, int band_x, int band_y);
/* Selects the sweeps' arithmetic (enum hydro_gpu_math) for later runs of
 * this context; no reference equivalent (the reference has one arithmetic).
 * Config error for an unknown mode. */
int hydro_gpu_set_math(hydro_gpu_ctx* ctx, int math);
/* Selects the step schedule (enum hydro_gpu_schedule; default AUTO) and the
 * fused step's rows per work item (0 = automatic) for later runs; no
 * reference equivalent (results do not depend on it).  Config error for an
 * unknown schedule. */
int hydro_gpu_set_schedule(hydro_gpu_ctx* ctx, int schedule, int seg);
/* What the next run of this context would do: *fused = 1 if it takes fused
 * steps; *share = the uniform-window share behind an AUTO choice (-1 before
 * the first completed run). */
int hydro_gpu_schedule_choice(hydro_gpu_ctx* ctx, int* fused, double* share);
/* Summed device milliseconds and launch count of the fused steps while
 * timing is on (hydro_gpu_set_timing). */
int hydro_gpu_fused_times(hydro_gpu_ctx* ctx, double* ms, long long* n);
/* Self-test of the device fp64 division (op 0), square root (op 1),
 * signed-zero-safe division (op 2) and density division (op 4: zero
 * numerators, denominators inside the fast-pass envelope [2^-256, 2^256))
 * and envelope-bounded division (op 5: no range test) fast paths against the
 * compiler's IEEE operations on n operand pairs (b ignored for sqrt), and of
 * the fast-pass minmod of two slopes (op 3) against the reference's
 * comparisons.
 * in_range[k] = 1 where the fast path applied. */
int hydro_gpu_math_selftest(int op, const double* a, const double* b, double* fast,
                            double* exact, int* in_range, size_t n);
/* Device pointer to the state and its pitch (doubles).  The state is tiled:
 * blocks of 32 grid rows x 8 columns x 4 variables; cell (i, j) of variable
 * v, i and j in [-1, n+2], with c = j + hydro_gpu_col_offset(),
 * ti = floor((i - 1) / 32), ri = i - 1 - 32 ti, is element
 * (((ti + 1) * (pitch / 8) + c / 8) * 4 + v) * 256 + ri * 8 + c % 8. */
int hydro_gpu_state(hydro_gpu_ctx* ctx, double** dev_ptr, size_t* pitch);
int hydro_gpu_col_offset(void);

/* ---- device-side audit (no grid download) ------------------------------ */
/* Per (variable, interior row) FNV-1a hash and plain sum of the current
 * state, 4*nx entries each (variable-major, rows in order); either pointer
 * may be NULL. */
int hydro_gpu_row_audit(hydro_gpu_ctx* ctx, uint64_t* row_hashes, double* row_sums);
/* Composable state hash: FNV-1a over the row hashes in (variable, global row)
 * order.  Equal to hydro_grid_state_hash of the downloaded planes; for row
 * slabs, the row hashes of all ranks in global order combine to the hash of
 * the whole grid (hydro_combine_row_hashes). */
int hydro_gpu_state_hash(hydro_gpu_ctx* ctx, uint64_t* out);
/* Volume-weighted interior totals (conservation_totals, audit.cpp:16-51):
 * per-row sums on the device, pairwise over rows on the host. */
int hydro_gpu_totals(hydro_gpu_ctx* ctx, double out[4]);

/* ---- host utilities (no device needed) --------------------------------- */
/* FNV-1a digest of the interior bytes (proj/src/audit.cpp:53-76). */
uint64_t hydro_grid_digest(const double* const planes[4], size_t row_stride,
                           int nx, int ny);
/* The same FNV-1a continued from state h over interior rows 1..nx of one
 * plane: the digest of a grid split into row slabs is the chain over
 * (plane, slab) in plane-major, slab order, starting from the FNV offset
 * basis 14695981039346656037. */
uint64_t hydro_fnv1a_rows(uint64_t h, const double* plane, size_t row_stride, int nx,
                          int ny);
/* The state hash of host Grid2D planes, and its combining step. */
uint64_t hydro_grid_state_hash(const double* const planes[4], size_t row_stride, int nx,
                               int ny);
uint64_t hydro_combine_row_hashes(const uint64_t* row_hashes, size_t n);
/* pairwise_sum of audit.cpp:16-25. */
double hydro_pairwise_sum(const double* v, size_t n);
/* Host initialiser for the case ids above; fills 4 planes (zeroing first,
 * like Grid2D's constructor) and the spacings. */
int hydro_init_case_host(int case_id, int nx, int ny, double gamma,
                         uint64_t seed, double* const planes[4],
                         size_t row_stride, double* dx, double* dy);

#ifdef __cplusplus
}
#endif

#endif /* HYDRO_GPU_H */
