// hydro_abi.cu -- the extern "C" boundary of libhydro_b200.so (include/hydro_gpu.h).
//
// Owns the device state of one grid (or one row slab of a multi-GPU grid):
// two row-interleaved state buffers used ping-pong (U_a -> column sweep ->
// U_b -> row sweep -> U_a), four 64-bit device slots (two dt limits, the
// latched error key, a pending compute_dt error), a stream and optional
// per-launch CUDA events.  Errors never cross the boundary as exceptions:
// each call returns a status mirroring hydro::ErrorCategory
// (proj/include/hydro/errors.hpp:10-18) and records a hydro_gpu_error whose
// message reproduces the reference's text, context included
// (proj/src/schedulers.cpp:23-26,80-91).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#if defined(__x86_64__) || defined(_M_X64)
#include <emmintrin.h>
#endif

#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <new>
#include <thread>
#include <vector>

#include "../../include/hydro_gpu.h"
#include "hydro_kernels.cuh"

using hb::cell_index;

struct hydro_gpu_ctx {
  hydro_gpu_cfg cfg;
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  double* A = nullptr;  // current state
  double* B = nullptr;  // column-sweep output
  size_t pitch = 0;
  size_t count = 0;     // doubles per state buffer
  // [0],[1] dt limits, [2] error, [3] dt error, [4] x / y work counters (2 x u32)
  unsigned long long* slots = nullptr;
  hydro_gpu_error last{};
  int seg_x = 0, seg_y = 0, block = 128;
  int band_x = 0, band_y = 0;  // claim-order bands (0 = automatic)
  hb::Geometry geo{};
  hb::Geometry geo_tol{};  // occupancy of the tolerance-mode sweeps
  int math = HYDRO_GPU_MATH_BITWISE;
  hb::TmaMaps maps{};
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  struct Pending { cudaEvent_t a, b; int kind; };
  std::vector<Pending> pending;
  size_t ev_next = 0;
  double ms[5] = {0, 0, 0, 0, 0};   // column sweeps, row sweeps, other, comm phases, fused steps
  long long n[5] = {0, 0, 0, 0, 0};
  // schedule (hydro_gpu_set_schedule): fused steps where they apply
  int schedule = HYDRO_GPU_SCHEDULE_AUTO;
  int seg_xy = 0;
  // AUTO: the current choice, and what it is decided from -- the share of
  // cell updates the last completed runs took by the uniform-window identity
  // (the sweeps' counters, copied into pinned memory at the end of every run)
  bool auto_fused = true;
  unsigned long long* stat_host = nullptr;     // pinned: cumulative counters after the last run
  unsigned long long stat_seen = 0;            // their sum when the choice was last made
  double stat_sweeps = 0;                      // cell-sweeps enqueued since then
  double stat_share = -1.0;                    // the share behind the current choice
  // ... and the device time per step of the last event-bracketed run of each
  // schedule ([0] split, [1] fused; -1 = not measured at the current share)
  cudaEvent_t run_ev[2] = {nullptr, nullptr};
  bool run_pending = false;                    // run_ev bracket a run not yet read
  int run_steps = 0;
  bool run_fused = false;
  double ms_step[2] = {-1.0, -1.0};
  double ms_share[2] = {-1.0, -1.0};
  // CUDA graphs of whole run_sequential calls, one per (steps, timing):
  // the 2*steps+3 launches replay without per-launch CPU and queue gaps.
  struct GraphEntry {
    int steps;
    bool timing;
    bool fused;
    cudaGraphExec_t exec;
    std::vector<Pending> events;  // event pairs recorded inside the graph
  };
  std::vector<GraphEntry> graphs;
  bool use_graphs = true;
  bool capturing = false;         // ev_begin/ev_end use dedicated graph events
  std::vector<cudaEvent_t> graph_events;
  size_t graph_next = 0;
  // peer-memory halo (hydro_gpu_set_halo_peers): own inbox of 2 parities x 2
  // sides, the neighbours' inboxes, IPC mappings to close
  double* inbox = nullptr;
  double* peer_up = nullptr;
  double* peer_dn = nullptr;
  std::vector<void*> ipc_opened;
  // multi-rank slab (hydro_gpu_comm_attach): the NCCL communicator of the
  // row-slab decomposition; hydro_gpu_run then runs the slab schedule
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  // pinned staging ring for pageable host planes (hydro_gpu_upload/download)
  double* stage[2] = {nullptr, nullptr};     // pinned host
  double* dstage[2] = {nullptr, nullptr};    // device (row format), bands
  double* rowstage = nullptr;                // device (row format), the whole grid
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  double* halo_buf = nullptr;                // send/recv blocks of the collective halo
};

namespace {

constexpr int kSlotErr = 2;
constexpr int kSlotDtErr = 3;
constexpr int kSlotCounters = 4;
constexpr int kSlotSkipped = 5;  // [5], [6]: x / y cell updates taken by the uniform-window identity
constexpr int kSlotFused = 7;    // fused step: work counter, finished CTAs (2 x u32)
constexpr int kSlots = 8;

const char* kFieldName[3] = {"rho", "pres", "internal energy"};

int set_err(hydro_gpu_ctx* c, int cat, const char* fmt, ...) {
  if (!c) return cat;
  c->last = hydro_gpu_error{};
  c->last.category = cat;
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(c->last.message, sizeof(c->last.message), fmt, ap);
  va_end(ap);
  return cat;
}

#define CUDA_TRY(ctx, call)                                                        \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return set_err((ctx), HYDRO_GPU_ERR_CUDA, "cuda: %s (%s:%d)", cudaGetErrorString(e_), \
                     __FILE__, __LINE__);                                          \
  } while (0)

bool valid_cfg(const hydro_gpu_cfg* c, char* why, size_t n) {
  if (c->ny < 4 || c->nx < 2) {
    std::snprintf(why, n, "grid interior must be at least 4x4, got %dx%d", c->nx, c->ny);
    return false;
  }
  if (c->wall_lo && c->wall_hi && c->nx < 4) {
    std::snprintf(why, n, "grid interior must be at least 4x4, got %dx%d", c->nx, c->ny);
    return false;
  }
  if (!(c->dx > 0.0) || !(c->dy > 0.0)) {
    std::snprintf(why, n, "cell sizes must be positive");
    return false;
  }
  if (!(c->gamma > 1.0)) {
    std::snprintf(why, n, "gamma must exceed 1");
    return false;
  }
  if (c->bc != HYDRO_GPU_BC_REFLECT && c->bc != HYDRO_GPU_BC_TRANSMIT) {
    std::snprintf(why, n, "unknown boundary kind %d", c->bc);
    return false;
  }
  if (c->flux != HYDRO_GPU_FLUX_HLLC && c->flux != HYDRO_GPU_FLUX_EXACT10) {
    std::snprintf(why, n, "unknown flux kind %d", c->flux);
    return false;
  }
  if (c->row0 < 0 || c->global_nx < c->row0 + c->nx) {
    std::snprintf(why, n, "slab rows [%d, %d) outside a %d-row grid", c->row0,
                  c->row0 + c->nx, c->global_nx);
    return false;
  }
  if (c->global_nx > (1 << 18) - 8 || c->ny > (1 << 18) - 8) {
    std::snprintf(why, n, "grid extent exceeds the 2^18-cell strip limit");
    return false;
  }
  return true;
}

double as_double(unsigned long long bits) {
  double d;
  std::memcpy(&d, &bits, sizeof d);
  return d;
}

// Event bracket for one launch (timing mode only).
void ev_begin(hydro_gpu_ctx* c, cudaEvent_t* a) {
  if (!c->timing) return;
  if (c->capturing) {  // events pre-created by launch_graph
    *a = c->graph_events[c->graph_next++];
    cudaEventRecordWithFlags(*a, c->stream, cudaEventRecordExternal);  // a graph node
    return;
  }
  if (c->ev_next + 2 > c->ev_pool.size()) {
    for (int k = 0; k < 64; ++k) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      c->ev_pool.push_back(e);
    }
  }
  *a = c->ev_pool[c->ev_next++];
  cudaEventRecord(*a, c->stream);
}

void ev_end(hydro_gpu_ctx* c, cudaEvent_t a, int kind) {
  if (!c->timing) return;
  if (c->capturing) {
    cudaEvent_t b = c->graph_events[c->graph_next++];
    cudaEventRecordWithFlags(b, c->stream, cudaEventRecordExternal);
    c->pending.push_back({a, b, kind});
    return;
  }
  cudaEvent_t b = c->ev_pool[c->ev_next++];
  cudaEventRecord(b, c->stream);
  c->pending.push_back({a, b, kind});
}

void harvest(hydro_gpu_ctx* c) {
  for (auto& p : c->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      c->ms[p.kind] += ms;
      c->n[p.kind] += 1;
    } else {
      cudaGetLastError();  // not recorded (e.g. an aborted capture): skip
    }
  }
  c->pending.clear();
  c->ev_next = 0;
}

hb::SweepArgs sweep_args(hydro_gpu_ctx* c, int axis, int step) {
  hb::SweepArgs a{};
  a.pitch = c->pitch;
  a.nx = c->cfg.nx;
  a.ny = c->cfg.ny;
  a.dx = axis == 0 ? c->cfg.dx : c->cfg.dy;
  a.spacing = c->cfg.dx < c->cfg.dy ? c->cfg.dx : c->cfg.dy;  // std::min(dx, dy)
  a.gamma = c->cfg.gamma;
  a.cfl = c->cfg.cfl;
  a.bc = c->cfg.bc;
  a.flux = c->cfg.flux;
  a.wall_lo = c->cfg.wall_lo;
  a.wall_hi = c->cfg.wall_hi;
  a.row0 = c->cfg.row0;
  a.limit_in = c->slots + (step & 1);
  a.limit_out = c->slots + ((step + 1) & 1);
  a.err = c->slots + kSlotErr;
  a.dt_err = c->slots + kSlotDtErr;
  a.counter = reinterpret_cast<unsigned*>(c->slots + kSlotCounters) + axis;
  a.counter_next = reinterpret_cast<unsigned*>(c->slots + kSlotCounters) + (1 - axis);
  a.skipped = c->slots + kSlotSkipped + axis;
  a.step = step;
  if (axis == 0) {
    a.src = c->A;
    a.dst = c->B;
    a.seg = c->seg_x;
    a.band = c->band_x;
  } else {
    a.src = c->B;
    a.dst = c->A;
    a.seg = c->seg_y;
    a.band = c->band_y;
    // rows produced by this step's row sweep feed the neighbours' column
    // sweep of step+1: inbox parity (step+1)&1
    const size_t blk = 8 * c->pitch, par = (size_t)((step + 1) & 1);
    if (c->peer_up) a.halo_up = c->peer_up + (par * 2 + 1) * blk;
    if (c->peer_dn) a.halo_dn = c->peer_dn + (par * 2 + 0) * blk;
  }
  return a;
}

void enqueue_x(hydro_gpu_ctx* c, int step, int explicit_dt, double dt) {
  hb::SweepArgs a = sweep_args(c, 0, step);
  a.explicit_dt = explicit_dt;
  a.dt_value = dt;
  cudaEvent_t e0{};
  ev_begin(c, &e0);
  if (c->math == HYDRO_GPU_MATH_TOLERANCE) hb::launch_sweep_x_tol(a, c->maps, c->geo_tol, c->stream);
  else hb::launch_sweep_x(a, c->maps, c->geo, c->stream);
  hb::launch_ghost_fix(c->B, c->pitch, c->cfg.nx, c->cfg.ny, c->cfg.bc, c->stream);
  ev_end(c, e0, 0);
}

void enqueue_y(hydro_gpu_ctx* c, int step, int explicit_dt, double dt, int want_limit) {
  hb::SweepArgs a = sweep_args(c, 1, step);
  a.explicit_dt = explicit_dt;
  a.dt_value = dt;
  a.want_limit = want_limit;
  cudaEvent_t e0{};
  ev_begin(c, &e0);
  if (c->math == HYDRO_GPU_MATH_TOLERANCE) hb::launch_sweep_y_tol(a, c->maps, c->geo_tol, c->stream);
  else hb::launch_sweep_y(a, c->maps, c->geo, c->stream);
  hb::launch_ghost_row_fix(c->A, c->pitch, c->cfg.nx, c->cfg.ny, c->cfg.bc, c->cfg.wall_hi, c->stream);
  ev_end(c, e0, 1);
}

// One fused step (hydro_fused.cuh): U_a -> U_b in a single launch when
// `a_to_b`, else U_b -> U_a; never the last step of a run.
void enqueue_xy(hydro_gpu_ctx* c, int step, bool a_to_b, bool last) {
  hb::SweepArgs a = sweep_args(c, 0, step);
  a.last_step = last ? 1 : 0;
  a.src = a_to_b ? c->A : c->B;
  a.dst = a_to_b ? c->B : c->A;
  a.dx2 = c->cfg.dy;
  a.want_limit = last ? 0 : 1;  // (the reference computes no dt after its last step)
  a.seg = c->seg_xy;
  a.counter = reinterpret_cast<unsigned*>(c->slots + kSlotFused);
  a.done = a.counter + 1;
  a.counter_next = nullptr;
  {  // rows produced by this step feed the neighbours' column phase of step+1: inbox parity (step+1)&1
    const size_t blk = 8 * c->pitch, par = (size_t)((step + 1) & 1);
    a.halo_up = c->peer_up ? c->peer_up + (par * 2 + 1) * blk : nullptr;
    a.halo_dn = c->peer_dn ? c->peer_dn + (par * 2 + 0) * blk : nullptr;
  }
  const CUtensorMap& ld = a_to_b ? c->maps.fa_load : c->maps.fb_load;
  const CUtensorMap& st = a_to_b ? c->maps.fb_store : c->maps.fa_store;
  cudaEvent_t e0{};
  ev_begin(c, &e0);
  if (c->math == HYDRO_GPU_MATH_TOLERANCE) hb::launch_sweep_xy_tol(a, ld, st, c->geo_tol, c->stream);
  else hb::launch_sweep_xy(a, ld, st, c->geo, c->stream);
  ev_end(c, e0, 4);
}

// The AUTO schedule's choice, remade whenever the stream is idle and a run has
// completed since the last one.  Fused steps stream the state once per step
// but run 8 warps per SM and redo a whole 120-column item when a fast pass
// leaves its range; split sweeps stream it twice with 16 warps and redo
// 32-strip items.  So fused wins on memory-bound flow (most updates
// uniform-window identities), split on dense flow and where a strong front
// keeps forcing redo passes on a small grid.  Two inputs, both from the
// context's own completed runs: the share of uniform-window updates (the
// sweeps' counters) and the event-timed device time per step of each
// schedule.  An untimed schedule is tried once (fused not on dense flow, share
// <= 0.2); a timing is forgotten when the share the other schedule measures
// has moved by more than 0.1 between two of its runs.  (The share alone does not decide for fused: a 256^2 blast is 99%
// uniform windows and 4x slower fused in the bitwise arithmetic.)  The results are bitwise the same either way;
// the first run of a context is fused.
constexpr double kAutoFusedShare = 0.6;
void auto_choose(hydro_gpu_ctx* c) {
  if (c->schedule != HYDRO_GPU_SCHEDULE_AUTO || !c->stat_host) return;
  if (c->stat_sweeps <= 0 && !c->run_pending) return;
  if (cudaStreamQuery(c->stream) != cudaSuccess) {
    cudaGetLastError();  // runs still in flight: keep the choice
    return;
  }
  if (c->stat_sweeps > 0) {
    const unsigned long long cur = c->stat_host[0] + c->stat_host[1];
    const unsigned long long seen = cur >= c->stat_seen ? c->stat_seen : 0;
    c->stat_share = (double)(cur - seen) / c->stat_sweeps;
    c->stat_seen = cur;
    c->stat_sweeps = 0;
  }
  const double share = c->stat_share;
  if (c->run_pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c->run_ev[0], c->run_ev[1]) == cudaSuccess) {
      const int r = c->run_fused ? 1 : 0;
      // the flow has changed since this schedule was last timed (shares are
      // compared per schedule: the two count uniform windows differently):
      // the other schedule's timing is stale
      if (c->ms_step[r] >= 0 && share >= 0 && c->ms_share[r] >= 0 &&
          std::fabs(share - c->ms_share[r]) > 0.1)
        c->ms_step[1 - r] = -1.0;
      c->ms_step[r] = (double)ms / c->run_steps;
      c->ms_share[r] = share;
    } else {
      cudaGetLastError();
    }
    c->run_pending = false;
  }
  const bool by_share = share < 0 || share >= kAutoFusedShare;
  if (c->ms_step[0] >= 0 && c->ms_step[1] >= 0) c->auto_fused = c->ms_step[1] <= c->ms_step[0];
  else if (c->ms_step[1] >= 0) c->auto_fused = false;                                // try split once
  else if (c->ms_step[0] >= 0 && share > 0.2) c->auto_fused = true;                  // try fused once
  else c->auto_fused = by_share;
}

bool fused_ok(const hydro_gpu_ctx* c);

// Event bracket around a run for auto_choose (not around event-instrumented
// runs, whose graphs carry timing nodes).
void auto_bracket_begin(hydro_gpu_ctx* c, int steps) {
  c->run_pending = false;
  if (c->schedule != HYDRO_GPU_SCHEDULE_AUTO || c->timing || steps < 2) return;
  for (int k = 0; k < 2; ++k)
    if (!c->run_ev[k] && cudaEventCreate(&c->run_ev[k]) != cudaSuccess) {
      cudaGetLastError();
      c->run_ev[k] = nullptr;
      return;
    }
  if (cudaEventRecord(c->run_ev[0], c->stream) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  c->run_steps = steps;
  c->run_fused = fused_ok(c);
  c->run_pending = true;
}
void auto_bracket_end(hydro_gpu_ctx* c) {
  if (!c->run_pending) return;
  if (cudaEventRecord(c->run_ev[1], c->stream) != cudaSuccess) {
    cudaGetLastError();
    c->run_pending = false;
  }
}

// Whether a run of this context takes fused steps (HLLC; whole domains and
// row slabs alike: a slab's fused step stores its halo rows into the
// neighbours' inboxes like the split row sweep).
bool fused_ok(const hydro_gpu_ctx* c) {
  const bool want = c->schedule == HYDRO_GPU_SCHEDULE_FUSED ||
                    (c->schedule == HYDRO_GPU_SCHEDULE_AUTO && c->auto_fused);
  // (row slabs with the exact-10 flux stay on the split sweeps)
  return want && (c->cfg.flux == HYDRO_GPU_FLUX_HLLC ||
                  (c->comm == nullptr && !c->peer_up && !c->peer_dn && c->cfg.wall_lo && c->cfg.wall_hi));
}

// wall_bc: x-wall ghost rows; full_bc: also the y-wall columns;
// limit_step >= 0: dt limit of that step into its slot.
void enqueue_prologue(hydro_gpu_ctx* c, int wall_bc, int full_bc, int limit_step) {
  hb::PrologueArgs p{};
  p.u = c->A;
  p.pitch = c->pitch;
  p.nx = c->cfg.nx;
  p.ny = c->cfg.ny;
  p.spacing = c->cfg.dx < c->cfg.dy ? c->cfg.dx : c->cfg.dy;
  p.gamma = c->cfg.gamma;
  p.bc = c->cfg.bc;
  p.wall_lo = wall_bc && c->cfg.wall_lo;
  p.wall_hi = wall_bc && c->cfg.wall_hi;
  p.row0 = c->cfg.row0;
  p.full_bc = full_bc;
  p.want_limit = limit_step >= 0;
  p.step = limit_step < 0 ? 0 : limit_step;
  p.limit_out = c->slots + (p.step & 1);
  p.err = c->slots + kSlotErr;
  p.dt_err = c->slots + kSlotDtErr;
  cudaEvent_t e0{};
  ev_begin(c, &e0);
  if (c->math == HYDRO_GPU_MATH_TOLERANCE) hb::launch_prologue_tol(p, c->stream);
  else hb::launch_prologue(p, c->stream);
  ev_end(c, e0, 2);
}

void enqueue_finish(hydro_gpu_ctx* c) {
  hb::FinishArgs f{};
  f.post_x = c->B;
  f.u = c->A;
  f.pitch = c->pitch;
  f.nx = c->cfg.nx;
  f.ny = c->cfg.ny;
  f.bc = c->cfg.bc;
  f.wall_lo = c->cfg.wall_lo;
  f.wall_hi = c->cfg.wall_hi;
  cudaEvent_t e0{};
  ev_begin(c, &e0);
  hb::launch_finish(f, c->stream);
  ev_end(c, e0, 2);
}

int reset_slots(hydro_gpu_ctx* c) {
  CUDA_TRY(c, cudaMemsetAsync(c->slots, 0xff, 4 * sizeof(unsigned long long), c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->slots + kSlotCounters, 0, sizeof(unsigned long long), c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->slots + kSlotFused, 0, sizeof(unsigned long long), c->stream));
  return 0;
}

void decode(unsigned long long key, hydro_gpu_error* e, bool with_step) {
  *e = hydro_gpu_error{};
  e->step = (int)(key >> 42);
  e->phase = (int)((key >> 40) & 3);
  e->strip = (int)((key >> 22) & 0x3ffff);
  e->loop = (int)((key >> 20) & 3);
  const int k = (int)((key >> 2) & 0x3ffff);
  e->field = (int)(key & 3);
  e->category = e->field == 3 ? HYDRO_GPU_ERR_VALIDATION : HYDRO_GPU_ERR_POSITIVITY;
  char body[200];
  if (e->phase == 0) {
    e->cell = k;  // column j of the failing cell; compute_dt has no strip context
    std::snprintf(body, sizeof body, "%s non-positive at cons_to_prim input",
                  kFieldName[e->field < 3 ? e->field : 0]);
  } else {
    e->cell = k - 2;  // k - kGhost
    const char* sweep = e->phase == 1 ? "column" : "row";
    if (e->field == 3)  // exact-10 mode (exact_riemann.cpp:55-57)
      std::snprintf(body, sizeof body,
                    "%s sweep strip %d: vacuum-generating Riemann states are out of scope", sweep,
                    e->strip);
    else
      std::snprintf(body, sizeof body, "%s sweep strip %d: %s non-positive at %sstrip cell %d",
                    sweep, e->strip, kFieldName[e->field], e->loop == 2 ? "updated " : "",
                    e->cell);
  }
  if (with_step)
    std::snprintf(e->message, sizeof e->message, "step %d: %s", e->step, body);
  else
    std::snprintf(e->message, sizeof e->message, "%s", body);
}

// Synchronises and converts a latched key into a status.
int finish_status(hydro_gpu_ctx* c, bool with_step) {
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  CUDA_TRY(c, cudaGetLastError());
  harvest(c);
  unsigned long long key = 0;
  CUDA_TRY(c, cudaMemcpy(&key, c->slots + kSlotErr, sizeof key, cudaMemcpyDeviceToHost));
  if (key == hb::kNoError) {
    c->last = hydro_gpu_error{};
    return HYDRO_GPU_OK;
  }
  decode(key, &c->last, with_step);
  return c->last.category;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

namespace {

// NCCL, resolved at run time (dlopen of libnccl.so.2 -- in a torch process
// the library torch already loaded): only multi-rank slabs need it.
struct NcclApi {
  bool ok = false;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_unique_id = (decltype(a.get_unique_id))dlsym(h, "ncclGetUniqueId");
    a.comm_init_rank = (decltype(a.comm_init_rank))dlsym(h, "ncclCommInitRank");
    a.all_reduce = (decltype(a.all_reduce))dlsym(h, "ncclAllReduce");
    a.comm_destroy = (decltype(a.comm_destroy))dlsym(h, "ncclCommDestroy");
    a.error_string = (decltype(a.error_string))dlsym(h, "ncclGetErrorString");
    a.ok = a.get_unique_id && a.comm_init_rank && a.all_reduce && a.comm_destroy && a.error_string;
    return a;
  }();
  return api;
}

#define NCCL_TRY(c, expr)                                                                   \
  do {                                                                                      \
    const ncclResult_t r_ = (expr);                                                         \
    if (r_ != ncclSuccess)                                                                  \
      return set_err(c, HYDRO_GPU_ERR_CUDA, "NCCL: %s (%s)", nccl().error_string(r_), #expr); \
  } while (0)

// Two grid rows of all four variables <-> a halo block (the inbox format:
// element (r, v, j) at (4 r + v) pitch + j + kColOff; the row sweep's peer
// stores write it): the state is tiled, so these are small kernels.
void rows_to_block(hydro_gpu_ctx* c, int i0, double* blk) {
  hb::launch_tiles_to_rows(c->A, c->pitch, blk, 0, -1, i0, 2, c->cfg.ny, c->stream);
}
void block_to_rows(hydro_gpu_ctx* c, const double* blk, int i0, double* state = nullptr) {
  hb::launch_rows_to_tiles(blk, 0, state ? state : c->A, c->pitch, -1, i0, 2, c->cfg.ny, c->stream);
}

// The slab's per-step exchange (compute_dt_parallel's min, schedulers.cpp:47-65,
// and the column sweep's InterfaceBuffer, decomposition.hpp:58-79): the step's
// dt limit min-allreduced over the ranks (u64 min: positive doubles order like
// their bits; the allreduce also orders every neighbour's peer-memory halo
// stores of the previous row sweep before this rank reads them), then the
// inbox copied into the ghost rows of `state` (the buffer holding the step's
// input: U_a, or U_b before every second fused step).
int enqueue_exchange(hydro_gpu_ctx* c, int step, double* state) {
  cudaEvent_t e0{};
  ev_begin(c, &e0);
  unsigned long long* lim = c->slots + (step & 1);
  NCCL_TRY(c, nccl().all_reduce(lim, lim, 1, ncclUint64, ncclMin, c->comm, c->stream));
  const size_t blk = 8 * c->pitch, par = (size_t)(step & 1);
  if (!c->cfg.wall_lo) block_to_rows(c, c->inbox + (par * 2 + 0) * blk, -1, state);
  if (!c->cfg.wall_hi) block_to_rows(c, c->inbox + (par * 2 + 1) * blk, c->cfg.nx + 1, state);
  CUDA_TRY(c, cudaGetLastError());
  ev_end(c, e0, 3);
  return HYDRO_GPU_OK;
}

// run_sequential's step order (schedulers.cpp:103-116) on the context: one
// domain, or -- with a communicator attached -- this rank's row slab with the
// per-step exchange and, at the end, the first error over all ranks (u64 min
// of the error slots: the keys order like the reference's reporting order).
int enqueue_run(hydro_gpu_ctx* c, int steps) {
  int rc = reset_slots(c);
  if (rc) return rc;
  const bool slab = c->comm != nullptr;
  enqueue_prologue(c, 1, 0, 0);
  if (slab && (c->peer_up || c->peer_dn)) {
    const size_t blk = 8 * c->pitch;
    if (c->peer_up) rows_to_block(c, 1, c->peer_up + 1 * blk);  // rows 1..2, parity 0
    if (c->peer_dn) rows_to_block(c, c->cfg.nx - 1, c->peer_dn);  // rows nx-1..nx
    CUDA_TRY(c, cudaGetLastError());
  }
  // fused schedule: pairs of fused steps (U_a -> U_b -> U_a) after a split
  // first step when the count is odd; the last one leaves the final ghost
  // bands behind (finish_kernel's job after a split last step)
  int f0 = steps, f1 = steps;  // fused steps [f0, f1)
  if (fused_ok(c) && steps >= 2) {
    f0 = steps % 2;
    f1 = steps;
  }
  for (int s = 0; s < steps; ++s) {
    if (s >= f0 && s < f1) {
      const bool a_to_b = ((s - f0) & 1) == 0;
      if (slab) {
        rc = enqueue_exchange(c, s, a_to_b ? c->A : c->B);
        if (rc) return rc;
      }
      if (s == f0)  // the dt slot the first fused step writes (a split step leaves it set)
        CUDA_TRY(c, cudaMemsetAsync(c->slots + ((s + 1) & 1), 0xff, sizeof(unsigned long long),
                                    c->stream));
      enqueue_xy(c, s, a_to_b, s + 1 == steps);
      continue;
    }
    if (slab) {
      rc = enqueue_exchange(c, s, c->A);
      if (rc) return rc;
    }
    enqueue_x(c, s, 0, 0.0);
    enqueue_y(c, s, 0, 0.0, s + 1 < steps);
  }
  if (f0 == f1) enqueue_finish(c);  // (a fused last step has left the final ghost bands)
  if (c->stat_host)  // the uniform-window counters for the AUTO schedule's next choice
    CUDA_TRY(c, cudaMemcpyAsync(c->stat_host, c->slots + kSlotSkipped, 2 * sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, c->stream));
  if (slab) {
    unsigned long long* keys = c->slots + kSlotErr;  // the error and the pending dt error
    NCCL_TRY(c, nccl().all_reduce(keys, keys, 2, ncclUint64, ncclMin, c->comm, c->stream));
  }
  return HYDRO_GPU_OK;
}

void drop_graphs(hydro_gpu_ctx* c) {
  for (auto& e : c->graphs) cudaGraphExecDestroy(e.exec);
  c->graphs.clear();
  for (auto ev : c->graph_events) cudaEventDestroy(ev);
  c->graph_events.clear();
}

// Captures (once) and launches the whole run as a CUDA graph.  Returns
// false if graphs cannot be used (legacy default stream, capture failure).
bool launch_graph(hydro_gpu_ctx* c, int steps) {
  if (!c->use_graphs || c->stream == nullptr || c->stream == cudaStreamLegacy) return false;
  if (c->timing && !c->pending.empty()) {  // the graph re-records its events
    cudaStreamSynchronize(c->stream);
    harvest(c);
  }
  hydro_gpu_ctx::GraphEntry* entry = nullptr;
  const bool fused = fused_ok(c);
  for (auto& e : c->graphs)
    if (e.steps == steps && e.timing == c->timing && e.fused == fused) entry = &e;
  if (!entry) {
    std::vector<hydro_gpu_ctx::Pending> saved;
    saved.swap(c->pending);
    if (c->timing) {  // two events per phase: prologue, 3 per step, finish, + a memset
      const size_t need = c->graph_events.size() + 2 * (3 * (size_t)steps + 3);
      c->graph_next = c->graph_events.size();
      while (c->graph_events.size() < need) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        c->graph_events.push_back(e);
      }
    }
    if (cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
      cudaGetLastError();
      c->pending.swap(saved);
      return false;
    }
    c->capturing = true;
    const int rc = enqueue_run(c, steps);
    c->capturing = false;
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(c->stream, &graph);
    cudaGraphExec_t exec = nullptr;
    if (rc != 0 || ec != cudaSuccess || !graph ||
        cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      c->pending.swap(saved);
      c->use_graphs = false;
      return false;
    }
    cudaGraphDestroy(graph);
    if (c->graphs.size() >= 8) {  // bounded cache: forget the oldest run length
      cudaGraphExecDestroy(c->graphs.front().exec);
      c->graphs.erase(c->graphs.begin());
    }
    c->graphs.push_back({steps, c->timing, fused, exec, {}});
    entry = &c->graphs.back();
    entry->events.swap(c->pending);
    c->pending.swap(saved);
    // (the first launch would upload the graph: not inside AUTO's event bracket)
    if (cudaGraphUpload(entry->exec, c->stream) != cudaSuccess) cudaGetLastError();
  }
  auto_bracket_begin(c, steps);  // after the capture: device time of the run alone
  if (cudaGraphLaunch(entry->exec, c->stream) != cudaSuccess) {
    cudaGetLastError();
    c->run_pending = false;
    return false;
  }
  auto_bracket_end(c);
  if (c->timing) c->pending.insert(c->pending.end(), entry->events.begin(), entry->events.end());
  return true;
}

}  // namespace

extern "C" {

int hydro_gpu_abi_version(void) { return HYDRO_GPU_ABI_VERSION; }

const char* hydro_gpu_status_string(int s) {
  switch (s) {
    case HYDRO_GPU_OK: return "ok";
    case HYDRO_GPU_ERR_CONFIG: return "config";
    case HYDRO_GPU_ERR_POSITIVITY: return "positivity";
    case HYDRO_GPU_ERR_PROTOCOL: return "protocol";
    case HYDRO_GPU_ERR_TASKGRAPH: return "task-graph";
    case HYDRO_GPU_ERR_EQUIVALENCE: return "equivalence";
    case HYDRO_GPU_ERR_IO: return "io";
    case HYDRO_GPU_ERR_VALIDATION: return "validation";
    case HYDRO_GPU_ERR_CUDA: return "cuda";
  }
  return "unknown";
}

int hydro_gpu_create(const hydro_gpu_cfg* cfg, hydro_gpu_ctx** out) {
  if (!cfg || !out) return HYDRO_GPU_ERR_CONFIG;
  *out = nullptr;
  hydro_gpu_cfg c = *cfg;
  if (c.global_nx <= 0) c.global_nx = c.nx + c.row0;
  char why[160];
  if (!valid_cfg(&c, why, sizeof why)) return HYDRO_GPU_ERR_CONFIG;
  auto* ctx = new (std::nothrow) hydro_gpu_ctx;
  if (!ctx) return HYDRO_GPU_ERR_CUDA;
  ctx->cfg = c;
  if (c.device >= 0) {
    if (cudaSetDevice(c.device) != cudaSuccess) {
      delete ctx;
      return HYDRO_GPU_ERR_CUDA;
    }
  }
  cudaGetDevice(&ctx->device);
  ctx->pitch = hb::pitch_for(c.ny);
  // rows -1..nx+2 plus one padding row read by the column sweep's prefetch
  ctx->count = hb::state_doubles(c.nx, ctx->pitch);  // tiled in 32-row blocks (hb::cell_index)
  const size_t bytes = ctx->count * sizeof(double);
  const size_t bytes_b = bytes;
  if (cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&ctx->A, bytes) != cudaSuccess || cudaMalloc(&ctx->B, bytes_b) != cudaSuccess ||
      cudaMalloc(&ctx->slots, kSlots * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMalloc(&ctx->inbox, 4 * 8 * ctx->pitch * sizeof(double)) != cudaSuccess) {
    hydro_gpu_destroy(ctx);
    cudaGetLastError();
    return HYDRO_GPU_ERR_CUDA;
  }
  ctx->stream = ctx->own_stream;
  if (const char* sch = std::getenv("HYDRO_GPU_SCHEDULE"))  // test / A-B override of the default
    ctx->schedule = std::strcmp(sch, "split") == 0   ? HYDRO_GPU_SCHEDULE_SPLIT
                    : std::strcmp(sch, "fused") == 0 ? HYDRO_GPU_SCHEDULE_FUSED
                                                     : HYDRO_GPU_SCHEDULE_AUTO;
  if (cudaMallocHost(&ctx->stat_host, 2 * sizeof(unsigned long long)) == cudaSuccess) {
    ctx->stat_host[0] = ctx->stat_host[1] = 0;
  } else {
    ctx->stat_host = nullptr;  // AUTO then keeps its first choice
    cudaGetLastError();
  }
  if (hb::query_geometry(&ctx->geo) != 0 || hb::query_geometry_tol(&ctx->geo_tol) != 0 ||
      !hb::make_tma_maps(&ctx->maps, ctx->A, ctx->B, ctx->pitch, c.nx, c.ny)) {
    hydro_gpu_destroy(ctx);
    cudaGetLastError();
    return HYDRO_GPU_ERR_CUDA;
  }
  cudaMemsetAsync(ctx->A, 0, bytes, ctx->stream);
  cudaMemsetAsync(ctx->B, 0, bytes_b, ctx->stream);
  cudaMemsetAsync(ctx->inbox, 0, 4 * 8 * ctx->pitch * sizeof(double), ctx->stream);
  cudaMemsetAsync(ctx->slots, 0xff, 4 * sizeof(unsigned long long), ctx->stream);
  cudaMemsetAsync(ctx->slots + kSlotCounters, 0, 4 * sizeof(unsigned long long), ctx->stream);
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    hydro_gpu_destroy(ctx);
    return HYDRO_GPU_ERR_CUDA;
  }
  *out = ctx;
  return HYDRO_GPU_OK;
}

int hydro_gpu_destroy(hydro_gpu_ctx* ctx) {
  if (!ctx) return HYDRO_GPU_OK;
  DeviceGuard g(ctx->device);
  if (ctx->own_stream) cudaStreamSynchronize(ctx->own_stream);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  drop_graphs(ctx);
  if (ctx->comm) nccl().comm_destroy(ctx->comm);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->A) cudaFree(ctx->A);
  if (ctx->B) cudaFree(ctx->B);
  if (ctx->slots) cudaFree(ctx->slots);
  if (ctx->stat_host) cudaFreeHost(ctx->stat_host);
  for (int k = 0; k < 2; ++k)
    if (ctx->run_ev[k]) cudaEventDestroy(ctx->run_ev[k]);
  for (void* p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
  if (ctx->inbox) cudaFree(ctx->inbox);
  if (ctx->halo_buf) cudaFree(ctx->halo_buf);
  if (ctx->rowstage) cudaFree(ctx->rowstage);
  for (int b = 0; b < 2; ++b) {
    if (ctx->dstage[b]) cudaFree(ctx->dstage[b]);
    if (ctx->stage[b]) cudaFreeHost(ctx->stage[b]);
    if (ctx->stage_ev[b]) cudaEventDestroy(ctx->stage_ev[b]);
  }
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
  return HYDRO_GPU_OK;
}

int hydro_gpu_last_error(const hydro_gpu_ctx* ctx, hydro_gpu_error* out) {
  if (!ctx || !out) return HYDRO_GPU_ERR_CONFIG;
  *out = ctx->last;
  return HYDRO_GPU_OK;
}

int hydro_gpu_use_own_stream(hydro_gpu_ctx* ctx) {
  if (!ctx) return HYDRO_GPU_ERR_CONFIG;
  ctx->stream = ctx->own_stream;
  return HYDRO_GPU_OK;
}

int hydro_gpu_set_stream(hydro_gpu_ctx* ctx, void* s) {
  if (!ctx) return HYDRO_GPU_ERR_CONFIG;
  // CUDA convention: a null handle is the (legacy) default stream.
  ctx->stream = (cudaStream_t)s;
  return HYDRO_GPU_OK;
}

}  // extern "C"

namespace {

// Host transfers.  The device state is tiled (hb::cell_index), so every
// transfer goes through the context's two device staging buffers in bands of
// plane rows: H2D of a band in the Grid2D row format, then a scatter kernel
// into the blocks (and the reverse for downloads), both on the context's
// stream.  Pageable host planes (a Grid2D's std::vectors, grid.hpp:63) are
// staged once more through a pinned two-buffer ring: the host copies of one
// band run on several threads while the DMA of the previous band is in
// flight -- a pageable cudaMemcpy is staged by the driver one buffer at a time.
constexpr size_t kStageBytes = 64u << 20;

bool pageable(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return at.type == cudaMemoryTypeUnregistered;
}

int ensure_stage(hydro_gpu_ctx* c, bool pinned) {
  for (int b = 0; b < 2; ++b) {
    if (!c->dstage[b]) CUDA_TRY(c, cudaMalloc(&c->dstage[b], kStageBytes));
    if (pinned && !c->stage[b]) CUDA_TRY(c, cudaMallocHost(&c->stage[b], kStageBytes));
    if (!c->stage_ev[b]) CUDA_TRY(c, cudaEventCreateWithFlags(&c->stage_ev[b], cudaEventDisableTiming));
  }
  return HYDRO_GPU_OK;
}

// memcpy with non-temporal stores (x86-64: SSE2 is baseline): the staging
// copies stream gigabytes once through the host, and regular stores would
// first read every destination line for ownership -- a third of the copy's
// memory traffic.  Unaligned heads and tails go through memcpy.
void stream_copy(char* dst, const char* src, size_t n) {
#if defined(__x86_64__) || defined(_M_X64)
  static const bool nt = [] {  // HYDRO_GPU_COPY_NT=0: plain memcpy (A/B)
    const char* e = std::getenv("HYDRO_GPU_COPY_NT");
    return !(e && e[0] == '0');
  }();
  if (n < 4096 || !nt) {
    std::memcpy(dst, src, n);
    return;
  }
  const size_t head = (16 - ((uintptr_t)dst & 15)) & 15;
  if (head) {
    std::memcpy(dst, src, head);
    dst += head;
    src += head;
    n -= head;
  }
  const size_t blocks = n / 64;
  for (size_t b = 0; b < blocks; ++b) {
    const __m128i x0 = _mm_loadu_si128((const __m128i*)(src) + 0);
    const __m128i x1 = _mm_loadu_si128((const __m128i*)(src) + 1);
    const __m128i x2 = _mm_loadu_si128((const __m128i*)(src) + 2);
    const __m128i x3 = _mm_loadu_si128((const __m128i*)(src) + 3);
    _mm_stream_si128((__m128i*)(dst) + 0, x0);
    _mm_stream_si128((__m128i*)(dst) + 1, x1);
    _mm_stream_si128((__m128i*)(dst) + 2, x2);
    _mm_stream_si128((__m128i*)(dst) + 3, x3);
    src += 64;
    dst += 64;
  }
  _mm_sfence();
  if (n & 63) std::memcpy(dst, src, n & 63);
#else
  std::memcpy(dst, src, n);
#endif
}

// rows [0, n) of `row_bytes` each, src/dst strides in bytes, on up to 16 threads
void par_copy_rows(char* dst, size_t dst_stride, const char* src, size_t src_stride, size_t n,
                   size_t row_bytes) {
  const size_t total = n * row_bytes;
  static const unsigned cap = [] {  // HYDRO_GPU_COPY_THREADS overrides the default of 16
    const char* e = std::getenv("HYDRO_GPU_COPY_THREADS");
    const int v = e ? std::atoi(e) : 0;
    return v > 0 ? (unsigned)v : 16u;
  }();
  unsigned nt = std::thread::hardware_concurrency();
  nt = nt < 1 ? 1 : (nt > cap ? cap : nt);
  if (total < (4u << 20)) nt = 1;
  // dense rows on both sides (a Grid2D plane <-> the pinned band): one copy
  // per thread
  const bool dense = dst_stride == row_bytes && src_stride == row_bytes;
  auto work = [&](size_t a, size_t b) {
    if (dense) {
      stream_copy(dst + a * row_bytes, src + a * row_bytes, (b - a) * row_bytes);
      return;
    }
    for (size_t r = a; r < b; ++r) stream_copy(dst + r * dst_stride, src + r * src_stride, row_bytes);
  };
  if (nt == 1) {
    work(0, n);
    return;
  }
  std::vector<std::thread> team;
  for (unsigned t = 0; t < nt; ++t) team.emplace_back(work, n * t / nt, n * (t + 1) / nt);
  for (auto& th : team) th.join();
}

// Grid rows [i_lo, i_lo + nrows) of the 4 host planes (hp[v] points at grid
// row i_lo's column -1, rows `row_stride` doubles apart) <-> the tiled state.
// host_sync: pageable planes (staged through pinned memory, synchronous);
// otherwise the copies are only enqueued (pinned planes that stay alive).
int transfer_rows(hydro_gpu_ctx* c, double* const hp[4], size_t row_stride, int i_lo, int nrows,
                  bool up, bool host_sync) {
  const int ny = c->cfg.ny;
  if (!host_sync && i_lo == -1 && nrows == c->cfg.nx + 4) {
    // pinned planes, the whole grid: all DMA through a grid-sized row-format
    // staging buffer, then one conversion kernel per plane -- the copies need
    // no SM, so they overlap other work on the device (e.g. another
    // context's run)
    const size_t plane = (size_t)nrows * (ny + 4);
    if (!c->rowstage) CUDA_TRY(c, cudaMalloc(&c->rowstage, 4 * plane * sizeof(double)));
    // all four planes' copies back to back, the conversions on one side of
    // them: the stream's DMA run is not broken by kernels waiting for SMs
    const size_t rb = (size_t)(ny + 4) * 8;
    if (up) {
      for (int v = 0; v < 4; ++v)
        CUDA_TRY(c, cudaMemcpy2DAsync(c->rowstage + v * plane, rb, hp[v], row_stride * 8, rb,
                                      nrows, cudaMemcpyHostToDevice, c->stream));
      for (int v = 0; v < 4; ++v)
        hb::launch_rows_to_tiles(c->rowstage + v * plane, ny + 4, c->A, c->pitch, v, -1, nrows,
                                 ny, c->stream);
    } else {
      for (int v = 0; v < 4; ++v)
        hb::launch_tiles_to_rows(c->A, c->pitch, c->rowstage + v * plane, ny + 4, v, -1, nrows,
                                 ny, c->stream);
      for (int v = 0; v < 4; ++v)
        CUDA_TRY(c, cudaMemcpy2DAsync(hp[v], row_stride * 8, c->rowstage + v * plane, rb, rb,
                                      nrows, cudaMemcpyDeviceToHost, c->stream));
    }
    CUDA_TRY(c, cudaGetLastError());
    return HYDRO_GPU_OK;
  }
  int rc = ensure_stage(c, host_sync);
  if (rc) return rc;
  const size_t row_bytes = (size_t)(ny + 4) * 8;
  const size_t band = kStageBytes / row_bytes;
  if (band == 0) return set_err(c, HYDRO_GPU_ERR_CONFIG, "rows too long to stage");
  struct Chunk { int v, r0, n; };
  std::vector<Chunk> chunks;
  for (int v = 0; v < 4; ++v)
    for (int r0 = 0; r0 < nrows; r0 += (int)band)
      chunks.push_back({v, r0, (int)std::min<size_t>(band, (size_t)(nrows - r0))});
  auto host = [&](const Chunk& k) { return hp[k.v] + (size_t)k.r0 * row_stride; };
  if (up) {
    for (size_t q = 0; q < chunks.size(); ++q) {
      const int b = (int)(q & 1);
      const Chunk& k = chunks[q];
      const double* src = host(k);
      size_t spitch = row_stride * 8;
      if (host_sync) {  // the pinned buffer's previous DMA is done
        CUDA_TRY(c, cudaEventSynchronize(c->stage_ev[b]));
        par_copy_rows((char*)c->stage[b], row_bytes, (const char*)src, spitch, k.n, row_bytes);
        src = c->stage[b];
        spitch = row_bytes;
      }
      CUDA_TRY(c, cudaMemcpy2DAsync(c->dstage[b], row_bytes, src, spitch, row_bytes, k.n,
                                    cudaMemcpyHostToDevice, c->stream));
      hb::launch_rows_to_tiles(c->dstage[b], ny + 4, c->A, c->pitch, k.v, i_lo + k.r0, k.n, ny,
                               c->stream);
      CUDA_TRY(c, cudaEventRecord(c->stage_ev[b], c->stream));
    }
  } else {
    auto issue = [&](size_t q) -> int {
      const int b = (int)(q & 1);
      const Chunk& k = chunks[q];
      hb::launch_tiles_to_rows(c->A, c->pitch, c->dstage[b], ny + 4, k.v, i_lo + k.r0, k.n, ny,
                               c->stream);
      if (host_sync)
        CUDA_TRY(c, cudaMemcpy2DAsync(c->stage[b], row_bytes, c->dstage[b], row_bytes, row_bytes,
                                      k.n, cudaMemcpyDeviceToHost, c->stream));
      else
        CUDA_TRY(c, cudaMemcpy2DAsync(host(k), row_stride * 8, c->dstage[b], row_bytes, row_bytes,
                                      k.n, cudaMemcpyDeviceToHost, c->stream));
      CUDA_TRY(c, cudaEventRecord(c->stage_ev[b], c->stream));
      return HYDRO_GPU_OK;
    };
    if (!host_sync) {
      for (size_t q = 0; q < chunks.size(); ++q)
        if ((rc = issue(q))) return rc;
      return HYDRO_GPU_OK;
    }
    if ((rc = issue(0))) return rc;
    for (size_t q = 0; q < chunks.size(); ++q) {
      const int b = (int)(q & 1);
      // chunk q+1 may not overwrite the pinned buffer chunk q-1 is copied out of
      if (q + 1 < chunks.size() && (rc = issue(q + 1))) return rc;
      CUDA_TRY(c, cudaEventSynchronize(c->stage_ev[b]));
      const Chunk& k = chunks[q];
      par_copy_rows((char*)host(k), row_stride * 8, (const char*)c->stage[b], row_bytes, k.n, row_bytes);
    }
  }
  if (host_sync) CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return HYDRO_GPU_OK;
}

bool any_pageable(const double* const planes[4]) {
  for (int v = 0; v < 4; ++v)
    if (planes[v] && pageable(planes[v])) return true;
  return false;
}

int check_planes(hydro_gpu_ctx* c, const double* const planes[4], size_t row_stride) {
  if (row_stride < (size_t)c->cfg.ny + 4)
    return set_err(c, HYDRO_GPU_ERR_CONFIG, "row stride %zu below ny+4", row_stride);
  for (int v = 0; v < 4; ++v)
    if (!planes[v]) return set_err(c, HYDRO_GPU_ERR_CONFIG, "null plane %d", v);
  return HYDRO_GPU_OK;
}

}  // namespace

extern "C" {

int hydro_gpu_upload_async(hydro_gpu_ctx* c, const double* const planes[4], size_t row_stride) {
  if (!c || !planes) return HYDRO_GPU_ERR_CONFIG;
  int rc = check_planes(c, planes, row_stride);
  if (rc) return rc;
  DeviceGuard g(c->device);
  return transfer_rows(c, const_cast<double* const*>(planes), row_stride, -1, c->cfg.nx + 4, true,
                       false);
}

int hydro_gpu_upload(hydro_gpu_ctx* c, const double* const planes[4], size_t row_stride) {
  if (!c || !planes) return HYDRO_GPU_ERR_CONFIG;
  int rc = check_planes(c, planes, row_stride);
  if (rc) return rc;
  DeviceGuard g(c->device);
  rc = transfer_rows(c, const_cast<double* const*>(planes), row_stride, -1, c->cfg.nx + 4, true,
                     any_pageable(planes));
  if (rc) return rc;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return HYDRO_GPU_OK;
}

int hydro_gpu_download_async(hydro_gpu_ctx* c, double* const planes[4], size_t row_stride) {
  if (!c || !planes) return HYDRO_GPU_ERR_CONFIG;
  int rc = check_planes(c, planes, row_stride);
  if (rc) return rc;
  DeviceGuard g(c->device);
  return transfer_rows(c, planes, row_stride, -1, c->cfg.nx + 4, false, false);
}

int hydro_gpu_download(hydro_gpu_ctx* c, double* const planes[4], size_t row_stride) {
  if (!c || !planes) return HYDRO_GPU_ERR_CONFIG;
  int rc = check_planes(c, planes, row_stride);
  if (rc) return rc;
  DeviceGuard g(c->device);
  rc = transfer_rows(c, planes, row_stride, -1, c->cfg.nx + 4, false, any_pageable(planes));
  if (rc) return rc;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return HYDRO_GPU_OK;
}

int hydro_gpu_download_rows(hydro_gpu_ctx* c, double* const planes[4], size_t row_stride,
                            int i_lo, int nrows) {
  if (!c || !planes || nrows < 0 || i_lo < -1 || i_lo + nrows > c->cfg.nx + 3)
    return HYDRO_GPU_ERR_CONFIG;
  int rc = check_planes(c, planes, row_stride);
  if (rc) return rc;
  DeviceGuard g(c->device);
  rc = transfer_rows(c, planes, row_stride, i_lo, nrows, false, any_pageable(planes));
  if (rc) return rc;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return HYDRO_GPU_OK;
}

int hydro_gpu_compare(hydro_gpu_ctx* a, hydro_gpu_ctx* b, double* max_rel) {
  if (!a || !b || !max_rel || a->cfg.nx != b->cfg.nx || a->cfg.ny != b->cfg.ny ||
      a->pitch != b->pitch || a->device != b->device)
    return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(a->device);
  CUDA_TRY(a, cudaStreamSynchronize(b->stream));
  unsigned long long* d = nullptr;
  CUDA_TRY(a, cudaMallocAsync(&d, sizeof *d, a->stream));
  CUDA_TRY(a, cudaMemsetAsync(d, 0, sizeof *d, a->stream));
  hb::launch_compare(a->A, b->A, a->pitch, a->cfg.nx, a->cfg.ny, d, a->stream);
  unsigned long long bits = 0;
  CUDA_TRY(a, cudaMemcpyAsync(&bits, d, sizeof bits, cudaMemcpyDeviceToHost, a->stream));
  CUDA_TRY(a, cudaFreeAsync(d, a->stream));
  CUDA_TRY(a, cudaStreamSynchronize(a->stream));
  *max_rel = as_double(bits);
  return HYDRO_GPU_OK;
}

int hydro_gpu_init_case(hydro_gpu_ctx* c, int case_id, uint64_t seed) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  if (case_id < 0 || case_id > 5) return set_err(c, HYDRO_GPU_ERR_CONFIG, "unknown case %d", case_id);
  DeviceGuard g(c->device);
  CUDA_TRY(c, cudaMemsetAsync(c->A, 0, c->count * sizeof(double), c->stream));
  hb::InitArgs a{};
  a.u = c->A;
  a.pitch = c->pitch;
  a.nx = c->cfg.nx;
  a.ny = c->cfg.ny;
  a.global_nx = c->cfg.global_nx;
  a.row0 = c->cfg.row0;
  a.case_id = case_id;
  a.gamma = c->cfg.gamma;
  a.dx = c->cfg.dx;
  a.dy = c->cfg.dy;
  a.seed = seed;
  hb::launch_init(a, c->stream);
  CUDA_TRY(c, cudaGetLastError());
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return HYDRO_GPU_OK;
}


int hydro_gpu_run_async(hydro_gpu_ctx* c, int steps) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  if (steps <= 0) return HYDRO_GPU_OK;
  if (steps > HYDRO_GPU_MAX_STEPS)
    return set_err(c, HYDRO_GPU_ERR_CONFIG, "more than %d steps in one call", HYDRO_GPU_MAX_STEPS);
  DeviceGuard g(c->device);
  auto_choose(c);
  c->stat_sweeps += 2.0 * steps * (double)c->cfg.nx * (double)c->cfg.ny;
  if (steps >= 2 && launch_graph(c, steps)) {
    CUDA_TRY(c, cudaGetLastError());
    return HYDRO_GPU_OK;
  }
  auto_bracket_begin(c, steps);
  int rc = enqueue_run(c, steps);
  if (rc) return rc;
  auto_bracket_end(c);
  CUDA_TRY(c, cudaGetLastError());
  return HYDRO_GPU_OK;
}

int hydro_gpu_sync(hydro_gpu_ctx* c) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  return finish_status(c, true);
}

int hydro_gpu_run(hydro_gpu_ctx* c, int steps, double* last_dt) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  if (steps < 0) return set_err(c, HYDRO_GPU_ERR_CONFIG, "negative step count");
  if (steps == 0) return HYDRO_GPU_OK;
  if (steps > HYDRO_GPU_MAX_STEPS)
    return set_err(c, HYDRO_GPU_ERR_CONFIG, "more than %d steps in one call", HYDRO_GPU_MAX_STEPS);
  DeviceGuard g(c->device);
  int rc = hydro_gpu_run_async(c, steps);
  if (rc) return rc;
  rc = finish_status(c, true);
  if (rc == HYDRO_GPU_OK && last_dt) {
    unsigned long long bits = 0;
    CUDA_TRY(c, cudaMemcpy(&bits, c->slots + ((steps - 1) & 1), sizeof bits,
                           cudaMemcpyDeviceToHost));
    *last_dt = c->cfg.cfl * as_double(bits);  // dt = model.cfl * limit (:241)
  }
  return rc;
}

int hydro_gpu_advance(hydro_gpu_ctx* c, double dt) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  int rc = reset_slots(c);
  if (rc) return rc;
  enqueue_prologue(c, 1, 0, -1);
  enqueue_x(c, 0, 1, dt);
  enqueue_y(c, 0, 1, dt, 0);
  enqueue_finish(c);
  return finish_status(c, false);
}

int hydro_gpu_compute_dt(hydro_gpu_ctx* c, double* dt) {
  if (!c || !dt) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  int rc = reset_slots(c);
  if (rc) return rc;
  enqueue_prologue(c, 0, 0, 0);
  rc = finish_status(c, false);
  if (rc) return rc;
  unsigned long long bits = 0;
  CUDA_TRY(c, cudaMemcpy(&bits, c->slots, sizeof bits, cudaMemcpyDeviceToHost));
  *dt = c->cfg.cfl * as_double(bits);
  return HYDRO_GPU_OK;
}

int hydro_gpu_run_until(hydro_gpu_ctx* c, double t_end, int* steps_out) {
  if (!c || !steps_out) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  *steps_out = 0;
  double t = 0.0;
  int steps = 0;
  int rc = reset_slots(c);
  if (rc) return rc;
  bool started = false;
  while (t < t_end) {  // schedulers.cpp:118-138
    if (steps == HYDRO_GPU_MAX_STEPS) {  // the error keys' step field is exhausted
      enqueue_finish(c);
      rc = finish_status(c, true);
      *steps_out = steps;
      return rc ? rc : set_err(c, HYDRO_GPU_ERR_CONFIG, "run_until stopped after %d steps",
                               HYDRO_GPU_MAX_STEPS);
    }
    if (!started) {
      enqueue_prologue(c, 1, 0, 0);
      started = true;
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    unsigned long long sl[4];
    CUDA_TRY(c, cudaMemcpy(sl, c->slots, sizeof sl, cudaMemcpyDeviceToHost));
    unsigned long long key = sl[kSlotErr] < sl[kSlotDtErr] ? sl[kSlotErr] : sl[kSlotDtErr];
    if (key != hb::kNoError) {
      *steps_out = steps;
      decode(key, &c->last, true);
      return c->last.category;
    }
    double dt = c->cfg.cfl * as_double(sl[steps & 1]);
    if (t + dt > t_end) dt = t_end - t;
    if (!(dt > 0.0) || t + dt == t) {
      // the reference applied the boundary before breaking out
      enqueue_prologue(c, 1, 1, -1);
      rc = finish_status(c, true);
      *steps_out = steps;
      return rc;
    }
    enqueue_x(c, steps, 1, dt);
    enqueue_y(c, steps, 1, dt, 1);
    t += dt;
    ++steps;
  }
  if (steps > 0) enqueue_finish(c);
  rc = finish_status(c, true);
  *steps_out = steps;
  return rc;
}

// ---- slab phases -----------------------------------------------------------

int hydro_gpu_slab_prologue(hydro_gpu_ctx* c, int step) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  int rc = reset_slots(c);
  if (rc) return rc;
  enqueue_prologue(c, 1, 0, step);
  CUDA_TRY(c, cudaGetLastError());
  return HYDRO_GPU_OK;
}

int hydro_gpu_limit_slot(hydro_gpu_ctx* c, int step, double** p) {
  if (!c || !p) return HYDRO_GPU_ERR_CONFIG;
  *p = reinterpret_cast<double*>(c->slots + (step & 1));
  return HYDRO_GPU_OK;
}

int hydro_gpu_error_slot(hydro_gpu_ctx* c, uint64_t** p) {
  if (!c || !p) return HYDRO_GPU_ERR_CONFIG;
  *p = reinterpret_cast<uint64_t*>(c->slots + kSlotErr);
  return HYDRO_GPU_OK;
}

int hydro_gpu_halo(hydro_gpu_ctx* c, double** send_lo, double** send_hi, double** recv_lo,
                   double** recv_hi, size_t* count) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  const size_t blk = 8 * c->pitch;
  if (!c->halo_buf) CUDA_TRY(c, cudaMalloc(&c->halo_buf, 4 * blk * sizeof(double)));
  if (send_lo) *send_lo = c->halo_buf;            // rows 1..2
  if (send_hi) *send_hi = c->halo_buf + blk;      // rows nx-1..nx
  if (recv_lo) *recv_lo = c->halo_buf + 2 * blk;  // rows -1..0
  if (recv_hi) *recv_hi = c->halo_buf + 3 * blk;  // rows nx+1..nx+2
  if (count) *count = blk;
  return HYDRO_GPU_OK;
}

int hydro_gpu_slab_halo_pack(hydro_gpu_ctx* c) {
  if (!c || !c->halo_buf) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  const size_t blk = 8 * c->pitch;
  rows_to_block(c, 1, c->halo_buf);
  rows_to_block(c, c->cfg.nx - 1, c->halo_buf + blk);
  CUDA_TRY(c, cudaGetLastError());
  return HYDRO_GPU_OK;
}

int hydro_gpu_slab_halo_unpack(hydro_gpu_ctx* c) {
  if (!c || !c->halo_buf) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  const size_t blk = 8 * c->pitch;
  if (!c->cfg.wall_lo) block_to_rows(c, c->halo_buf + 2 * blk, -1);
  if (!c->cfg.wall_hi) block_to_rows(c, c->halo_buf + 3 * blk, c->cfg.nx + 1);
  CUDA_TRY(c, cudaGetLastError());
  return HYDRO_GPU_OK;
}

int hydro_gpu_inbox(hydro_gpu_ctx* c, double** inbox, size_t* count) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  if (inbox) *inbox = c->inbox;
  if (count) *count = 8 * c->pitch;
  return HYDRO_GPU_OK;
}

int hydro_gpu_inbox_ipc_handle(hydro_gpu_ctx* c, void* handle64) {
  if (!c || !handle64) return HYDRO_GPU_ERR_CONFIG;
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  DeviceGuard g(c->device);
  cudaIpcMemHandle_t h;
  CUDA_TRY(c, cudaIpcGetMemHandle(&h, c->inbox));
  std::memcpy(handle64, &h, sizeof h);
  return HYDRO_GPU_OK;
}

int hydro_gpu_ipc_open(hydro_gpu_ctx* c, const void* handle64, double** peer_inbox) {
  if (!c || !handle64 || !peer_inbox) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof h);
  void* p = nullptr;
  CUDA_TRY(c, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  c->ipc_opened.push_back(p);
  *peer_inbox = static_cast<double*>(p);
  return HYDRO_GPU_OK;
}

int hydro_gpu_set_halo_peers(hydro_gpu_ctx* c, double* upper_inbox, double* lower_inbox) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  if ((upper_inbox && c->cfg.wall_lo) || (lower_inbox && c->cfg.wall_hi))
    return set_err(c, HYDRO_GPU_ERR_CONFIG, "a physical wall has no halo neighbour");
  c->peer_up = upper_inbox;
  c->peer_dn = lower_inbox;
  return HYDRO_GPU_OK;
}

int hydro_gpu_comm_unique_id(void* id128) {
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
  if (!id128) return HYDRO_GPU_ERR_CONFIG;
  if (!nccl().ok) return HYDRO_GPU_ERR_CUDA;
  ncclUniqueId id;
  if (nccl().get_unique_id(&id) != ncclSuccess) return HYDRO_GPU_ERR_CUDA;
  std::memcpy(id128, &id, sizeof id);
  return HYDRO_GPU_OK;
}

int hydro_gpu_comm_attach(hydro_gpu_ctx* c, const void* id128, int nranks, int rank) {
  if (!c || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return HYDRO_GPU_ERR_CONFIG;
  if (!nccl().ok) return set_err(c, HYDRO_GPU_ERR_CUDA, "libnccl.so.2 not loadable");
  if (nranks > 1 && ((!c->cfg.wall_lo && !c->peer_up) || (!c->cfg.wall_hi && !c->peer_dn)))
    return set_err(c, HYDRO_GPU_ERR_CONFIG,
                   "the slab's halo neighbours must be mapped first (hydro_gpu_set_halo_peers)");
  DeviceGuard g(c->device);
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclComm_t comm = nullptr;
  NCCL_TRY(c, nccl().comm_init_rank(&comm, nranks, id, rank));
  if (c->comm) nccl().comm_destroy(c->comm);
  c->comm = comm;
  c->nranks = nranks;
  c->rank = rank;
  drop_graphs(c);  // hydro_gpu_run now runs the slab schedule
  return HYDRO_GPU_OK;
}

int hydro_gpu_slab_halo_out(hydro_gpu_ctx* c, int step) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  const size_t blk = 8 * c->pitch, par = (size_t)(step & 1);
  if (c->peer_up) rows_to_block(c, 1, c->peer_up + (par * 2 + 1) * blk);
  if (c->peer_dn) rows_to_block(c, c->cfg.nx - 1, c->peer_dn + (par * 2 + 0) * blk);
  CUDA_TRY(c, cudaGetLastError());
  return HYDRO_GPU_OK;
}

int hydro_gpu_slab_inbox_in(hydro_gpu_ctx* c, int step) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  const size_t blk = 8 * c->pitch, par = (size_t)(step & 1);
  if (!c->cfg.wall_lo) block_to_rows(c, c->inbox + (par * 2 + 0) * blk, -1);  // ghost rows -1..0
  if (!c->cfg.wall_hi) block_to_rows(c, c->inbox + (par * 2 + 1) * blk, c->cfg.nx + 1);
  CUDA_TRY(c, cudaGetLastError());
  return HYDRO_GPU_OK;
}

int hydro_gpu_slab_sweep_x(hydro_gpu_ctx* c, int step) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  enqueue_x(c, step, 0, 0.0);
  CUDA_TRY(c, cudaGetLastError());
  return HYDRO_GPU_OK;
}

int hydro_gpu_slab_sweep_y(hydro_gpu_ctx* c, int step) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  enqueue_y(c, step, 0, 0.0, 1);
  CUDA_TRY(c, cudaGetLastError());
  return HYDRO_GPU_OK;
}

// Run bookkeeping of a caller that drives the slab's steps itself
// (hydro_gpu_group): remakes the AUTO schedule's choice, counts the run's
// sweeps and says whether the run takes fused steps.
int hydro_gpu_slab_run_begin(hydro_gpu_ctx* c, int steps, int* fused) {
  if (!c || !fused) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  auto_choose(c);
  c->stat_sweeps += 2.0 * steps * (double)c->cfg.nx * (double)c->cfg.ny;
  *fused = fused_ok(c) ? 1 : 0;
  return HYDRO_GPU_OK;
}

// One fused step of a slab whose steps are driven from outside: the inbox
// copied into the ghost rows of the step's input buffer (halo != 0), then the
// step.  phase 0: U_a -> U_b, 1: U_b -> U_a; first: the run's first fused
// step; last: the run's last step.
int hydro_gpu_slab_step_xy(hydro_gpu_ctx* c, int step, int phase, int first, int last, int halo) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  double* state = phase == 0 ? c->A : c->B;
  if (halo) {
    const size_t blk = 8 * c->pitch, par = (size_t)(step & 1);
    if (!c->cfg.wall_lo) block_to_rows(c, c->inbox + (par * 2 + 0) * blk, -1, state);
    if (!c->cfg.wall_hi) block_to_rows(c, c->inbox + (par * 2 + 1) * blk, c->cfg.nx + 1, state);
  }
  if (first)
    CUDA_TRY(c, cudaMemsetAsync(c->slots + ((step + 1) & 1), 0xff, sizeof(unsigned long long),
                                c->stream));
  enqueue_xy(c, step, phase == 0, last != 0);
  CUDA_TRY(c, cudaGetLastError());
  return HYDRO_GPU_OK;
}

// End of such a run: the final ghost bands after a split last step, and the
// uniform-window counters for the AUTO schedule's next choice.
int hydro_gpu_slab_run_end(hydro_gpu_ctx* c, int fused_last) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  if (!fused_last) enqueue_finish(c);
  if (c->stat_host)
    CUDA_TRY(c, cudaMemcpyAsync(c->stat_host, c->slots + kSlotSkipped, 2 * sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaGetLastError());
  return HYDRO_GPU_OK;
}

int hydro_gpu_slab_finish(hydro_gpu_ctx* c) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  enqueue_finish(c);
  CUDA_TRY(c, cudaGetLastError());
  return HYDRO_GPU_OK;
}

int hydro_gpu_decode_error(hydro_gpu_ctx* c, uint64_t key, hydro_gpu_error* out) {
  if (!c || !out) return HYDRO_GPU_ERR_CONFIG;
  if (key == hb::kNoError) {
    *out = hydro_gpu_error{};
    return HYDRO_GPU_OK;
  }
  decode(key, out, true);
  c->last = *out;
  return out->category;
}

// ---- instrumentation ---------------------------------------------------------

int hydro_gpu_set_timing(hydro_gpu_ctx* c, int on) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  c->timing = on != 0;
  return HYDRO_GPU_OK;
}

int hydro_gpu_kernel_times(hydro_gpu_ctx* c, double* ms_x, double* ms_y, double* ms_o,
                           long long* n_x, long long* n_y, long long* n_o) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  harvest(c);
  if (ms_x) *ms_x = c->ms[0];
  if (ms_y) *ms_y = c->ms[1];
  if (ms_o) *ms_o = c->ms[2];
  if (n_x) *n_x = c->n[0];
  if (n_y) *n_y = c->n[1];
  if (n_o) *n_o = c->n[2];
  return HYDRO_GPU_OK;
}

int hydro_gpu_reset_counters(hydro_gpu_ctx* c) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  cudaStreamSynchronize(c->stream);
  c->pending.clear();
  c->ev_next = 0;
  for (int k = 0; k < 5; ++k) {
    c->ms[k] = 0;
    c->n[k] = 0;
  }
  CUDA_TRY(c, cudaMemset(c->slots + kSlotSkipped, 0, 2 * sizeof(unsigned long long)));
  if (c->stat_host) c->stat_host[0] = c->stat_host[1] = 0;
  c->stat_seen = 0;
  c->stat_sweeps = 0;
  c->run_pending = false;
  return HYDRO_GPU_OK;
}

int hydro_gpu_skipped(hydro_gpu_ctx* c, uint64_t* x, uint64_t* y) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  unsigned long long v[2] = {0, 0};
  CUDA_TRY(c, cudaMemcpy(v, c->slots + kSlotSkipped, sizeof v, cudaMemcpyDeviceToHost));
  if (x) *x = v[0];
  if (y) *y = v[1];
  return HYDRO_GPU_OK;
}

int hydro_gpu_fused_times(hydro_gpu_ctx* c, double* ms, long long* n) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  harvest(c);
  if (ms) *ms = c->ms[4];
  if (n) *n = c->n[4];
  return HYDRO_GPU_OK;
}

int hydro_gpu_schedule_choice(hydro_gpu_ctx* c, int* fused, double* share) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  if (fused) *fused = fused_ok(c) ? 1 : 0;
  if (share) *share = c->stat_share;
  return HYDRO_GPU_OK;
}

int hydro_gpu_set_schedule(hydro_gpu_ctx* c, int schedule, int seg) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  if ((schedule != HYDRO_GPU_SCHEDULE_SPLIT && schedule != HYDRO_GPU_SCHEDULE_FUSED &&
       schedule != HYDRO_GPU_SCHEDULE_AUTO) || seg < 0)
    return set_err(c, HYDRO_GPU_ERR_CONFIG, "unknown schedule");
  if (schedule != c->schedule || seg != c->seg_xy) drop_graphs(c);
  c->schedule = schedule;
  c->seg_xy = seg;
  return HYDRO_GPU_OK;
}

int hydro_gpu_comm_times(hydro_gpu_ctx* c, double* ms, long long* n) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  harvest(c);
  if (ms) *ms = c->ms[3];
  if (n) *n = c->n[3];
  return HYDRO_GPU_OK;
}

int hydro_gpu_tune(hydro_gpu_ctx* c, int seg_x, int seg_y, int block) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  if (seg_x < 0 || seg_y < 0 || (block != 0 && block != 128))
    return set_err(c, HYDRO_GPU_ERR_CONFIG, "bad launch geometry");
  c->seg_x = seg_x;
  c->seg_y = seg_y;
  drop_graphs(c);  // launch geometry is baked into captured graphs
  return HYDRO_GPU_OK;
}

int hydro_gpu_tune_order(hydro_gpu_ctx* c, int band_x, int band_y) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  c->band_x = band_x;
  c->band_y = band_y;
  drop_graphs(c);
  return HYDRO_GPU_OK;
}

int hydro_gpu_set_math(hydro_gpu_ctx* c, int math) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  if (math != HYDRO_GPU_MATH_BITWISE && math != HYDRO_GPU_MATH_TOLERANCE)
    return set_err(c, HYDRO_GPU_ERR_CONFIG, "unknown math mode");
  if (math != c->math) drop_graphs(c);  // the sweep kernels are baked into captured graphs
  c->math = math;
  return HYDRO_GPU_OK;
}

int hydro_gpu_row_audit(hydro_gpu_ctx* c, uint64_t* row_hashes, double* row_sums) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  DeviceGuard g(c->device);
  const size_t n = 4 * (size_t)c->cfg.nx;
  unsigned long long* dh = nullptr;
  double* ds = nullptr;
  CUDA_TRY(c, cudaMallocAsync(&dh, n * sizeof(unsigned long long), c->stream));
  CUDA_TRY(c, cudaMallocAsync(&ds, n * sizeof(double), c->stream));
  hb::launch_row_audit(c->A, c->pitch, c->cfg.nx, c->cfg.ny, dh, ds, c->stream);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && row_hashes)
    e = cudaMemcpyAsync(row_hashes, dh, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                        c->stream);
  if (e == cudaSuccess && row_sums)
    e = cudaMemcpyAsync(row_sums, ds, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream);
  cudaFreeAsync(dh, c->stream);
  cudaFreeAsync(ds, c->stream);
  CUDA_TRY(c, e);
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return HYDRO_GPU_OK;
}

int hydro_gpu_state_hash(hydro_gpu_ctx* c, uint64_t* out) {
  if (!c || !out) return HYDRO_GPU_ERR_CONFIG;
  std::vector<uint64_t> h(4 * (size_t)c->cfg.nx);
  const int rc = hydro_gpu_row_audit(c, h.data(), nullptr);
  if (rc) return rc;
  *out = hydro_combine_row_hashes(h.data(), h.size());
  return HYDRO_GPU_OK;
}

int hydro_gpu_totals(hydro_gpu_ctx* c, double out[4]) {
  if (!c || !out) return HYDRO_GPU_ERR_CONFIG;
  const int nx = c->cfg.nx;
  std::vector<double> s(4 * (size_t)nx);
  const int rc = hydro_gpu_row_audit(c, nullptr, s.data());
  if (rc) return rc;
  const double vol = c->cfg.dx * c->cfg.dy;
  for (int v = 0; v < 4; ++v) out[v] = vol * hydro_pairwise_sum(s.data() + (size_t)v * nx, nx);
  return HYDRO_GPU_OK;
}

int hydro_gpu_math_selftest(int op, const double* a, const double* b, double* fast,
                            double* exact, int* in_range, size_t n) {
  if (op < 0 || op > 5 || !a || !fast || !exact || !in_range) return HYDRO_GPU_ERR_CONFIG;
  double *da = nullptr, *db = nullptr, *df = nullptr, *dr = nullptr;
  int* dk = nullptr;
  const size_t bytes = n * sizeof(double);
  int rc = HYDRO_GPU_OK;
  if (cudaMalloc(&da, bytes) || cudaMalloc(&db, bytes) || cudaMalloc(&df, bytes) ||
      cudaMalloc(&dr, bytes) || cudaMalloc(&dk, n * sizeof(int))) {
    rc = HYDRO_GPU_ERR_CUDA;
  } else {
    cudaMemcpy(da, a, bytes, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b ? b : a, bytes, cudaMemcpyHostToDevice);
    hb::launch_math_selftest(op, da, db, df, dr, dk, n, 0);
    if (cudaDeviceSynchronize() != cudaSuccess) rc = HYDRO_GPU_ERR_CUDA;
    cudaMemcpy(fast, df, bytes, cudaMemcpyDeviceToHost);
    cudaMemcpy(exact, dr, bytes, cudaMemcpyDeviceToHost);
    cudaMemcpy(in_range, dk, n * sizeof(int), cudaMemcpyDeviceToHost);
  }
  cudaFree(da);
  cudaFree(db);
  cudaFree(df);
  cudaFree(dr);
  cudaFree(dk);
  cudaGetLastError();
  return rc;
}

int hydro_gpu_col_offset(void) { return hb::kColOff; }

int hydro_gpu_state(hydro_gpu_ctx* c, double** p, size_t* pitch) {
  if (!c) return HYDRO_GPU_ERR_CONFIG;
  if (p) *p = c->A;
  if (pitch) *pitch = c->pitch;
  return HYDRO_GPU_OK;
}

}  // extern "C"
