// hydro_group.cu -- one host thread driving a row-slab decomposition over
// several GPUs (the context the reference's single-threaded
// driver holds for n_gpus > 1).
//
// Built entirely on the per-device C-ABI: one hydro_gpu_ctx per slab (its own
// device and stream), the peer-memory halo of hydro_gpu_set_halo_peers with
// plain device pointers (cudaDeviceEnablePeerAccess, no IPC), and the dt
// min across slabs as a one-warp kernel per device that reads every slab's
// limit slot over NVLink -- the single-process twin of the torch.distributed
// driver (paper_2106_13465_b200/slab.py, NCCL min-allreduce) and of
// compute_dt_parallel's slot min (proj/src/schedulers.cpp:47-65, paths
// relative to /root/reference/).
//
// Ordering is stream/event order only, no kernel waits on another device.
// Per step every slab records an event after its row sweep; the leader slab's
// stream (slab 0) waits on all of them, runs the dt-min kernel -- it reads
// every slab's limit slot over NVLink and writes the minimum into all of
// them -- and records one event that every other slab's stream waits on
// before copying its inbox into its ghost rows and running its sweeps: 2(N-1)
// cross-stream waits per step instead of N(N-1).  That join orders (a) each
// neighbour's peer stores of step s-1 before the inbox copy of step s, (b)
// every slot read and write of step s before any slab's row sweep of step s+1
// rewrites that parity, and (c) the inbox copy of step s before a neighbour's
// row sweep of step s+1 rewrites that parity.  A whole run is captured once
// per step count as one (multi-device) CUDA graph from the leader's stream
// and replayed, so a run costs O(1) host calls.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/hydro_gpu.h"
#include "hydro_kernels.cuh"

namespace {

constexpr int kMaxSlabs = 64;

struct SlotTable {
  unsigned long long* slot[kMaxSlabs];
  int n;
};

// Every slot = min over slabs of the step's dt limit (positive doubles order
// like their bits; a slab without cells contributes the empty sentinel ~0).
__global__ void group_limit_min_kernel(SlotTable t) {
  unsigned long long v = ~0ull;
  for (int k = threadIdx.x; k < t.n; k += 32) {
    const unsigned long long x = *(volatile const unsigned long long*)t.slot[k];
    v = x < v ? x : v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  __syncwarp();
  for (int k = threadIdx.x; k < t.n; k += 32) *(volatile unsigned long long*)t.slot[k] = v;
}

struct Guard {
  int prev = -1;
  explicit Guard(int dev) {
    cudaGetDevice(&prev);
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~Guard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

struct hydro_gpu_group {
  hydro_gpu_cfg cfg{};
  int n = 0;
  std::vector<int> device;
  std::vector<int> row0, rows;
  std::vector<hydro_gpu_ctx*> ctx;
  std::vector<cudaStream_t> stream;
  std::vector<cudaEvent_t> done;
  cudaEvent_t lead = nullptr;  // the leader's dt-min of the step is done
  // captured runs, one per (step count, schedule) (bounded cache; the key is
  // 2 * steps + fused)
  std::vector<std::pair<int, cudaGraphExec_t>> graphs;
  bool fused = false;  // the current run takes fused steps (every slab agrees)
  bool use_graphs = true;
  int math = HYDRO_GPU_MATH_BITWISE;
  hydro_gpu_error last{};
};

namespace {

int fail(hydro_gpu_group* g, int cat, const char* msg) {
  g->last = hydro_gpu_error{};
  g->last.category = cat;
  std::snprintf(g->last.message, sizeof g->last.message, "%s", msg);
  return cat;
}

int cuda_fail(hydro_gpu_group* g, cudaError_t e) {
  cudaGetLastError();
  return fail(g, HYDRO_GPU_ERR_CUDA, cudaGetErrorString(e));
}

#define GROUP_CUDA(g, call)                      \
  do {                                           \
    const cudaError_t e_ = (call);               \
    if (e_ != cudaSuccess) return cuda_fail(g, e_); \
  } while (0)

// A slab's status: keep its message as the group's.
int slab_rc(hydro_gpu_group* g, int k, int rc) {
  if (rc) hydro_gpu_last_error(g->ctx[k], &g->last);
  return rc;
}

void drop_graphs(hydro_gpu_group* g) {
  for (auto& e : g->graphs) cudaGraphExecDestroy(e.second);
  g->graphs.clear();
}

void destroy(hydro_gpu_group* g) {
  if (!g->device.empty()) {
    Guard d(g->device[0]);
    drop_graphs(g);
    if (g->lead) cudaEventDestroy(g->lead);
  }
  for (int k = 0; k < (int)g->ctx.size(); ++k) {
    Guard d(g->device[k]);
    if (g->ctx[k]) hydro_gpu_destroy(g->ctx[k]);
    if (k < (int)g->done.size() && g->done[k]) cudaEventDestroy(g->done[k]);
    if (k < (int)g->stream.size() && g->stream[k]) cudaStreamDestroy(g->stream[k]);
  }
  delete g;
}

// The step's join: the leader waits for every slab's row sweep of the
// previous step, takes the min of all limit slots of `step` into all of them,
// and every other slab waits for that.
int enqueue_limit_min(hydro_gpu_group* g, int step) {
  SlotTable t{};
  t.n = g->n;
  for (int k = 0; k < g->n; ++k) {
    double* p = nullptr;
    hydro_gpu_limit_slot(g->ctx[k], step, &p);
    t.slot[k] = reinterpret_cast<unsigned long long*>(p);
  }
  for (int k = 1; k < g->n; ++k) {
    Guard d(g->device[k]);
    GROUP_CUDA(g, cudaEventRecord(g->done[k], g->stream[k]));
  }
  Guard d0(g->device[0]);
  for (int k = 1; k < g->n; ++k) GROUP_CUDA(g, cudaStreamWaitEvent(g->stream[0], g->done[k], 0));
  group_limit_min_kernel<<<1, 32, 0, g->stream[0]>>>(t);
  GROUP_CUDA(g, cudaGetLastError());
  GROUP_CUDA(g, cudaEventRecord(g->lead, g->stream[0]));
  for (int k = 1; k < g->n; ++k) {
    Guard d(g->device[k]);
    GROUP_CUDA(g, cudaStreamWaitEvent(g->stream[k], g->lead, 0));
  }
  return HYDRO_GPU_OK;
}

// run_sequential over the slabs: the reference's per-step order with the dt
// min and the halo between the slabs' sweeps (see the file comment).
int enqueue_group_run(hydro_gpu_group* g, int steps) {
  const bool halo = g->n > 1;
  for (int k = 0; k < g->n; ++k) {
    int rc = hydro_gpu_slab_prologue(g->ctx[k], 0);
    if (!rc && halo) rc = hydro_gpu_slab_halo_out(g->ctx[k], 0);
    if (rc) return slab_rc(g, k, rc);
  }
  // fused schedule (hydro_fused.cuh): pairs of fused steps after one split
  // step when the count is odd, like hydro_gpu_run
  const int f0 = g->fused && steps >= 2 ? steps % 2 : steps;
  for (int s = 0; s < steps; ++s) {
    int rc = enqueue_limit_min(g, s);
    if (rc) return rc;
    for (int k = 0; k < g->n; ++k) {
      if (s >= f0) {
        rc = hydro_gpu_slab_step_xy(g->ctx[k], s, (s - f0) & 1, s == f0, s + 1 == steps, halo);
      } else {
        if (halo) rc = hydro_gpu_slab_inbox_in(g->ctx[k], s);
        if (!rc) rc = hydro_gpu_slab_sweep_x(g->ctx[k], s);
        if (!rc) rc = hydro_gpu_slab_sweep_y(g->ctx[k], s);
      }
      if (rc) return slab_rc(g, k, rc);
    }
  }
  for (int k = 0; k < g->n; ++k) {
    const int rc = hydro_gpu_slab_run_end(g->ctx[k], f0 < steps);
    if (rc) return slab_rc(g, k, rc);
  }
  return HYDRO_GPU_OK;
}

// Captures (once per step count) the whole run from the leader's stream --
// the other slabs' streams fork from it and join back -- and launches it.
// Returns false if graphs cannot be used (the caller enqueues directly).
bool launch_group_graph(hydro_gpu_group* g, int steps) {
  if (!g->use_graphs) return false;
  Guard d0(g->device[0]);
  cudaGraphExec_t exec = nullptr;
  const int key = 2 * steps + (g->fused ? 1 : 0);
  for (auto& e : g->graphs)
    if (e.first == key) exec = e.second;
  if (!exec) {
    if (cudaStreamBeginCapture(g->stream[0], cudaStreamCaptureModeRelaxed) != cudaSuccess) {
      cudaGetLastError();
      g->use_graphs = false;
      return false;
    }
    bool ok = cudaEventRecord(g->lead, g->stream[0]) == cudaSuccess;
    for (int k = 1; ok && k < g->n; ++k) {  // fork
      Guard d(g->device[k]);
      ok = cudaStreamWaitEvent(g->stream[k], g->lead, 0) == cudaSuccess;
    }
    ok = ok && enqueue_group_run(g, steps) == HYDRO_GPU_OK;
    for (int k = 1; ok && k < g->n; ++k) {  // join
      {
        Guard d(g->device[k]);
        ok = cudaEventRecord(g->done[k], g->stream[k]) == cudaSuccess;
      }
      ok = ok && cudaStreamWaitEvent(g->stream[0], g->done[k], 0) == cudaSuccess;
    }
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(g->stream[0], &graph);
    if (!ok || ec != cudaSuccess || !graph || cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      g->use_graphs = false;
      g->last = hydro_gpu_error{};
      return false;
    }
    cudaGraphDestroy(graph);
    if (g->graphs.size() >= 8) {
      cudaGraphExecDestroy(g->graphs.front().second);
      g->graphs.erase(g->graphs.begin());
    }
    g->graphs.push_back({key, exec});
  }
  if (cudaGraphLaunch(exec, g->stream[0]) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return true;
}

}  // namespace

extern "C" {

int hydro_gpu_group_create(const hydro_gpu_cfg* cfg, int n_gpus, const int* devices,
                           hydro_gpu_group** out) {
  // every slab needs the 2 rows its neighbours' halos take from it
  if (!cfg || !out || n_gpus < 1 || n_gpus > kMaxSlabs || cfg->nx < 2 * n_gpus)
    return HYDRO_GPU_ERR_CONFIG;
  *out = nullptr;
  auto* g = new hydro_gpu_group();
  g->cfg = *cfg;
  g->n = n_gpus;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
    cudaGetLastError();
    delete g;
    return HYDRO_GPU_ERR_CUDA;
  }
  // split_range (proj/src/decomposition.cpp:9-16): the first nx % n slabs
  // get one extra row
  const int base = cfg->nx / n_gpus, extra = cfg->nx % n_gpus;
  for (int k = 0; k < n_gpus; ++k) {
    const int dev = devices ? devices[k] : k % ndev;
    if (dev < 0 || dev >= ndev) {
      delete g;
      return HYDRO_GPU_ERR_CONFIG;
    }
    g->device.push_back(dev);
    g->rows.push_back(base + (k < extra ? 1 : 0));
    g->row0.push_back(k * base + std::min(k, extra));
  }
  // peer access between every pair of distinct devices (the dt min reads all
  // slabs' slots; the halo stores go to the neighbours)
  for (int k = 0; k < n_gpus; ++k)
    for (int j = 0; j < n_gpus; ++j) {
      const int a = g->device[k], b = g->device[j];
      if (a == b) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, a, b);
      if (!can) {
        destroy(g);
        return HYDRO_GPU_ERR_CUDA;
      }
      Guard d(a);
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        destroy(g);
        return HYDRO_GPU_ERR_CUDA;
      }
      cudaGetLastError();
    }
  for (int k = 0; k < n_gpus; ++k) {
    hydro_gpu_cfg c = *cfg;
    c.nx = g->rows[k];
    c.device = g->device[k];
    c.row0 = g->row0[k];
    c.global_nx = cfg->nx;
    c.wall_lo = k == 0;
    c.wall_hi = k == n_gpus - 1;
    hydro_gpu_ctx* h = nullptr;
    const int rc = hydro_gpu_create(&c, &h);
    g->ctx.push_back(h);
    if (rc) {
      destroy(g);
      return rc;
    }
    Guard d(g->device[k]);
    cudaStream_t s = nullptr;
    cudaEvent_t ev = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      g->stream.push_back(s);
      g->done.push_back(ev);
      destroy(g);
      return HYDRO_GPU_ERR_CUDA;
    }
    g->stream.push_back(s);
    g->done.push_back(ev);
    hydro_gpu_set_stream(h, s);
  }
  {
    Guard d(g->device[0]);
    if (cudaEventCreateWithFlags(&g->lead, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      destroy(g);
      return HYDRO_GPU_ERR_CUDA;
    }
  }
  for (int k = 0; k < n_gpus; ++k) {
    double *up = nullptr, *dn = nullptr;
    if (k > 0) hydro_gpu_inbox(g->ctx[k - 1], &up, nullptr);
    if (k < n_gpus - 1) hydro_gpu_inbox(g->ctx[k + 1], &dn, nullptr);
    const int rc = hydro_gpu_set_halo_peers(g->ctx[k], up, dn);
    if (rc) {
      destroy(g);
      return rc;
    }
  }
  *out = g;
  return HYDRO_GPU_OK;
}

int hydro_gpu_group_destroy(hydro_gpu_group* g) {
  if (!g) return HYDRO_GPU_ERR_CONFIG;
  destroy(g);
  return HYDRO_GPU_OK;
}

int hydro_gpu_group_last_error(const hydro_gpu_group* g, hydro_gpu_error* out) {
  if (!g || !out) return HYDRO_GPU_ERR_CONFIG;
  *out = g->last;
  return HYDRO_GPU_OK;
}

int hydro_gpu_group_slabs(const hydro_gpu_group* g, int* n, int* row0, int* rows, int* devices) {
  if (!g || !n) return HYDRO_GPU_ERR_CONFIG;
  *n = g->n;
  for (int k = 0; k < g->n; ++k) {
    if (row0) row0[k] = g->row0[k];
    if (rows) rows[k] = g->rows[k];
    if (devices) devices[k] = g->device[k];
  }
  return HYDRO_GPU_OK;
}

// Full-grid planes in the reference layout: slab k takes global plane rows
// row0 .. row0 + rows + 3 (its interior and 2 rows either side).
int hydro_gpu_group_upload(hydro_gpu_group* g, const double* const planes[4], size_t row_stride) {
  if (!g || !planes) return HYDRO_GPU_ERR_CONFIG;
  for (int k = 0; k < g->n; ++k) {
    const double* p[4];
    for (int v = 0; v < 4; ++v) p[v] = planes[v] ? planes[v] + (size_t)g->row0[k] * row_stride : nullptr;
    const int rc = hydro_gpu_upload_async(g->ctx[k], p, row_stride);
    if (rc) return slab_rc(g, k, rc);
  }
  for (int k = 0; k < g->n; ++k) {
    Guard d(g->device[k]);
    GROUP_CUDA(g, cudaStreamSynchronize(g->stream[k]));
  }
  return HYDRO_GPU_OK;
}

// Gathers each slab's own rows (the outer slabs also their wall ghost rows);
// interior slab boundaries' ghost rows are halo copies and are skipped.
int hydro_gpu_group_download(hydro_gpu_group* g, double* const planes[4], size_t row_stride) {
  if (!g || !planes) return HYDRO_GPU_ERR_CONFIG;
  if (row_stride < (size_t)g->cfg.ny + 4) return fail(g, HYDRO_GPU_ERR_CONFIG, "row stride below ny+4");
  for (int k = 0; k < g->n; ++k) {
    const int lo = k == 0 ? 0 : 2, hi = k == g->n - 1 ? g->rows[k] + 4 : g->rows[k] + 2;
    double* p[4];
    for (int v = 0; v < 4; ++v) {
      if (!planes[v]) return fail(g, HYDRO_GPU_ERR_CONFIG, "null plane");
      p[v] = planes[v] + (size_t)(g->row0[k] + lo) * row_stride;
    }
    // plane rows lo .. hi-1 of the slab = grid rows lo-1 .. hi-2
    const int rc = hydro_gpu_download_rows(g->ctx[k], p, row_stride, lo - 1, hi - lo);
    if (rc) return slab_rc(g, k, rc);
  }
  return HYDRO_GPU_OK;
}

int hydro_gpu_group_set_math(hydro_gpu_group* g, int math) {
  if (!g) return HYDRO_GPU_ERR_CONFIG;
  if (math != g->math) drop_graphs(g);  // the sweep kernels are baked into captured graphs
  g->math = math;
  for (int k = 0; k < g->n; ++k) {
    const int rc = hydro_gpu_set_math(g->ctx[k], math);
    if (rc) return slab_rc(g, k, rc);
  }
  return HYDRO_GPU_OK;
}

int hydro_gpu_group_init_case(hydro_gpu_group* g, int case_id, uint64_t seed) {
  if (!g) return HYDRO_GPU_ERR_CONFIG;
  for (int k = 0; k < g->n; ++k) {
    const int rc = hydro_gpu_init_case(g->ctx[k], case_id, seed);
    if (rc) return slab_rc(g, k, rc);
  }
  return HYDRO_GPU_OK;
}

// run_sequential over the slabs: the reference's per-step order with the dt
// min and the halo between the slabs' sweeps (see the file comment).
int hydro_gpu_group_run(hydro_gpu_group* g, int steps, double* last_dt) {
  if (!g || steps < 0 || steps > HYDRO_GPU_MAX_STEPS) return HYDRO_GPU_ERR_CONFIG;
  if (steps == 0) return HYDRO_GPU_OK;
  Guard d0(g->device[0]);
  g->fused = true;  // fused steps if every slab's schedule takes them
  for (int k = 0; k < g->n; ++k) {
    int f = 0;
    const int rc = hydro_gpu_slab_run_begin(g->ctx[k], steps, &f);
    if (rc) return slab_rc(g, k, rc);
    g->fused = g->fused && f != 0;
  }
  if (!(steps >= 2 && launch_group_graph(g, steps))) {
    const int rc = enqueue_group_run(g, steps);
    if (rc) return rc;
  }
  // first error in the reference's order: the minimum key over the slabs
  unsigned long long key = hb::kNoError;
  for (int k = 0; k < g->n; ++k) {
    uint64_t* slot = nullptr;
    hydro_gpu_error_slot(g->ctx[k], &slot);
    unsigned long long v = 0;
    Guard d(g->device[k]);
    GROUP_CUDA(g, cudaStreamSynchronize(g->stream[k]));
    GROUP_CUDA(g, cudaMemcpy(&v, slot, sizeof v, cudaMemcpyDeviceToHost));
    key = v < key ? v : key;
  }
  if (key != hb::kNoError) {
    const int rc = hydro_gpu_decode_error(g->ctx[0], key, &g->last);
    return rc ? rc : HYDRO_GPU_ERR_POSITIVITY;
  }
  if (last_dt) {  // the last step's dt: cfl * its (all-slab) limit (euler_kernel.cpp:241)
    double* slot = nullptr;
    hydro_gpu_limit_slot(g->ctx[0], steps - 1, &slot);
    double lim = 0.0;
    Guard d(g->device[0]);
    GROUP_CUDA(g, cudaMemcpy(&lim, slot, sizeof lim, cudaMemcpyDeviceToHost));
    *last_dt = g->cfg.cfl * lim;
  }
  return HYDRO_GPU_OK;
}

}  // extern "C"
