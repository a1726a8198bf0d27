// gpu_strategy.hpp -- header-only C++ adaptor that plugs libhydro_b200.so into
// the reference hydro2d as one more execution strategy.
//
// It is written against the reference's own types (include it from a tree
// that has proj/include on the include path) and the C-ABI in hydro_gpu.h:
//
//   reference                                        this adaptor
//   run_sequential(Grid2D&, const GasModel&, int)    run_gpu(grid, model, steps)
//     (proj/include/hydro/schedulers.hpp:24)
//   advance_sequential(Grid2D&, GasModel, double)    advance_gpu(grid, model, dt)
//     (schedulers.hpp:21)
//   run_until(Grid2D&, const GasModel&, double)      run_until_gpu(grid, model, t_end)
//     (schedulers.hpp:28)
//   compute_dt(const Grid2D&, const GasModel&)       compute_dt_gpu(grid, model)
//     (euler_kernel.hpp:75)
//
// Same argument meaning, same in-place mutation of the caller-owned Grid2D
// (every plane, ghosts included, ends bitwise equal to the reference's), and
// the same error behaviour: a positivity failure throws hydro::Error with
// ErrorCategory::Positivity and the reference's message, e.g.
// "step 3: column sweep strip 17: rho non-positive at strip cell -2"
// (schedulers.cpp:23-26,80-91); configuration problems throw ConfigError; a
// CUDA failure (no reference counterpart) throws std::runtime_error, which
// hydrobench reports as "error: internal: ..." (tools/hydrobench.cpp:156-159).
// See INTEGRATION.md for the run_strategy hook.
#pragma once

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hydro/errors.hpp"
#include "hydro/grid.hpp"
#include "hydro/types.hpp"
#include "hydro_gpu.h"

namespace hydro {

struct GpuOptions {
  int device = -1;                    // CUDA device; -1 = current (gpus == 1)
  int gpus = 1;                       // > 1: row slabs on devices 0..gpus-1 (hydro_gpu_group),
                                      // all on `device` if it is >= 0
  int bc = HYDRO_GPU_BC_REFLECT;      // the reference's walls; TRANSMIT for BASELINE configs
  int flux = HYDRO_GPU_FLUX_HLLC;     // the reference hot path; EXACT10 = BASELINE's solver
  int math = HYDRO_GPU_MATH_BITWISE;  // the reference's bits; TOLERANCE = max_rel <= 1e-12
};

namespace gpu_detail {

[[noreturn]] inline void raise(int status, const std::string& message) {
  switch (status) {
    case HYDRO_GPU_ERR_CONFIG: throw ConfigError(message);
    case HYDRO_GPU_ERR_POSITIVITY: throw Error(ErrorCategory::Positivity, message);
    case HYDRO_GPU_ERR_CUDA: throw std::runtime_error(message);
    default: throw Error(static_cast<ErrorCategory>(status - 1), message);
  }
}

// One device-resident copy of a Grid2D for the duration of a call.
class Context {
 public:
  Context(const Grid2D& g, const GasModel& m, const GpuOptions& o) {
    hydro_gpu_cfg cfg{};
    cfg.nx = g.nx();
    cfg.ny = g.ny();
    cfg.dx = g.dx();
    cfg.dy = g.dy();
    cfg.gamma = m.gamma;
    cfg.cfl = m.cfl;
    cfg.bc = o.bc;
    cfg.flux = o.flux;
    cfg.device = o.device;
    cfg.row0 = 0;
    cfg.global_nx = g.nx();
    cfg.wall_lo = cfg.wall_hi = 1;
    const int rc = hydro_gpu_create(&cfg, &ctx_);
    if (rc != HYDRO_GPU_OK)
      raise(rc, std::string("hydro_gpu_create: ") + hydro_gpu_status_string(rc));
    const int mrc = o.math == HYDRO_GPU_MATH_BITWISE ? HYDRO_GPU_OK : hydro_gpu_set_math(ctx_, o.math);
    if (mrc != HYDRO_GPU_OK) {
      hydro_gpu_destroy(ctx_);
      raise(mrc, "hydro_gpu_set_math: unknown math mode");
    }
  }
  ~Context() { hydro_gpu_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  void download(Grid2D& g) {
    double* planes[4];
    for (int v = 0; v < kNumVars; ++v) planes[v] = &g.at(Var(v), -1, -1);
    check(hydro_gpu_download(ctx_, planes, g.ny() + 2 * kGhost));
  }
  void check(int rc) {
    if (rc == HYDRO_GPU_OK) return;
    hydro_gpu_error e{};
    hydro_gpu_last_error(ctx_, &e);
    raise(rc, e.message);
  }
  hydro_gpu_ctx* get() { return ctx_; }

 private:
  hydro_gpu_ctx* ctx_ = nullptr;
};

// The context of the previous call, kept for the next one: the reference's
// callers are single-threaded and a run_benchmark / validation
// sequence steps grids of one geometry again and again, so consecutive calls
// with the same geometry, model and options reuse its device buffers, tensor
// maps and captured CUDA graphs instead of allocating and capturing afresh.
// The grid's pageable planes are staged through the context's pinned ring
// (hydro_gpu_upload / hydro_gpu_download).
struct CacheKey {
  int nx = 0, ny = 0, bc = 0, flux = 0, device = 0, math = 0;
  double dx = 0, dy = 0, gamma = 0, cfl = 0;
  bool operator==(const CacheKey& o) const {
    return nx == o.nx && ny == o.ny && bc == o.bc && flux == o.flux && device == o.device &&
           math == o.math && dx == o.dx && dy == o.dy && gamma == o.gamma && cfl == o.cfl;
  }
};

struct Cache {
  std::unique_ptr<Context> ctx;
  CacheKey key;
};

inline Cache& cache() {
  thread_local Cache c;
  return c;
}

inline Context& cached_context(const Grid2D& g, const GasModel& m, const GpuOptions& o) {
  const CacheKey k{g.nx(), g.ny(), o.bc, o.flux, o.device, o.math, g.dx(), g.dy(), m.gamma, m.cfl};
  Cache& c = cache();
  if (!c.ctx || !(c.key == k)) {
    c.ctx.reset();
    c.ctx = std::make_unique<Context>(g, m, o);
    c.key = k;
  }
  return *c.ctx;
}

// Grid2D::at(...) const returns by value; the planes are contiguous vectors,
// so the address of cell (-1,-1) is taken through a non-const view.
inline const double* plane(const Grid2D& g, int v) {
  return &const_cast<Grid2D&>(g).at(Var(v), -1, -1);
}

}  // namespace gpu_detail

// Frees the context kept between calls (device memory, pinned staging).
inline void release_gpu_cache() { gpu_detail::cache().ctx.reset(); }

// run_sequential over row slabs on several GPUs driven by this thread
// (hydro_gpu_group: peer-memory halo, on-device dt min), bitwise equal to
// the single-device run.
inline double run_gpu_slabs(Grid2D& grid, const GasModel& model, int steps,
                            const GpuOptions& opt) {
  hydro_gpu_cfg cfg{};
  cfg.nx = grid.nx();
  cfg.ny = grid.ny();
  cfg.dx = grid.dx();
  cfg.dy = grid.dy();
  cfg.gamma = model.gamma;
  cfg.cfl = model.cfl;
  cfg.bc = opt.bc;
  cfg.flux = opt.flux;
  cfg.device = -1;
  // device >= 0: every slab on that device (a single-GPU check of the slab path)
  std::vector<int> devices(opt.gpus > 0 ? opt.gpus : 1, opt.device);
  hydro_gpu_group* g = nullptr;
  int rc = hydro_gpu_group_create(&cfg, opt.gpus, opt.device >= 0 ? devices.data() : nullptr, &g);
  if (rc != HYDRO_GPU_OK)
    gpu_detail::raise(rc, std::string("hydro_gpu_group_create: ") + hydro_gpu_status_string(rc));
  auto fail = [&](int status) {
    hydro_gpu_error e{};
    hydro_gpu_group_last_error(g, &e);
    hydro_gpu_group_destroy(g);
    gpu_detail::raise(status, e.message);
  };
  if (opt.math != HYDRO_GPU_MATH_BITWISE && (rc = hydro_gpu_group_set_math(g, opt.math)) != HYDRO_GPU_OK)
    fail(rc);
  const double* in[4];
  double* out[4];
  for (int v = 0; v < kNumVars; ++v) {
    in[v] = gpu_detail::plane(grid, v);
    out[v] = &grid.at(Var(v), -1, -1);
  }
  if ((rc = hydro_gpu_group_upload(g, in, grid.ny() + 2 * kGhost)) != HYDRO_GPU_OK) fail(rc);
  double last_dt = 0.0;
  const int run_rc = hydro_gpu_group_run(g, steps, &last_dt);
  if ((rc = hydro_gpu_group_download(g, out, grid.ny() + 2 * kGhost)) != HYDRO_GPU_OK) fail(rc);
  if (run_rc != HYDRO_GPU_OK) fail(run_rc);
  hydro_gpu_group_destroy(g);
  return last_dt;
}

// run_sequential on the GPU: `steps` steps of BC -> dt -> column sweep ->
// BC -> row sweep, bitwise equal to the reference; returns the last dt.
inline double run_gpu(Grid2D& grid, const GasModel& model, int steps,
                      const GpuOptions& opt = {}) {
  if (opt.gpus > 1) return run_gpu_slabs(grid, model, steps, opt);
  gpu_detail::Context& ctx = gpu_detail::cached_context(grid, model, opt);
  const double* planes[4];
  for (int v = 0; v < kNumVars; ++v) planes[v] = gpu_detail::plane(grid, v);
  ctx.check(hydro_gpu_upload(ctx.get(), planes, grid.ny() + 2 * kGhost));
  double last_dt = 0.0;
  const int rc = hydro_gpu_run(ctx.get(), steps, &last_dt);
  ctx.download(grid);
  ctx.check(rc);
  return last_dt;
}

inline void advance_gpu(Grid2D& grid, const GasModel& model, double dt,
                        const GpuOptions& opt = {}) {
  gpu_detail::Context& ctx = gpu_detail::cached_context(grid, model, opt);
  const double* planes[4];
  for (int v = 0; v < kNumVars; ++v) planes[v] = gpu_detail::plane(grid, v);
  ctx.check(hydro_gpu_upload(ctx.get(), planes, grid.ny() + 2 * kGhost));
  const int rc = hydro_gpu_advance(ctx.get(), dt);
  ctx.download(grid);
  ctx.check(rc);
}

inline int run_until_gpu(Grid2D& grid, const GasModel& model, double t_end,
                         const GpuOptions& opt = {}) {
  gpu_detail::Context& ctx = gpu_detail::cached_context(grid, model, opt);
  const double* planes[4];
  for (int v = 0; v < kNumVars; ++v) planes[v] = gpu_detail::plane(grid, v);
  ctx.check(hydro_gpu_upload(ctx.get(), planes, grid.ny() + 2 * kGhost));
  int steps = 0;
  const int rc = hydro_gpu_run_until(ctx.get(), t_end, &steps);
  ctx.download(grid);
  ctx.check(rc);
  return steps;
}

inline double compute_dt_gpu(const Grid2D& grid, const GasModel& model,
                             const GpuOptions& opt = {}) {
  gpu_detail::Context& ctx = gpu_detail::cached_context(grid, model, opt);
  const double* planes[4];
  for (int v = 0; v < kNumVars; ++v) planes[v] = gpu_detail::plane(grid, v);
  ctx.check(hydro_gpu_upload(ctx.get(), planes, grid.ny() + 2 * kGhost));
  double dt = 0.0;
  ctx.check(hydro_gpu_compute_dt(ctx.get(), &dt));
  return dt;
}

}  // namespace hydro
