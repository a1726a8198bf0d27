// hydrobench_gpu -- the reference's `hydrobench run` / `bench` command surface
// with one more strategy, "gpu", served by libhydro_b200.so through
// include/hydro/gpu_strategy.hpp.  Everything else -- RunConfig, make_case,
// run_strategy for the CPU strategies, grid_checksum/format_checksum, the CSV
// report and the "error: <category>: <message>" convention -- is the
// unmodified reference library (proj/src, linked as objects).  CLI11 is not
// vendored in the reference tree, so flags are parsed by hand with the same
// names (proj/tools/hydrobench.cpp:93-137).
//
//   hydrobench_gpu run --case blast --nx 48 --ny 48 --steps 5 --strategy gpu
//   hydrobench_gpu bench --case blast --nx 2048 --ny 2048 --steps 10 --strategy gpu
//   extra: --case corner_blast|sod_x|random (BASELINE configs), --bc reflect|transmit,
//          --flux hllc|exact10 and --math bitwise|tolerance (gpu strategy), --gpus N (row slabs on GPUs 0..N-1,
//          one host thread; with --device D all N slabs share GPU D),
//          --seed N (random field), --device N
#include <chrono>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "hydro/audit.hpp"
#include "hydro/bench.hpp"
#include "hydro/errors.hpp"
#include "hydro/gpu_strategy.hpp"
#include "hydro_gpu.h"

namespace {

struct Args {
  hydro::RunConfig config;
  std::string command;
  std::string bc = "reflect";
  std::string flux = "hllc";
  std::string math = "bitwise";
  int device = -1;
  int gpus = 1;
};

Args parse(int argc, char** argv) {
  Args a;
  if (argc < 2) throw hydro::ConfigError("usage: hydrobench_gpu run|bench [--option value]...");
  a.command = argv[1];
  for (int k = 2; k < argc; ++k) {
    const std::string key = argv[k];
    if (k + 1 >= argc) throw hydro::ConfigError("option " + key + " needs a value");
    const std::string val = argv[++k];
    auto& c = a.config;
    if (key == "--case") c.case_name = val;
    else if (key == "--nx") c.nx = std::stoi(val);
    else if (key == "--ny") c.ny = std::stoi(val);
    else if (key == "--steps") c.steps = std::stoi(val);
    else if (key == "--strategy") c.strategy = val;
    else if (key == "--workers") c.workers = {std::stoi(val)};
    else if (key == "--gamma") c.gamma = std::stod(val);
    else if (key == "--cfl") c.cfl = std::stod(val);
    else if (key == "--seed") c.seed = std::stoull(val);
    else if (key == "--output") c.output = val;
    else if (key == "--bc") a.bc = val;
    else if (key == "--flux") a.flux = val;
    else if (key == "--math") a.math = val;
    else if (key == "--gpus") a.gpus = std::stoi(val);
    else if (key == "--device") a.device = std::stoi(val);
    else throw hydro::ConfigError("unknown option " + key);
  }
  return a;
}

// The reference's cases through its own make_case; the BASELINE cases
// through the library's host initialiser (bitwise equal to the oracle's).
hydro::Grid2D build_case(const Args& a) {
  const auto& c = a.config;
  if (c.case_name == "blast" || c.case_name == "sod" || c.case_name == "uniform")
    return hydro::make_case(c);
  int id = -1;
  if (c.case_name == "corner_blast") id = HYDRO_GPU_CASE_CORNER_BLAST;
  if (c.case_name == "sod_x") id = HYDRO_GPU_CASE_SOD_X;
  if (c.case_name == "random") id = HYDRO_GPU_CASE_RANDOM;
  if (id < 0) throw hydro::ConfigError("unknown case '" + c.case_name + "'");
  hydro::Grid2D g(c.nx, c.ny, 1.0 / c.nx, 1.0 / c.ny);
  double* planes[4];
  for (int v = 0; v < 4; ++v) planes[v] = &g.at(hydro::Var(v), -1, -1);
  double dx = 0, dy = 0;
  if (hydro_init_case_host(id, c.nx, c.ny, c.gamma, c.seed, planes, c.ny + 4, &dx, &dy) != 0)
    throw hydro::ConfigError("cannot build case '" + c.case_name + "'");
  return g;
}

void step(hydro::Grid2D& grid, const Args& a, int steps) {
  hydro::RunConfig c = a.config;
  c.steps = steps;
  if (c.strategy == "gpu") {
    hydro::GpuOptions opt;
    opt.device = a.device;
    opt.bc = a.bc == "transmit" ? HYDRO_GPU_BC_TRANSMIT : HYDRO_GPU_BC_REFLECT;
    if (a.flux != "hllc" && a.flux != "exact10")
      throw hydro::ConfigError("unknown flux '" + a.flux + "'");
    opt.flux = a.flux == "exact10" ? HYDRO_GPU_FLUX_EXACT10 : HYDRO_GPU_FLUX_HLLC;
    if (a.math != "bitwise" && a.math != "tolerance")
      throw hydro::ConfigError("unknown math mode '" + a.math + "'");
    opt.math = a.math == "tolerance" ? HYDRO_GPU_MATH_TOLERANCE : HYDRO_GPU_MATH_BITWISE;
    if (a.gpus < 1) throw hydro::ConfigError("--gpus must be at least 1");
    opt.gpus = a.gpus;
    hydro::run_gpu(grid, hydro::GasModel{c.gamma, c.cfl}, steps, opt);
  } else {
    if (a.bc != "reflect")
      throw hydro::ConfigError("the CPU strategies only have reflective walls");
    if (a.flux != "hllc")
      throw hydro::ConfigError("the CPU strategies only have the HLLC flux");
    if (a.math != "bitwise")
      throw hydro::ConfigError("the CPU strategies only have the reference's arithmetic");
    hydro::run_strategy(grid, c, c.workers[0]);
  }
}

int cmd_run(const Args& a) {
  hydro::Grid2D grid = build_case(a);
  const auto t0 = std::chrono::steady_clock::now();
  step(grid, a, a.config.steps);
  const double seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const std::string line = hydro::format_checksum(hydro::grid_checksum(grid));
  std::printf("case=%s %dx%d steps=%d strategy=%s workers=%d time_s=%.3f\n",
              a.config.case_name.c_str(), grid.nx(), grid.ny(), a.config.steps,
              a.config.strategy.c_str(), a.config.workers[0], seconds);
  std::printf("checksum %s\n", line.c_str());
  if (!a.config.output.empty()) hydro::write_text_file(a.config.output, line + "\n");
  return 0;
}

// run_benchmark's protocol (bench.cpp:92-152): one untimed warm-up step from
// a copy of the initial grid, then the timed run, reported as CSV.
int cmd_bench(const Args& a) {
  const hydro::Grid2D initial = build_case(a);
  {
    hydro::Grid2D warm = initial;
    step(warm, a, 1);
  }
  hydro::Grid2D grid = initial;
  const auto t0 = std::chrono::steady_clock::now();
  step(grid, a, a.config.steps);
  const double seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const auto records = hydro::make_records({1}, {seconds}, hydro::grid_checksum(grid).digest);
  const std::string csv = hydro::render_csv(records);
  std::fputs(csv.c_str(), stdout);
  std::printf("# %.6g cell-steps/s\n",
              (double)grid.nx() * grid.ny() * a.config.steps / seconds);
  if (!a.config.output.empty()) hydro::write_text_file(a.config.output, csv);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    if (a.command == "run") return cmd_run(a);
    if (a.command == "bench") return cmd_bench(a);
    throw hydro::ConfigError("unknown subcommand '" + a.command + "' (run or bench)");
  } catch (const hydro::Error& e) {
    std::fprintf(stderr, "error: %s: %s\n", hydro::to_string(e.category()), e.what());
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: internal: %s\n", e.what());
    return 1;
  }
}
