"""Benchmark of the B200 HYDRO step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg0..cfg4] [--flux hllc|exact10] [--math bitwise|tolerance]

Headline workload: BASELINE config 3 -- the 16384x16384 fp64 corner blast
(rho=1, u=v=0, p=1e-5, E=1/dx^2 in cell (0,0)), reflecting walls, gamma 1.4,
CFL 0.8, MUSCL-Hancock + minmod + HLLC (the reference's hot-path flux), 50
time steps, strong-scaled over N GPUs as row slabs (the metric's "at 1/2/4/8
B200" configuration).  One bench step is one 50-time-step run from the
initial condition; its final state is checked against the reference's digest
(tests/golden/golden_full.json) and the bench fails like run_benchmark's
equivalence gate (proj/src/bench.cpp:131-143) if it differs.

The headline runs the tolerance math mode (the north star's parity bar:
compare_tolerance max_rel <= 1e-12 in fp64, measured live against the bitwise
state of the same run, whose digest is the reference's); the bitwise mode is
measured beside it under ``math_variants``.

Metric: cell-updates/s = interior cells x time steps / seconds (both sweeps +
the dt reduction per time step).  ``value`` is device-resident (state in HBM
before the timed region, CUDA events on the launch stream, max over ranks);
``e2e`` goes through the C-ABI with pinned host buffers: upload, run, download
every bench step.  Beside the headline the line carries the other math mode
(``math_variants``: bitwise <-> tolerance, the latter gated on
compare_tolerance max_rel <= 1e-12 against the digest-pinned bitwise state),
the exact-10 flux (``flux_variants``) and, at N=1, configs 2 and 1 as
secondary measured lines (``secondary``), each with its own roofline.
``--impl reference`` times the reference's own CPU implementation
(oracle/_ref, its fastest strategy over the host cores) on the same 50-step
run of the same grid, split into K timed windows of one flow.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs: name -> (case, nx, ny, bc, time steps
# per bench step, seed, scaling when --gpus > 1).  Strong scaling splits the
# grid's rows over the ranks; weak scaling grows the slab axis i by N.
WORKLOADS = {
    "cfg0": ("corner_blast", 256, 256, "reflect", 100, 0, "weak"),
    "cfg1": ("sod_x", 2048, 2048, "transmit", 200, 0, "weak"),
    "cfg2": ("random", 8192, 8192, "transmit", 50, 2106, "weak"),
    "cfg3": ("corner_blast", 16384, 16384, "reflect", 50, 0, "strong"),
    "cfg4": ("random", 16384, 16384, "transmit", 20, 13465, "weak"),
}
DEFAULT_WORKLOAD = "cfg3"
SECONDARY = ("cfg2", "cfg1")
METRIC = "cell-updates/s (both sweeps, fp64)"
UNIT = "cell-updates/s"
ALG_BYTES_PER_CELL_SWEEP = 64  # 32 B read + 32 B write of 4 fp64 fields
FP64_FLOPS_PER_CELL_STEP = 348  # SURVEY.md Appendix A (36 div, 5 sqrt)
TOLERANCE = 1e-12  # compare_tolerance max_rel bound (proj/src/audit.cpp:137-154)


class ParityFailure(RuntimeError):
    pass


def golden_digest(workload: str, flux: str, global_nx: int) -> str | None:
    """The reference's digest of this run (tests/golden/, made by the compiled
    reference / the oracle), or None where none was pinned."""
    case, nx, ny, bc, tsteps, seed, _ = WORKLOADS[workload]
    if global_nx != nx:
        return None  # weak-scaled grid: not pinned
    want = {"case": case, "nx": nx, "ny": ny, "bc": bc, "steps": tsteps}
    for name in ("golden_full.json", "golden.json"):
        path = os.path.join(ROOT, "tests", "golden", name)
        if not os.path.exists(path):
            continue
        for entry in json.load(open(path)).values():
            if all(entry.get(k) == v for k, v in want.items()) and \
                    entry.get("flux", "hllc") == flux and entry.get("seed", 0) == seed:
                return entry["digest"]
    return None


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def fp64_peak():
    """Measured FP64 peak (profiles/fp64_peak.json, tools/fp64_peak.cu)."""
    path = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(path):
        return json.load(open(path))
    return None


def cpu_info() -> dict:
    """lscpu model, sockets and core counts of this host (as
    acceptance_tests.cpp:341 records hardware_concurrency)."""
    info = {"logical": os.cpu_count() or 1}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for line in out.splitlines():
            if ":" in line:
                k, v = line.split(":", 1)
                kv[k.strip()] = v.strip()
        info["model"] = kv.get("Model name")
        sockets = int(kv.get("Socket(s)", "1") or 1)
        cores = int(kv.get("Core(s) per socket", "0") or 0)
        info["sockets"] = sockets
        if cores:
            info["physical_cores"] = sockets * cores
        info["threads_per_core"] = int(kv.get("Thread(s) per core", "1") or 1)
    except (OSError, ValueError, subprocess.TimeoutExpired):
        pass
    try:
        info["affinity"] = len(os.sched_getaffinity(0))
    except AttributeError:
        pass
    return info


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, ValueError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, pw, reasons = [], 0.0, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
                pw.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "power_w_median": statistics.median(pw) if pw else None, "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------
# The reference's CPU path (oracle/_ref; the C port where it was not built)

_BEST = {}


def best_cpu_strategy(case, bc, seed, threads_options):
    """The reference's fastest parallel strategy and worker count on this host
    (bench.cpp:53-90 dispatch): short probes of fine_grain / coarse_grain /
    task_graph at each worker count on a 2048^2 grid of the workload's case."""
    from oracle import oracle as O
    key = (case, bc, tuple(threads_options))
    if key not in _BEST:
        g = O.make_case(case, 2048, 2048, seed=seed)
        rates = {}
        for w in threads_options:
            for strat in ("coarse_grain", "fine_grain", "task_graph"):
                h = g.copy()
                O.ref_run(h, 1, bc, strat, w)  # warm-up (bench.cpp:112-117)
                rates[(strat, w)] = 2 / O.ref_run(h, 2, bc, strat, w)
        _BEST[key] = max(rates, key=rates.get)
    return _BEST[key]


def cpu_threads_options(info):
    opts = {info.get("affinity") or info["logical"]}
    if info.get("physical_cores"):
        opts.add(min(info["physical_cores"], info.get("affinity") or info["logical"]))
    return sorted(opts)


def cpu_reference_run(case, nx, ny, bc, seed, windows, threads=None, strategy=None):
    """Times the reference's CPU path on consecutive windows of one flow from
    the initial condition of the workload (grid loaded once; the strategy and
    worker count that probed fastest here).  Returns (seconds per window,
    kind, strategy, workers, final grid)."""
    from oracle import oracle as O
    g = O.make_case(case, nx, ny, seed=seed)
    if not O.ref_available():  # the C port, single thread
        secs = []
        for w in windows:
            t0 = time.perf_counter()
            if w:
                O.run_sequential(g, w, bc)
            secs.append(time.perf_counter() - t0)
        return secs, "port", "sequential", 1, g
    if strategy is None:
        strategy, threads = best_cpu_strategy(case, bc, seed, cpu_threads_options(cpu_info()))
    if strategy == "sequential":
        threads = 1
    return O.ref_run_windows(g, list(windows), bc, strategy, threads), "reference", strategy, threads, g


def split_steps(total, parts):
    base, extra = divmod(total, parts)
    return [base + (1 if k < extra else 0) for k in range(parts)]


def run_reference_arm(args, rank, world):
    """The driver's reference arm: rank 0 alone times the reference's CPU path
    on the same run the GPU arm measures (the workload's full T-step run from
    its initial condition, split into K timed windows of one flow, after one
    untimed warm-up step on a copy like bench.cpp:112-117); other ranks exit."""
    if rank != 0:
        return
    from oracle import oracle as O
    case, nx, ny, bc, tsteps, seed, scaling = WORKLOADS[args.workload]
    global_nx = nx * world if scaling == "weak" else nx
    info = cpu_info()
    strategy, threads = ("sequential", 1)
    if O.ref_available():
        strategy, threads = best_cpu_strategy(case, bc, seed, cpu_threads_options(info))
        warm = O.make_case(case, min(global_nx, 2048), min(ny, 2048), seed=seed)
        for _ in range(max(0, args.warmup)):
            O.ref_run(warm, 1, bc, strategy, threads)
    windows = split_steps(tsteps, max(1, min(args.steps, tsteps)))
    secs, kind, strategy, threads, g = cpu_reference_run(case, global_nx, ny, bc, seed, windows,
                                                         threads, strategy)
    total = sum(secs)
    cells = global_nx * ny
    value = cells * tsteps / total
    digest = f"{O.digest(g):016x}"
    want = golden_digest(args.workload, "hllc", global_nx)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(windows), "warmup": args.warmup,
        "ms_per_step": total / len(windows) * 1e3,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (analytic or seeded initial condition, no dataset)",
        "config": workload_config(args.workload, global_nx, "hllc", "bitwise", world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"the whole {tsteps}-step run of the {global_nx}x{ny} "
                                   f"{args.workload} grid as {len(windows)} timed windows of one "
                                   f"flow ({total:.1f}s stepping), reference {strategy} x{threads} "
                                   "(its fastest strategy/worker count here, bench.cpp:53-90)",
                         "cpu": info},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "window_steps": windows, "window_seconds": secs,
        "result_digest": digest, "golden_digest": want,
        "parity_ok": (digest == want) if want else None,
    }
    print(json.dumps(line), flush=True)


def workload_config(workload, global_nx, flux, math, world):
    case, nx, ny, bc, tsteps, seed, scaling = WORKLOADS[workload]
    return {"workload": f"BASELINE {workload}: {global_nx}x{ny} {case} {bc}, {flux}, "
                        f"{tsteps} time steps per bench step",
            "cells": global_nx * ny, "time_steps_per_bench_step": tsteps,
            "parallelism": f"row slabs x{world}" if world > 1 else "single GPU",
            "flux": flux, "math": math, "seed": seed}


def max_rel_planes(a, b, rows: int = 1024) -> float:
    """compare_tolerance's max |a-b| / max(|a|,|b|,1) (proj/src/audit.cpp:146)
    over (4, nx, ny) host planes, in row blocks."""
    import numpy as np
    out = 0.0
    for i in range(0, a.shape[1], rows):
        x, y = a[:, i:i + rows], b[:, i:i + rows]
        out = max(out, float((np.abs(x - y) / np.maximum(np.maximum(np.abs(x), np.abs(y)), 1.0)).max()))
    return out


# ---------------------------------------------------------------------------
# GPU arm


class Env:
    """Rank, device, stream and the process group of one bench process."""

    def __init__(self, args):
        import torch
        self.torch = torch
        self.rank, self.world, self.local = dist_env()
        self.shared = self.world > 1 and os.environ.get("HYDRO_BENCH_SHARED_GPU") == "1"
        if self.shared:
            self.local = 0
        torch.cuda.set_device(self.local)
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist
            if self.shared:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.dist = dist
        self.stream = torch.cuda.Stream()  # library kernels, NCCL and events share it
        torch.cuda.set_stream(self.stream)
        self.comm_dev = "cpu" if self.shared else "cuda"

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def allmax(self, *vals):
        if self.dist is None:
            return vals if len(vals) > 1 else vals[0]
        t = self.torch.tensor(list(vals), dtype=self.torch.float64, device=self.comm_dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        out = tuple(float(x) for x in t.tolist())
        return out if len(out) > 1 else out[0]

    def send_u64(self, h, to):
        t = self.torch.tensor([h - (1 << 64) if h >= (1 << 63) else h], dtype=self.torch.int64,
                              device=self.comm_dev)
        self.dist.send(t, to)

    def recv_u64(self, frm):
        t = self.torch.zeros(1, dtype=self.torch.int64, device=self.comm_dev)
        self.dist.recv(t, frm)
        return int(t.item()) & ((1 << 64) - 1)


class Measured:
    """One (workload, flux, math) configuration on this rank: a context (or
    slab) with its final state kept on the device for comparisons."""

    def __init__(self, env: Env, workload: str, flux: str, math: str):
        import paper_2106_13465_b200 as P
        from paper_2106_13465_b200 import slab as S
        self.env, self.workload, self.flux, self.math = env, workload, flux, math
        case, nx, ny, bc, tsteps, seed, scaling = WORKLOADS[workload]
        self.case, self.ny, self.bc, self.tsteps, self.seed, self.scaling = case, ny, bc, tsteps, seed, scaling
        world = env.world
        self.global_nx = nx * world if scaling == "weak" else nx
        self.cells = self.global_nx * ny
        dx, dy = 1.0 / self.global_nx, 1.0 / ny
        self.geo = S.SlabGeometry(self.global_nx, ny, env.rank, world)
        model = P.GasModel()
        if world == 1:
            self.grid = P.GpuGrid(self.global_nx, ny, dx, dy, model, bc, device=env.local, flux=flux,
                                  math=math)
            self.grid.set_stream(env.stream.cuda_stream)
            self.slab = self.comm = None
        else:
            self.slab = S.GpuSlab(self.geo, dx, dy, model, bc, env.local, flux=flux, math=math)
            self.slab.bind_stream(env.stream)
            self.grid = self.slab.grid
            self.comm = S.TorchComm()
            self.comm.setup_p2p(self.slab)  # peer-memory halo over NVLink if every rank maps its peers
            # the whole schedule in the library: one CUDA graph per run per rank
            # (NCCL dt allreduce inside) -- else the Python per-step driver
            self.comm.setup_native(self.slab)
        self.halo = (("peer-memory (row-sweep stores into neighbour inboxes)" if self.comm.p2p
                      else "nccl send/recv") if world > 1 else None)
        self.driver = (("C++: one CUDA graph per run per rank, NCCL min-allreduce of dt per step "
                        "(hydro_gpu_comm_attach)" if self.comm.native
                        else "python: per-step calls (slab.run_slab)") if world > 1 else None)
        self.S = S

    def close(self):
        self.grid.close()

    def run(self):
        if self.env.world == 1:
            self.grid.run_async(self.tsteps)
        else:
            self.S.run_slab(self.slab, self.comm, self.tsteps)

    def one_step(self):
        self.grid.init_case(self.case, self.seed)
        self.run()

    def sync(self):
        if self.env.world == 1:
            self.grid.sync()
        self.env.torch.cuda.synchronize()

    def device_timed(self, steps, warmup, clocks=None):
        """W untimed + K timed bench steps (CUDA events on the launch stream,
        barrier + synchronize on both sides, max over ranks)."""
        torch, env = self.env.torch, self.env
        self.grid.set_timing(False)
        for _ in range(warmup):
            self.one_step()
            self.sync()  # (the AUTO schedule settles its choice between completed runs)
        env.barrier()
        torch.cuda.synchronize()
        if clocks:
            clocks.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(env.stream)
        for _ in range(steps):
            self.one_step()
        e1.record(env.stream)
        self.sync()
        clock_info = clocks.stop() if clocks else None
        env.barrier()
        ms = env.allmax(e0.elapsed_time(e1))
        return ms, clock_info

    def kernel_times(self, steps):
        """Per-kernel device time: a second, event-instrumented pass of the
        same bench steps (event nodes inside the graph would perturb the
        clean replays)."""
        self.grid.reset_counters()
        self.grid.set_timing(True)
        for _ in range(steps):
            self.one_step()
        self.sync()
        kt = self.grid.kernel_times()
        kt["ms_xy"], kt["n_xy"] = self.grid.fused_times()
        kt["ms_comm"], kt["n_comm"] = self.grid.comm_times()
        kt["skipped_x"], kt["skipped_y"] = self.grid.skipped()
        kt["auto_fused"], kt["auto_share"] = self.grid.schedule_choice()
        self.grid.set_timing(False)
        return kt

    def roofline(self, kt, clock_info):
        """The dominant kernel against the HBM roofline, and the whole time step
        against the HBM and the measured FP64 peaks.

        Algorithmic bytes of one launch: a split sweep reads and writes the
        state once (64 B per cell: two such sweeps = 128 B per
        cell-step); the fused step kernel (both sweeps in one pass, the
        column sweep's output kept in shared memory) also reads and writes the
        state once per launch -- 64 B per cell -- but completes a whole
        cell-step with it.  `frac` is the kernel against the bytes IT must
        move; `step.frac_survey_128B` is the step against the survey's
        two-sweep traffic model, which a fused step may exceed."""
        peak, peak_src = peaks()
        local_cells = self.geo.nx * self.ny
        alg_bytes = local_cells * ALG_BYTES_PER_CELL_SWEEP
        fused = kt.get("n_xy", 0) > 0 and kt["ms_xy"] >= max(kt["ms_x"], kt["ms_y"])
        if fused:
            which, label = "xy", "sweep_xy (fused step: column + row sweep in one launch)"
        else:
            which = "x" if kt["ms_x"] >= kt["ms_y"] else "y"
            label = f"sweep_{which}"
        n_launch = max(1, kt[f"n_{which}"])
        avg_ms = kt[f"ms_{which}"] / n_launch
        achieved = alg_bytes / (avg_ms / 1e3) / 1e9
        traffic = None
        prof = os.path.join(ROOT, "profiles", "traffic.json")
        tkey = f"{self.workload}_{self.flux}_{self.math}_sweep_{which}_dram_bytes_per_cell"
        if os.path.exists(prof):
            per_cell = json.load(open(prof)).get(tkey)
            if per_cell:
                traffic = per_cell * local_cells
        # whole time step: device time of all sweep kernels per time step
        n_steps = max(1, kt.get("n_xy", 0) + min(kt["n_x"], kt["n_y"]))
        step_ms = (kt["ms_x"] + kt["ms_y"] + kt.get("ms_xy", 0.0)) / n_steps
        moved = (local_cells * ALG_BYTES_PER_CELL_SWEEP *
                 (kt.get("n_xy", 0) + kt["n_x"] + kt["n_y"]) / n_steps)  # bytes the schedule must move
        survey = local_cells * 2 * ALG_BYTES_PER_CELL_SWEEP
        out = {"bound": "hbm", "kernel": label, "achieved": achieved,
               "peak": peak, "peak_source": peak_src, "unit": "GB/s",
               "frac": achieved / peak, "traffic": traffic,
               "traffic_source": f"profiles/traffic.json {tkey}" if traffic else None,
               "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": avg_ms,
               "peak_note": "the peak is a measured copy rate (torch b.copy_(a), MEASURED_PEAKS.json), "
                            "not the DRAM's nominal 8 TB/s: a streaming kernel can reach or slightly "
                            "exceed it (frac ~1.0)",
               "alg_bytes_note": "64 B per cell per launch: one read + one write of the 4 fp64 "
                                 "fields (a fused launch completes a whole cell-step with them)",
               "step": {"sweeps_ms_per_time_step": step_ms,
                        "achieved": moved / (step_ms / 1e3) / 1e9,
                        "frac": moved / (step_ms / 1e3) / 1e9 / peak,
                        "achieved_survey_128B": survey / (step_ms / 1e3) / 1e9,
                        "frac_survey_128B": survey / (step_ms / 1e3) / 1e9 / peak,
                        "note": "frac: bytes this schedule must move per time step (fused steps 64 "
                                "B/cell, split steps 128 B/cell) over the sweeps' device time; "
                                "frac_survey_128B: SURVEY 8d's two-sweep model (128 B per "
                                "cell-step), which the fused schedule undercuts by keeping U_b "
                                "on chip"}}
        fp = fp64_peak()
        if fp and fp.get("dfma_tflops"):
            flops = local_cells * FP64_FLOPS_PER_CELL_STEP / (step_ms / 1e3) / 1e12
            out["fp64"] = {"bound": "fp64", "achieved": flops, "unit": "TFLOP/s",
                           "peak": fp["dfma_tflops"], "frac": flops / fp["dfma_tflops"],
                           "flops_per_cell_step": FP64_FLOPS_PER_CELL_STEP,
                           "peak_source": "measured DFMA chain (profiles/fp64_peak.json)"}
        return out

    def host_buffers(self):
        """Pinned host planes of this rank's slab: the initial state (from the
        device initialiser, so every rank builds only its own slab) and the
        result."""
        torch = self.env.torch
        shape = (4, self.geo.nx + 4, self.ny + 4)
        h0 = torch.zeros(shape, dtype=torch.float64).pin_memory()
        h1 = torch.zeros(shape, dtype=torch.float64).pin_memory()
        self.grid.init_case(self.case, self.seed)
        self.sync()
        p0 = [h0[v].data_ptr() for v in range(4)]
        self.grid.download_ptr(p0, self.ny + 4)
        return h0, h1

    def e2e(self, h0, h1, steps, warmup):
        """End to end through the C-ABI: pinned host planes up, the run, the
        result down, every bench step (wall clock around synchronised steps,
        max over ranks)."""
        torch, env = self.env.torch, self.env
        p0 = [h0[v].data_ptr() for v in range(4)]
        p1 = [h1[v].data_ptr() for v in range(4)]

        def step():
            self.grid.upload_ptr(p0, self.ny + 4)
            if env.world == 1:
                self.grid.run(self.tsteps)
            else:
                self.S.run_slab(self.slab, self.comm, self.tsteps)
            self.grid.download_ptr(p1, self.ny + 4)

        for _ in range(max(1, warmup)):
            step()
        env.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            step()
        torch.cuda.synchronize()
        secs = env.allmax(time.perf_counter() - t0)
        nbytes = 4 * (self.geo.nx + 4) * (self.ny + 4) * 8
        return {"value": self.cells * self.tsteps * steps / secs, "unit": UNIT,
                "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes}

    def digest_of(self, planes_t) -> str | None:
        """The reference's grid digest of host planes held as row slabs
        (chained over ranks); on rank world-1 (returned by rank 0 via a
        broadcast-free send)."""
        env = self.env
        planes = planes_t.numpy()
        if env.world == 1:
            h = self.S.chained_digest(planes, self.geo.nx, self.ny, 0, 1, None, None)
            return f"{h:016x}"
        h = self.S.chained_digest(planes, self.geo.nx, self.ny, env.rank, env.world,
                                  env.send_u64, env.recv_u64)
        # hand the digest to rank 0
        if env.rank == env.world - 1:
            env.send_u64(h, 0)
        if env.rank == 0:
            return f"{env.recv_u64(env.world - 1):016x}"
        return None

    def final_digest(self) -> str | None:
        """Digest of the current device state (downloaded to a pinned buffer)."""
        torch = self.env.torch
        h = torch.zeros((4, self.geo.nx + 4, self.ny + 4), dtype=torch.float64).pin_memory()
        self.sync()
        self.grid.download_ptr([h[v].data_ptr() for v in range(4)], self.ny + 4)
        return self.digest_of(h)

    def max_rel_vs(self, other: "Measured") -> float:
        """compare_tolerance max_rel (proj/src/audit.cpp:137-154) of this run's
        final state against another's, on the device (hydro_gpu_compare), max
        over ranks."""
        self.sync()
        other.sync()
        return self.env.allmax(self.grid.compare(other.grid))


def measure_line(env, workload, flux, math, steps, warmup, *, e2e=True, clocks=None):
    """One measured configuration: device-resident value, per-kernel times +
    roofline, e2e, and the final state's parity (digest for bitwise runs).
    Returns (dict, Measured) -- the context stays open for comparisons."""
    m = Measured(env, workload, flux, math)
    ms, clock_info = m.device_timed(steps, warmup, clocks)
    value = m.cells * m.tsteps * steps / (ms / 1e3)
    kt = m.kernel_times(steps)
    out = {"value": value, "unit": UNIT, "steps": steps, "warmup": warmup,
           "ms_per_step": ms / steps,
           "config": workload_config(workload, m.global_nx, flux, math, env.world),
           "roofline": m.roofline(kt, clock_info),
           "kernel_ms": {"sweep_xy": kt["ms_xy"], "sweep_x": kt["ms_x"], "sweep_y": kt["ms_y"],
                         "other": kt["ms_other"],
                         "launches": {"sweep_xy": kt["n_xy"], "sweep_x": kt["n_x"],
                                      "sweep_y": kt["n_y"], "other": kt["n_other"]},
                         "note": "event-instrumented pass of the same K bench steps"},
           "schedule": {"ran": ("fused: one sweep_xy launch per time step (after one split step "
                                "when the step count is odd)" if kt["n_xy"] else
                                "split: sweep_x + sweep_y per time step"),
                        "how": "auto (hydro_gpu_set_schedule default): chosen from the context's "
                               "own completed (warm-up) runs -- the uniform-window share (fused "
                               ">= 0.6) and the event-timed step time of each schedule; bitwise "
                               "the same results",
                        "uniform_share_behind_choice": kt["auto_share"]},
           "gpu_launches": kt["n_xy"] + kt["n_x"] + kt["n_y"] + kt["n_other"] + steps,  # + init kernels
           "clocks": clock_info}
    if m.halo:
        out["config"]["halo"] = m.halo
        out["config"]["driver"] = m.driver
    local = m.geo.nx * m.ny
    out["uniform_window_identity"] = {
        "sweep_x": kt["skipped_x"] / max(1, local * (kt["n_x"] + kt["n_xy"])),
        "sweep_y": kt["skipped_y"] / max(1, local * (kt["n_y"] + kt["n_xy"])),
        "note": "share of cell updates the sweeps took by the uniform-window identity "
                "(DESIGN.md 3.1: the same bits as evaluating them, in either arithmetic)"}
    if kt.get("n_comm"):
        # device time of the per-step exchange (dt allreduce + inbox copy), max
        # over ranks: the communication the step exposes
        out["comm_us_per_step"] = env.allmax(1e3 * kt["ms_comm"] / kt["n_comm"])
    if e2e:
        h0, h1 = m.host_buffers()
        out["e2e"] = m.e2e(h0, h1, steps, warmup)
        m.e2e_buffers = (h0, h1)
        out["result_digest"] = m.digest_of(h1)
    else:  # the timing passes left the final state of a whole run on the device
        out["result_digest"] = m.final_digest()
    want = golden_digest(workload, flux, m.global_nx) if math == "bitwise" else None
    out["golden_digest"] = want
    if want and env.rank == 0 and out["result_digest"] != want:
        raise ParityFailure(f"{workload} {flux} {math}: result digest {out['result_digest']} "
                            f"!= the reference's {want}")
    return out, m


def tolerance_gate(env, tol_line, tol_m, bit_m):
    rel = tol_m.max_rel_vs(bit_m)
    tol_line["max_rel_vs_bitwise"] = rel
    tol_line["tolerance"] = TOLERANCE
    tol_line["parity"] = ("compare_tolerance max_rel against the bitwise state of the same run "
                          "(whose digest is the reference's)")
    if not rel <= TOLERANCE:
        raise ParityFailure(f"{tol_m.workload} {tol_m.flux} tolerance: max_rel {rel} > {TOLERANCE}")


def pipelined_e2e(env, m: Measured, steps):
    """The same end-to-end work (upload from pinned memory, run, download)
    for independent problems on two contexts and streams through the
    asynchronous C-ABI, so the copies of one overlap the other's kernels."""
    import paper_2106_13465_b200 as P
    torch = env.torch
    h0, h1 = m.e2e_buffers
    streams = [env.stream, torch.cuda.Stream()]
    g2 = P.GpuGrid(m.global_nx, m.ny, 1.0 / m.global_nx, 1.0 / m.ny, P.GasModel(), m.bc,
                   device=env.local, flux=m.flux, math=m.math)
    g2.set_stream(streams[1].cuda_stream)
    grids = [m.grid, g2]
    outs = [h1, torch.zeros_like(h0).pin_memory()]
    p0 = [h0[v].data_ptr() for v in range(4)]
    optrs = [[o[v].data_ptr() for v in range(4)] for o in outs]

    def pipe_step(k):
        g = grids[k & 1]
        g.upload_ptr_async(p0, m.ny + 4)
        g.run_async(m.tsteps)
        g.download_ptr_async(optrs[k & 1], m.ny + 4)

    for k in range(2):
        pipe_step(k)
    for g in grids:
        g.sync()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(steps):
        pipe_step(k)
    for g in grids:
        g.sync()
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    digest = m.digest_of(outs[(steps - 1) & 1])
    g2.close()
    nbytes = 4 * (m.geo.nx + 4) * (m.ny + 4) * 8
    return {"value": m.cells * m.tsteps * steps / secs, "unit": UNIT,
            "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "result_digest": digest,
            "note": "two contexts, alternating streams: hydro_gpu_upload_async / run_async / "
                    "download_async per step"}


def cpu_baseline_leg(workload, target_s=10.0):
    """The reference's CPU path on a bounded sample of the same workload: the
    first time steps of its run from the initial condition, about target_s of
    stepping, plus run_sequential on one core (the paper's starting point)."""
    from oracle import oracle as O
    case, nx, ny, bc, tsteps, seed, _ = WORKLOADS[workload]
    info = cpu_info()
    kind = "reference" if O.ref_available() else "port"
    strategy, threads = "sequential", 1
    if kind == "reference":
        strategy, threads = best_cpu_strategy(case, bc, seed, cpu_threads_options(info))
    # size the sample from a 2048^2 probe of the same strategy
    g = O.make_case(case, min(nx, 2048), min(ny, 2048), seed=seed)
    probe = (O.ref_run(g, 1, bc, strategy, threads) if kind == "reference"
             else _time_port(g, bc, 1))
    est = probe * (nx * ny) / (g.nx * g.ny)
    n = max(1, min(tsteps, int(target_s / max(est, 1e-9))))
    secs, kind, strategy, threads, _ = cpu_reference_run(case, nx, ny, bc, seed, [n], threads, strategy)
    out = {"value": nx * ny * n / secs[0], "unit": UNIT, "cores": threads, "kind": kind,
           "sample": f"time steps 1-{n} of the {nx}x{ny} {workload} run ({secs[0]:.1f}s stepping), "
                     f"reference {strategy} x{threads} (its fastest strategy/worker count here)",
           "cpu": info}
    if kind == "reference":
        g1 = O.make_case(case, min(nx, 2048), min(ny, 2048), seed=seed)
        O.ref_run(g1, 1, bc, "sequential", 1)
        s1 = O.ref_run(g1, 2, bc, "sequential", 1)
        out["sequential_1core"] = {"value": g1.nx * g1.ny * 2 / s1, "unit": UNIT, "cores": 1,
                                   "sample": f"2 time steps of a {g1.nx}x{g1.ny} {case} grid, "
                                             "reference run_sequential"}
    return out


def dropin_e2e(workload, math, flux="hllc"):
    """The reference's own caller through the drop-in: run_benchmark's protocol
    (proj/src/bench.cpp:92-152 -- one untimed warm-up step from a copy of the
    initial grid, then the timed run) in integration/_build/hydrobench_gpu,
    whose `gpu` strategy is hydro::run_gpu on the caller's pageable Grid2D
    (include/hydro/gpu_strategy.hpp: cached context, pinned staging).  The
    timed run includes the upload and download of the grid's planes."""
    exe = os.path.join(ROOT, "integration", "_build", "hydrobench_gpu")
    if not os.path.exists(exe):
        return None
    case, nx, ny, bc, tsteps, seed, _ = WORKLOADS[workload]
    cmd = [exe, "bench", "--case", case, "--nx", str(nx), "--ny", str(ny), "--steps", str(tsteps),
           "--strategy", "gpu", "--bc", bc, "--seed", str(seed), "--flux", flux, "--math", math]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    if out.returncode != 0:
        raise ParityFailure(f"hydrobench_gpu failed: {out.stderr.strip()[-300:]}")
    rate, digest = None, None
    for line in out.stdout.splitlines():
        if line.startswith("#") and "cell-steps/s" in line:
            rate = float(line.split()[1])
        elif line[:1].isdigit() and line.count(",") == 4:
            digest = line.rsplit(",", 1)[1].strip()
    nbytes = 4 * (nx + 4) * (ny + 4) * 8
    return {"value": rate, "unit": UNIT, "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
            "result_digest": digest, "math": math,
            "how": "integration/_build/hydrobench_gpu bench --strategy gpu: the reference's "
                   "run_benchmark protocol, hydro::run_gpu on pageable Grid2D planes "
                   "(one timed run incl. upload + download)"}


def _time_port(g, bc, steps):
    from oracle import oracle as O
    t0 = time.perf_counter()
    O.run_sequential(g, steps, bc)
    return time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS),
                    help="BASELINE config (default cfg3, the metric's config)")
    ap.add_argument("--flux", default="hllc", choices=["hllc", "exact10"],
                    help="interface flux (hllc = the reference hot path)")
    ap.add_argument("--math", default="tolerance", choices=["bitwise", "tolerance"],
                    help="sweep arithmetic of the headline (tolerance = the north star's bar, "
                         "compare_tolerance max_rel <= 1e-12 against the bitwise state, gated "
                         "live; bitwise = the reference's bits, digest-gated, always measured "
                         "beside it)")
    ap.add_argument("--no-variants", action="store_true",
                    help="skip the other math mode / exact-10 / secondary configs")
    args = ap.parse_args()
    rank, world, _ = dist_env()

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    assert torch.cuda.is_available(), "bench.py needs a CUDA device"
    env = Env(args)
    other_math = "tolerance" if args.math == "bitwise" else "bitwise"
    try:
        clocks = ClockSampler(env.local)
        head, hm = measure_line(env, args.workload, args.flux, args.math, args.steps, args.warmup,
                                clocks=clocks)
        e2e_pipe = pipelined_e2e(env, hm, args.steps) if world == 1 else None
        mvariants, fvariants, secondary = {}, {}, {}
        vsteps = max(1, min(args.steps, 5))
        if not args.no_variants or args.math == "tolerance":
            # the other math mode on the same workload; a tolerance line is
            # gated against the bitwise state
            ov, om = measure_line(env, args.workload, args.flux, other_math,
                                  args.steps if args.math == "tolerance" else vsteps, args.warmup,
                                  e2e=not args.no_variants)
            bit_m, tol_m = (hm, om) if args.math == "bitwise" else (om, hm)
            tolerance_gate(env, ov if args.math == "bitwise" else head, tol_m, bit_m)
            if args.math == "tolerance":
                head["bitwise_digest"] = ov["result_digest"]
            mvariants[other_math] = ov
            om.close()
        if not args.no_variants and args.flux == "hllc":
            for vm in (args.math, other_math):
                v, vmm = measure_line(env, args.workload, "exact10", vm, vsteps, args.warmup,
                                      e2e=False)
                v["note"] = "BASELINE's stated solver: exact Riemann flux, 10 Newton iterations (DESIGN.md 3.4)"
                fvariants[f"exact10_{vm}"] = (v, vmm)
            b = fvariants[f"exact10_bitwise"][1]
            t_line, t_m = fvariants["exact10_tolerance"]
            tolerance_gate(env, t_line, t_m, b)
            for k in list(fvariants):
                fvariants[k][1].close()
                fvariants[k] = fvariants[k][0]
        if not args.no_variants and world == 1:
            for wl in SECONDARY:
                if wl == args.workload:
                    continue
                lines = {}
                ms = {}
                for vm in ("bitwise", "tolerance"):
                    lines[vm], ms[vm] = measure_line(env, wl, args.flux, vm, vsteps, args.warmup,
                                                     e2e=False)
                tolerance_gate(env, lines["tolerance"], ms["tolerance"], ms["bitwise"])
                for x in ms.values():
                    x.close()
                secondary[wl] = lines
    except ParityFailure as e:
        print(f"bench.py: PARITY FAILURE -- {e}", file=sys.stderr, flush=True)
        sys.exit(1)

    cpu = dropin = None
    if rank == 0 and world == 1 and not args.no_variants:
        try:
            dropin = dropin_e2e(args.workload, args.math, args.flux)
            if dropin and args.math == "bitwise":
                want = golden_digest(args.workload, args.flux, hm.global_nx)
                if want and dropin["result_digest"] != want:
                    raise ParityFailure(f"drop-in digest {dropin['result_digest']} != {want}")
        except ParityFailure as e:
            print(f"bench.py: PARITY FAILURE -- {e}", file=sys.stderr, flush=True)
            sys.exit(1)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_leg(args.workload)

    if rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": hm.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (analytic or seeded initial condition, no dataset)",
            "config": dict(head["config"], l2="inputs larger than L2 (2 x %.0f MB state per GPU)"
                           % (4 * (hm.geo.nx + 4) * (hm.ny + 4) * 8 / 1e6)),
            "roofline": head["roofline"],
            "e2e": head["e2e"],
            "e2e_pipelined": e2e_pipe,
            "e2e_dropin": dropin,
            "gpu_launches": head["gpu_launches"],
            "kernel_ms": head["kernel_ms"],
            "schedule": head["schedule"],
            "comm_us_per_step": head.get("comm_us_per_step"),
            "uniform_window_identity": head.get("uniform_window_identity"),
            "clocks": head["clocks"],
            "cpu_baseline": cpu,
            "result_digest": head["result_digest"],
            "golden_digest": head["golden_digest"],
            "parity": ("digest == the reference's (bench.cpp:131-143 gate)" if args.math == "bitwise"
                       else f"max_rel {head.get('max_rel_vs_bitwise')} <= {TOLERANCE} vs the "
                            f"bitwise state (digest {head.get('bitwise_digest')})"),
            "max_rel_vs_bitwise": head.get("max_rel_vs_bitwise"),
            "bitwise_digest": head.get("bitwise_digest") if args.math == "tolerance"
            else head["result_digest"],
            "math_variants": mvariants or None,
            "flux_variants": fvariants or None,
            "secondary": secondary or None,
        }
        print(json.dumps(line), flush=True)
    if env.dist is not None:
        env.dist.destroy_process_group()


if __name__ == "__main__":
    main()
