"""Benchmark of the B200 HYDRO step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (N=1): BASELINE config 1 -- 2048x2048 fp64 Sod shock along x,
transmissive boundaries, gamma 1.4, CFL 0.8, MUSCL-Hancock + minmod + HLLC
(the reference's hot-path flux), 200 time steps.  One bench "step" is one
such 200-time-step run from the initial condition.  For N>1 the grid grows
along i by N (weak scaling: each rank holds a 2048x2048 row slab, halo swap
+ dt min-allreduce over NCCL every time step).

Metric: cell-updates/s = interior cells x time steps / seconds (both sweeps +
the dt reduction per time step).  ``value`` is device-resident (state in HBM
before the timed region, CUDA events on the launch stream, max over ranks);
``e2e`` goes through the C-ABI with pinned host buffers: upload, run, download
every bench step.  An hllc run also measures the exact-10 flux mode (BASELINE's
stated solver) on the same workload under ``flux_variants``, and a bitwise run
the tolerance math mode (``--math tolerance``: compare_tolerance max_rel <=
1e-12 instead of bit-identical) under ``math_variants``, with
its measured max_rel against the bitwise result.
``--impl reference`` times the reference's own CPU
implementation (oracle/_ref, its fastest strategy over all host threads) on a
bounded sample of the same workload.
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

# BASELINE.json configs: name -> (case, nx per GPU, ny, bc,
# time steps per bench step, seed, scaling when --gpus > 1)
WORKLOADS = {
    "cfg0": ("corner_blast", 256, 256, "reflect", 100, 0, "weak"),
    "cfg1": ("sod_x", 2048, 2048, "transmit", 200, 0, "weak"),
    "cfg2": ("random", 8192, 8192, "transmit", 50, 2106, "weak"),
    "cfg3": ("corner_blast", 16384, 16384, "reflect", 50, 0, "strong"),
    "cfg4": ("random", 16384, 16384, "transmit", 20, 13465, "weak"),
}
NX = NY = 2048
TSTEPS = 200
CASE, BC = "sod_x", "transmit"
SEED = 0
SCALING = "weak"
METRIC = "cell-updates/s (both sweeps, fp64)"
UNIT = "cell-updates/s"
ALG_BYTES_PER_CELL_SWEEP = 64  # 32 B read + 32 B write of 4 fp64 fields


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


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
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


_BEST_STRATEGY = None


def best_cpu_strategy(threads: int) -> str:
    """The reference's fastest parallel strategy on this host (bench.cpp:53-90
    dispatch): a short probe of fine_grain / coarse_grain / task_graph at
    `threads` workers on the workload grid."""
    global _BEST_STRATEGY
    if _BEST_STRATEGY is None:
        from oracle import oracle as O
        g = O.make_case(CASE, NX, NY, seed=SEED)
        rates = {}
        for strat in ("coarse_grain", "fine_grain", "task_graph"):
            h = g.copy()
            O.ref_run(h, 1, BC, strat, threads)  # warm-up (bench.cpp:112-117)
            secs = O.ref_run(h, 3, BC, strat, threads)
            rates[strat] = 3 / secs
        _BEST_STRATEGY = max(rates, key=rates.get)
    return _BEST_STRATEGY


def cpu_reference_sample(steps_per_chunk: int, threads: int, min_seconds: float = 0.0,
                         strategy: str | None = None):
    """Times the reference's own CPU path (oracle/_ref, its fastest parallel
    strategy over `threads` host threads) -- or the C port if the compiled
    reference is absent -- on chunks of `steps_per_chunk` time steps of the
    workload, continuing the same flow until at least `min_seconds` of
    stepping was timed.  Returns (cell-steps/s, kind, seconds, threads, steps,
    strategy)."""
    from oracle import oracle as O
    g = O.make_case(CASE, NX, NY, seed=SEED)
    kind = "reference" if O.ref_available() else "port"
    strat = "sequential"
    if kind == "reference":
        strat = strategy or best_cpu_strategy(threads)
        if strat == "sequential":
            threads = 1
        O.ref_run(g.copy(), 1, BC, strat, threads)  # warm-up (bench.cpp:112-117)
    else:
        threads = 1
    secs, steps = 0.0, 0
    while steps == 0 or secs < min_seconds:
        if kind == "reference":
            secs += O.ref_run(g, steps_per_chunk, BC, strat, threads)
        else:
            t0 = time.perf_counter()
            O.run_sequential(g, steps_per_chunk, BC)
            secs += time.perf_counter() - t0
        steps += steps_per_chunk
    return NX * NY * steps / secs, kind, secs, threads, steps, strat


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    sample_steps = 20
    vals, kind = [], None
    for k in range(args.warmup + args.steps):
        v, kind, secs, used, _, strat = cpu_reference_sample(sample_steps, threads)
        if k >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": NX * NY * sample_steps / value * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (analytic or seeded initial condition, no dataset)",
        "config": {"workload": f"BASELINE {args.workload} sample: {NX}x{NY} {CASE} {BC}, "
                               f"{sample_steps} time steps per bench step",
                   "cells": NX * NY, "time_steps_per_bench_step": sample_steps,
                   "parallelism": f"cpu {strat} x{used}"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": kind,
                         "sample": f"{sample_steps} time steps of the {NX}x{NY} {args.workload} grid, "
                                   f"reference {strat} (its fastest strategy here, "
                                   "bench.cpp:53-90 dispatch)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def max_rel(a, b, rows: int = 1024) -> float:
    """compare_tolerance's max |a-b| / max(|a|,|b|,1) (proj/src/audit.cpp:146)
    over (4, nx, ny) planes, in row blocks to bound host memory."""
    import numpy as np
    out = 0.0
    for i in range(0, a.shape[1], rows):
        x, y = a[:, i:i + rows], b[:, i:i + rows]
        out = max(out, float((np.abs(x - y) / np.maximum(np.maximum(np.abs(x), np.abs(y)), 1.0)).max()))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="cfg1", choices=sorted(WORKLOADS),
                    help="BASELINE config (default cfg1, the metric's config)")
    ap.add_argument("--flux", default="hllc", choices=["hllc", "exact10"],
                    help="interface flux (hllc = the reference hot path)")
    ap.add_argument("--math", default="bitwise", choices=["bitwise", "tolerance"],
                    help="sweep arithmetic (bitwise = the reference's bits)")
    ap.add_argument("--no-variants", action="store_true",
                    help="skip the exact-10 flux / tolerance-math sub-measurements")
    args = ap.parse_args()
    global NX, NY, TSTEPS, CASE, BC, SEED, SCALING
    CASE, NX, NY, BC, TSTEPS, SEED, SCALING = WORKLOADS[args.workload]
    rank, world, local = dist_env()

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import numpy as np
    import torch

    import paper_2106_13465_b200 as P
    from paper_2106_13465_b200 import slab as S

    assert torch.cuda.is_available(), "bench.py needs a CUDA device"
    # HYDRO_BENCH_SHARED_GPU=1: code-path check of the N>1 bench on a 1-GPU box
    # (every rank on cuda:0, gloo for the host-side dt allreduce, so no kernel
    # waits on another rank) -- its numbers are not measurements
    shared = world > 1 and os.environ.get("HYDRO_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    model = P.GasModel()
    # weak scaling grows the slab axis i by the GPU count;
    # strong scaling splits one grid
    global_nx = NX * world if SCALING == "weak" else NX
    dx, dy = 1.0 / global_nx, 1.0 / NY
    stream = torch.cuda.Stream()  # a real stream: library kernels, NCCL and events share it
    torch.cuda.set_stream(stream)

    geo = S.SlabGeometry(global_nx, NY, rank, world)
    if world == 1:
        grid = P.GpuGrid(NX, NY, dx, dy, model, BC, device=local, flux=args.flux, math=args.math)
        grid.set_stream(stream.cuda_stream)
        slab = None
    else:
        slab = S.GpuSlab(geo, dx, dy, model, BC, local, flux=args.flux, math=args.math)
        slab.bind_stream(stream)
        grid = slab.grid
        comm = S.TorchComm()
        comm.setup_p2p(slab)  # peer-memory halo over NVLink if every rank can map its peers

    def one_step():
        grid.init_case(CASE, SEED)
        if world == 1:
            grid.run_async(TSTEPS)
        else:
            S.run_slab(slab, comm, TSTEPS)

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        one_step()
    if world == 1:
        grid.sync()
    torch.cuda.synchronize()

    # ---- device-resident timed region -----------------------------------
    # Clean replays (the per-step launch pairs run as one CUDA graph); the
    # per-kernel durations for the roofline come from a second, event-
    # instrumented pass of the same K steps below, because event nodes inside
    # the graph perturb the timing they measure.
    clocks = ClockSampler(local)
    grid.set_timing(False)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        one_step()
    e1.record(stream)
    torch.cuda.synchronize()
    clock_info = clocks.stop()
    if world == 1:
        grid.sync()
    barrier()
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    cells = global_nx * NY
    value = cells * TSTEPS * args.steps / (ms / 1e3)

    # ---- per-kernel device time (CUDA events around every launch) ----------
    grid.reset_counters()
    grid.set_timing(True)
    for _ in range(args.steps):
        one_step()
    torch.cuda.synchronize()
    kt = grid.kernel_times()
    grid.set_timing(False)
    launches = kt["n_x"] + kt["n_y"] + kt["n_other"] + args.steps  # + init kernels

    # ---- end-to-end through the C-ABI with pinned host buffers --------------
    host0 = torch.zeros((4, geo.nx + 4, NY + 4), dtype=torch.float64).pin_memory()
    host = torch.zeros_like(host0).pin_memory()
    init = P.make_case(CASE, global_nx, NY, model, seed=SEED) if world == 1 else None
    if init is not None:
        host0.copy_(torch.from_numpy(init.planes))
    else:
        full = P.make_case(CASE, global_nx, NY, model, seed=SEED)
        host0.copy_(torch.from_numpy(S.slab_planes(full.planes, global_nx, world, rank)))
        del full
    ptrs0 = [host0[v].data_ptr() for v in range(4)]
    ptrs = [host[v].data_ptr() for v in range(4)]

    def e2e_step():
        grid.upload_ptr(ptrs0, NY + 4)
        if world == 1:
            grid.run(TSTEPS)
        else:
            S.run_slab(slab, comm, TSTEPS)
        grid.download_ptr(ptrs, NY + 4)

    for _ in range(max(1, args.warmup)):
        e2e_step()
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = cells * TSTEPS * args.steps / e2e_s
    plane_bytes = 4 * (geo.nx + 4) * (NY + 4) * 8

    # ---- the same end-to-end work pipelined over two contexts -------------
    # Independent problems through the asynchronous C-ABI
    # (hydro_gpu_upload_async / run_async / download_async): each bench step
    # still uploads its inputs from pinned memory, runs and downloads its
    # result, but on alternating contexts and streams, so the copies of one
    # overlap the other's kernels.
    e2e_pipe = None
    if world == 1:
        streams = [stream, torch.cuda.Stream()]
        grids = [grid, P.GpuGrid(NX, NY, dx, dy, model, BC, device=local, flux=args.flux,
                                 math=args.math)]
        grids[1].set_stream(streams[1].cuda_stream)
        outs = [host, torch.zeros_like(host0).pin_memory()]
        optrs = [[o[v].data_ptr() for v in range(4)] for o in outs]

        def pipe_step(k):
            g2, st = grids[k & 1], streams[k & 1]
            g2.upload_ptr_async(ptrs0, NY + 4)
            g2.run_async(TSTEPS)
            g2.download_ptr_async(optrs[k & 1], NY + 4)

        for k in range(2):
            pipe_step(k)
        for g2 in grids:
            g2.sync()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(args.steps):
            pipe_step(k)
        for g2 in grids:
            g2.sync()
        torch.cuda.synchronize()
        pipe_s = time.perf_counter() - t0
        last = outs[(args.steps - 1) & 1].numpy()
        e2e_pipe = {"value": cells * TSTEPS * args.steps / pipe_s, "unit": UNIT,
                    "h2d_bytes_per_step": plane_bytes, "d2h_bytes_per_step": plane_bytes,
                    "result_digest": f"{P.grid_digest(P.Grid2D(NX, NY, dx, dy, last)):016x}",
                    "note": "two contexts, alternating streams: hydro_gpu_upload_async / "
                            "run_async / download_async per step"}
        grids[1].close()

    # result check of the e2e leg against the digest of the first run
    digest = P.grid_digest(P.Grid2D(geo.nx, NY, dx, dy, host.numpy())) if world == 1 else None

    # ---- roofline of the dominant sweep kernel ------------------------------
    peak, peak_src = peaks()
    which = "x" if kt["ms_x"] >= kt["ms_y"] else "y"
    n_launch = max(1, kt[f"n_{which}"])
    avg_ms = kt[f"ms_{which}"] / n_launch
    alg_bytes = geo.nx * NY * ALG_BYTES_PER_CELL_SWEEP
    achieved = alg_bytes / (avg_ms / 1e3) / 1e9
    # measured DRAM bytes per cell of that sweep (ncu --set full capture,
    # profiles/traffic.json), scaled to this launch's cells
    traffic = None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        per_cell = json.load(open(prof)).get(f"sweep_{which}_dram_bytes_per_cell")
        if per_cell:
            traffic = per_cell * geo.nx * NY

    # the bound that actually binds: FP64-pipe lane
    # instructions of that kernel per cell (ncu, config 1 / hllc only) over
    # 148 SMs x 64 FP64 lanes x the SM clock sampled during the timed region
    fp64 = None
    if os.path.exists(prof) and args.workload == "cfg1" and args.flux == "hllc" and args.math == "bitwise":
        per_cell = json.load(open(prof)).get(f"sweep_{which}_fp64_instr_per_cell")
        sms = torch.cuda.get_device_properties(local).multi_processor_count
        mhz = (clock_info or {}).get("sm_mhz") or 1965.0
        if per_cell:
            ach = per_cell * geo.nx * NY / (avg_ms / 1e3)
            pk = sms * 64 * mhz * 1e6
            fp64 = {"bound": "fp64", "achieved": ach, "peak": pk, "unit": "FP64 lane-instr/s",
                    "frac": ach / pk, "instr_per_cell": per_cell,
                    "peak_source": f"{sms} SMs x 64 FP64 lanes x {mhz:.0f} MHz (sampled)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, kind, secs, used, nsteps, strat = cpu_reference_sample(10, threads, min_seconds=10.0)
        cpu = {"value": v, "unit": UNIT, "cores": used, "kind": kind,
               "sample": f"{nsteps} time steps of the {NX}x{NY} {args.workload} grid ({secs:.1f}s timed), "
                         f"reference {strat} (its fastest strategy here) over {used} host threads"}
        if kind == "reference":  # the paper's single-core starting point, run_sequential
            v1, _, secs1, _, n1, _ = cpu_reference_sample(2, 1, min_seconds=3.0,
                                                          strategy="sequential")
            cpu["sequential_1core"] = {
                "value": v1, "unit": UNIT, "cores": 1,
                "sample": f"{n1} time steps, reference run_sequential ({secs1:.1f}s timed)"}

    # ---- variants on the same workload, same protocol, reported beside the
    # headline line: the other flux of BASELINE's configs (exact Riemann, 10
    # Newton iterations) and the tolerance math mode ---------------------------
    vhost = torch.zeros_like(host0).pin_memory()
    vptrs = [vhost[v].data_ptr() for v in range(4)]

    def variant(vflux, vmath):
        if world == 1:
            vgrid = P.GpuGrid(NX, NY, dx, dy, model, BC, device=local, flux=vflux, math=vmath)
            vgrid.set_stream(stream.cuda_stream)
            vslab = None
        else:
            vslab = S.GpuSlab(geo, dx, dy, model, BC, local, flux=vflux, math=vmath)
            vslab.bind_stream(stream)
            vgrid = vslab.grid
            comm.setup_p2p(vslab)

        def vrun():
            if world == 1:
                vgrid.run_async(TSTEPS)
            else:
                S.run_slab(vslab, comm, TSTEPS)

        vsteps = max(1, min(args.steps, 5))
        for _ in range(args.warmup):
            vgrid.init_case(CASE, SEED)
            vrun()
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(vsteps):
            vgrid.init_case(CASE, SEED)
            vrun()
        e1.record(stream)
        torch.cuda.synchronize()
        vms = e0.elapsed_time(e1)
        barrier()
        t0 = time.perf_counter()
        for _ in range(vsteps):
            vgrid.upload_ptr(ptrs0, NY + 4)
            vrun()
            vgrid.download_ptr(vptrs, NY + 4)
        torch.cuda.synchronize()
        ve2e = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([vms, ve2e], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            vms, ve2e = float(t[0].item()), float(t[1].item())
        vgrid.close()
        vdigest = (P.grid_digest(P.Grid2D(geo.nx, NY, dx, dy, vhost.numpy()))
                   if world == 1 else None)
        return {"value": cells * TSTEPS * vsteps / (vms / 1e3), "unit": UNIT,
                "steps": vsteps, "warmup": args.warmup, "ms_per_step": vms / vsteps,
                "e2e": {"value": cells * TSTEPS * vsteps / ve2e, "unit": UNIT,
                        "h2d_bytes_per_step": plane_bytes, "d2h_bytes_per_step": plane_bytes},
                "result_digest": f"{vdigest:016x}" if vdigest is not None else None}

    variants = mvariants = None
    if args.flux == "hllc" and not args.no_variants:
        v = variant("exact10", args.math)
        v["note"] = ("BASELINE's stated solver: exact Riemann flux, 10 Newton iterations "
                     "(DESIGN.md 3.4)" + ("; bitwise equal to the oracle's restatement"
                                          if args.math == "bitwise" else ""))
        variants = {"exact10": v}
        # kept for the tolerance/exact-10 comparison below (small grids only)
        ex_state = vhost.numpy()[:, 2:geo.nx + 2, 2:NY + 2].copy() if geo.nx * NY <= (1 << 26) else None
    if args.math == "bitwise" and not args.no_variants:
        v = variant(args.flux, "tolerance")
        # the tolerance run's final state against the bitwise one (this rank's
        # slab; the bitwise result carries the reference's digest)
        rel = max_rel(host.numpy()[:, 2:geo.nx + 2, 2:NY + 2], vhost.numpy()[:, 2:geo.nx + 2, 2:NY + 2])
        if dist is not None:
            t = torch.tensor([rel], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            rel = float(t.item())
        v["max_rel_vs_bitwise"] = rel
        v["tolerance"] = 1e-12
        v["note"] = ("tolerance math mode (hydro_gpu_set_math, DESIGN.md 3.6): uncorrected "
                     "reciprocal quotients and square roots; compare_tolerance max_rel against the bitwise "
                     "result of this run (the reference's state) <= 1e-12")
        mvariants = {"tolerance": v}
        if args.flux == "hllc" and variants:
            v = variant("exact10", "tolerance")
            v["note"] = "tolerance math mode with the exact-10 flux (DESIGN.md 3.6)"
            if ex_state is not None and world == 1:
                v["max_rel_vs_bitwise"] = max_rel(ex_state, vhost.numpy()[:, 2:geo.nx + 2, 2:NY + 2])
            mvariants["tolerance_exact10"] = v

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": SCALING, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (analytic or seeded initial condition, no dataset)",
            "config": {"workload": f"BASELINE {args.workload}: {global_nx}x{NY} {CASE} {BC}, "
                                   f"{args.flux}, {TSTEPS} time steps per bench step",
                       "cells": cells, "time_steps_per_bench_step": TSTEPS,
                       "parallelism": f"row slabs x{world}" if world > 1 else "single GPU",
                       "halo": (("peer-memory (row-sweep stores into neighbour inboxes)"
                                 if comm.p2p else "nccl send/recv") if world > 1 else None),
                       "l2": "inputs larger than L2 (2 x %.0f MB state per GPU)"
                             % (4 * (geo.nx + 4) * (NY + 4) * 8 / 1e6),
                       "flux": args.flux, "math": args.math, "seed": SEED},
            "roofline": {"bound": "hbm", "kernel": f"sweep_{which}", "achieved": achieved,
                         "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": avg_ms,
                         "fp64_pipe": fp64},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": plane_bytes,
                    "d2h_bytes_per_step": plane_bytes},
            "e2e_pipelined": e2e_pipe,
            "gpu_launches": launches,
            "kernel_ms": {"sweep_x": kt["ms_x"], "sweep_y": kt["ms_y"], "other": kt["ms_other"],
                          "note": "event-instrumented pass of the same K bench steps"},
            "clocks": clock_info,
            "cpu_baseline": cpu,
            "result_digest": f"{digest:016x}" if digest is not None else None,
            "flux_variants": variants,
            "math_variants": mvariants,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
