"""Fused vs split schedule on the GPU: bitwise equality of every plane (ghosts
included) and the last dt, then event-timed ms per step of both schedules.

    python tools/fused_check.py [--quick]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_13465_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--quick", action="store_true")
ap.add_argument("--time", nargs="*", default=["cfg3", "cfg2", "cfg1"])
a = ap.parse_args()

model = P.GasModel()


def run(nx, ny, case, bc, steps, math, schedule, seed=0, flux="hllc", seg=0, splits=(None,)):
    with P.GpuGrid(nx, ny, 1.0 / nx, 1.0 / ny, model, bc, device=0, flux=flux, math=math) as g:
        g.set_schedule(schedule, seg)
        g.init_case(case, seed)
        dts = []
        for k in splits:
            dts.append(g.run(k if k else steps))
        grid = P.Grid2D(nx, ny, 1.0 / nx, 1.0 / ny)
        g.download(grid.planes)
        return grid.planes.copy(), dts


cases = [
    (64, 64, "corner_blast", "reflect", 10),
    (96, 160, "random", "transmit", 9),
    (130, 250, "random", "reflect", 7),
    (33, 241, "sod_x", "transmit", 12),
    (257, 121, "corner_blast", "reflect", 6),
    (300, 97, "random", "transmit", 5),
    (4, 40, "random", "transmit", 5),
    (512, 512, "corner_blast", "reflect", 20),
    (1000, 1000, "random", "transmit", 8),
]
if a.quick:
    cases = cases[:4]
bad = 0
for nx, ny, case, bc, steps in cases:
    for math in ("bitwise", "tolerance"):
        for seg in (0, 16):
            t0 = time.time()
            ps, ds = run(nx, ny, case, bc, steps, math, "split", seed=7)
            pf, df = run(nx, ny, case, bc, steps, math, "fused", seed=7, seg=seg)
            same = np.array_equal(ps.view(np.uint64), pf.view(np.uint64)) and ds == df
            if not same:
                bad += 1
                diff = np.argwhere(ps.view(np.uint64) != pf.view(np.uint64))
                print(f"MISMATCH {nx}x{ny} {case} {bc} {steps} {math} seg={seg}: "
                      f"{len(diff)} cells, first {diff[:6].tolist()} dt {ds} {df}", flush=True)
            else:
                print(f"ok {nx}x{ny} {case} {bc} steps={steps} {math} seg={seg} "
                      f"({time.time() - t0:.1f}s)", flush=True)
# split runs (run 3 + run 4 = run 7) and a run of 2 steps
for math in ("bitwise", "tolerance"):
    ps, ds = run(200, 180, "random", "reflect", 7, math, "split", seed=3)
    pf, df = run(200, 180, "random", "reflect", 7, math, "fused", seed=3, splits=(3, 4))
    print("split 3+4:", "ok" if np.array_equal(ps, pf) and ds[-1] == df[-1] else "MISMATCH", flush=True)
    bad += 0 if np.array_equal(ps, pf) else 1
print("mismatches:", bad, flush=True)

WL = {"cfg3": (16384, "corner_blast", "reflect", 50), "cfg2": (8192, "random", "transmit", 50),
      "cfg1": (2048, "sod_x", "transmit", 200), "cfg4": (16384, "random", "transmit", 20)}
for w in a.time:
    n, case, bc, steps = WL[w]
    for math in ("tolerance", "bitwise"):
        res = {}
        for sch in ("split", "fused"):
            with P.GpuGrid(n, n, 1.0 / n, 1.0 / n, model, bc, device=0, math=math) as g:
                g.set_schedule(sch)
                g.init_case(case, 2106 if case == "random" else 0)
                g.run(steps)  # warm-up (graph capture)
                g.init_case(case, 2106 if case == "random" else 0)
                g.set_timing(True)
                g.reset_counters()
                g.run(steps)
                kt = g.kernel_times()
                fm, fn = g.fused_times()
                h = g.state_hash()
            tot = kt["ms_x"] + kt["ms_y"] + kt["ms_other"] + fm
            res[sch] = (tot, h)
            print(f"{w} {math} {sch}: {tot:.2f} ms for {steps} steps ({tot / steps:.3f} ms/step; "
                  f"fused {fn} x {fm / max(fn, 1):.3f} ms, x {kt['n_x']} x "
                  f"{kt['ms_x'] / max(kt['n_x'], 1):.3f}, y {kt['ms_y'] / max(kt['n_y'], 1):.3f}) "
                  f"hash {h:016x}", flush=True)
        print(f"{w} {math}: speed-up {res['split'][0] / res['fused'][0]:.3f}x, hashes "
              f"{'equal' if res['split'][1] == res['fused'][1] else 'DIFFER'}", flush=True)
