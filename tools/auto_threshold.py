"""Fused vs split step time against the uniform-window share, on a corner blast
growing through a 2048^2 grid (the data behind the AUTO schedule's threshold;
not a benchmark).    python tools/auto_threshold.py [--math tolerance]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_13465_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--math", default="tolerance")
ap.add_argument("--n", type=int, default=2048)
ap.add_argument("--marks", type=int, nargs="*", default=[200, 600, 1000, 1400, 1800, 2400, 3000])
a = ap.parse_args()
n = a.n
res = {}
for sch in ("split", "fused"):
    with P.GpuGrid(n, n, 1.0 / n, 1.0 / n, P.GasModel(), "reflect", device=0, math=a.math) as g:
        g.set_schedule(sch)
        g.init_case("corner_blast", 0)
        done = 0
        for mark in a.marks:
            g.run(mark - done - 20)
            g.reset_counters()
            g.set_timing(True)
            g.run(20)
            kt = g.kernel_times()
            fm, fn = g.fused_times()
            sx, sy = g.skipped()
            g.set_timing(False)
            done = mark
            ms = (kt["ms_x"] + kt["ms_y"] + fm) / 20
            share = (sx + sy) / (2.0 * 20 * n * n)
            res.setdefault(mark, {})[sch] = (ms, share)
for mark, r in res.items():
    print(f"step {mark:5d}: uniform share {r['split'][1]:.3f} (split count) / {r['fused'][1]:.3f} (fused count)  "
          f"split {r['split'][0]:.4f} ms  fused {r['fused'][0]:.4f} ms  fused/split {r['fused'][0] / r['split'][0]:.3f}")
