"""Sweep times and uniform-window identity counts on BASELINE grids (tools
only, not a benchmark).  python tools/ab_skip.py cfg3 [tolerance]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_13465_b200 as P  # noqa: E402
from bench import WORKLOADS  # noqa: E402

cfg = sys.argv[1]
math = sys.argv[2] if len(sys.argv) > 2 else "bitwise"
flux = sys.argv[3] if len(sys.argv) > 3 else "hllc"
case, nx, ny, bc, ts, seed, _ = WORKLOADS[cfg]
with P.GpuGrid(nx, ny, 1.0 / nx, 1.0 / ny, P.GasModel(), bc, device=0, math=math,
               flux=flux) as g:
    g.init_case(case, seed)
    g.run(3)
    g.reset_counters()
    g.set_timing(True)
    g.run(ts - 3)
    t = g.kernel_times()
    sx, sy = g.skipped()
    cells = nx * ny * t["n_x"]
    print(f"{cfg} {math} {flux}: x {t['ms_x'] / t['n_x']:.4f} ms  y {t['ms_y'] / t['n_y']:.4f} ms  "
          f"skipped x {sx / cells:.4f} y {sy / cells:.4f}", flush=True)
