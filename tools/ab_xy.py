"""Separate x / y launch geometry sweeps (segment length, claim band) on a
BASELINE grid (tools only, not a benchmark).
    python tools/ab_xy.py cfg3 tolerance "sx,bx;..." "sy,by;..." """
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_13465_b200 as P  # noqa: E402
from bench import WORKLOADS  # noqa: E402

cfg, math, xs, ys = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
case, nx, ny, bc, ts, seed, _ = WORKLOADS[cfg]
xo = [tuple(int(v) for v in p.split(",")) for p in xs.split(";")]
yo = [tuple(int(v) for v in p.split(",")) for p in ys.split(";")]
n = max(len(xo), len(yo))
with P.GpuGrid(nx, ny, 1.0 / nx, 1.0 / ny, P.GasModel(), bc, device=0, math=math) as g:
    for k in range(n):
        sx, bx = xo[min(k, len(xo) - 1)]
        sy, by = yo[min(k, len(yo) - 1)]
        g.tune(sx, sy, 0)
        g.tune_order(bx, by)
        g.init_case(case, seed)
        g.run(3)
        g.reset_counters()
        g.set_timing(True)
        g.run(4)
        t = g.kernel_times()
        g.set_timing(False)
        print(f"{cfg} {math} x(seg {sx}, band {bx}) {t['ms_x'] / t['n_x']:.4f} ms   "
              f"y(seg {sy}, band {by}) {t['ms_y'] / t['n_y']:.4f} ms", flush=True)
