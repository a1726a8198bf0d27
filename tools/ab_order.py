"""A/B of the sweeps' claim order (hydro_gpu_tune_order) and segment length
on BASELINE grids: event-timed sweeps after a few untimed steps.  Not a
benchmark (tools only).

    python tools/ab_order.py --cfg cfg3 --bands 0,-1,4,16,64 [--segs 0,64]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_13465_b200 as P  # noqa: E402
from bench import WORKLOADS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg3")
ap.add_argument("--bands", default="0,1000000")
ap.add_argument("--segs", default="0")
ap.add_argument("--math", default="bitwise")
ap.add_argument("--flux", default="hllc")
ap.add_argument("--pre", type=int, default=3)
ap.add_argument("--steps", type=int, default=4)
a = ap.parse_args()
case, nx, ny, bc, ts, seed, _ = WORKLOADS[a.cfg]
with P.GpuGrid(nx, ny, 1.0 / nx, 1.0 / ny, P.GasModel(), bc, device=0, flux=a.flux, math=a.math) as g:
    for seg in [int(x) for x in a.segs.split(",")]:
        for band in [int(x) for x in a.bands.split(",")]:
            g.tune(seg, seg, 0)
            g.tune_order(band, band)
            g.init_case(case, seed)
            g.run(a.pre)
            g.reset_counters()
            g.set_timing(True)
            g.run(a.steps)
            t = g.kernel_times()
            g.set_timing(False)
            print(f"{a.cfg} {a.math} seg={seg} band={band}: x {t['ms_x'] / t['n_x']:.4f} ms  "
                  f"y {t['ms_y'] / t['n_y']:.4f} ms", flush=True)
