"""Short config-1 run for ncu captures (not a benchmark: numbers printed under
ncu are never bench values).

    python tools/profile_step.py [--nx 2048] [--steps 4] [--case sod_x] [--bc transmit]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2106_13465_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nx", type=int, default=2048)
ap.add_argument("--ny", type=int, default=0)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--case", default="sod_x")
ap.add_argument("--bc", default="transmit")
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--seg", type=int, nargs=3, default=[0, 0, 0])
ap.add_argument("--pre", type=int, default=2, help="untimed steps before the timed ones")
ap.add_argument("--flux", default="hllc")
ap.add_argument("--math", default="bitwise")
ap.add_argument("--schedule", default="split")
ap.add_argument("--fseg", type=int, default=0, help="rows per fused work item (0 = automatic)")
a = ap.parse_args()
ny = a.ny or a.nx
with P.GpuGrid(a.nx, ny, 1.0 / a.nx, 1.0 / ny, P.GasModel(), a.bc, device=0, flux=a.flux,
               math=a.math) as g:
    g.tune(*a.seg)
    g.set_schedule(a.schedule, a.fseg)
    g.init_case(a.case, a.seed)
    g.run(a.pre)  # warm-up / advance the flow: init, prologue, sweeps, finish
    g.set_timing(True)
    g.run(a.steps)
    t = g.kernel_times()
    fm, fn = g.fused_times()
print({k: round(v, 4) if isinstance(v, float) else v for k, v in t.items()})
if fn:
    print("ms per fused step %.4f (%d launches)" % (fm / fn, fn))
print("ms per sweep_x %.4f  sweep_y %.4f" % (t["ms_x"] / max(1, t["n_x"]), t["ms_y"] / max(1, t["n_y"])))
