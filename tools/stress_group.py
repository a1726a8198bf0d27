"""Repeats the single-process group parity check (tests/test_gpu_parity.py::
test_single_process_group_equals_one_domain) many times to surface rare
ordering bugs (tools only).   python tools/stress_group.py [reps]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_13465_b200 as P  # noqa: E402

MODEL = P.GasModel()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
cases = [(2, "sod_x", "transmit", "hllc"), (3, "random", "transmit", "hllc"),
         (5, "corner_blast", "reflect", "hllc"), (3, "random", "reflect", "exact10"),
         (8, "random", "transmit", "hllc")]
nx, ny, steps = 77, 52, 30
bad = 0
for n, case, bc, flux in cases:
    one = P.make_case(case, nx, ny, MODEL, seed=9)
    dt_one = P.run_gpu(one, MODEL, steps, bc, flux=flux)
    fails = 0
    for r in range(reps):
        grp = P.make_case(case, nx, ny, MODEL, seed=9)
        with P.GpuGroup(nx, ny, grp.dx, grp.dy, MODEL, bc, devices=[0] * n, flux=flux) as g:
            g.upload(grp.planes)
            dt_grp = g.run(steps)
            g.download(grp.planes)
        ok = dt_grp == dt_one and np.array_equal(grp.planes, one.planes)
        if not ok:
            fails += 1
            d = np.argwhere(grp.planes != one.planes)
            print(f"  rep {r}: dt {dt_grp == dt_one}, {len(d)} cells differ, first {d[:4].tolist()}",
                  flush=True)
    bad += fails
    print(f"{n} {case} {bc} {flux}: {fails}/{reps} mismatches", flush=True)
sys.exit(1 if bad else 0)
