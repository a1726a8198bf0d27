"""Tolerance of a non-bitwise build against the bitwise one (experiment tool).

    python tools/tol_check.py base.so other.so[:tolerance] [...] -- runs each
    library (optionally in a math mode) in its own process on the same cases,
    then prints compare_tolerance's max_rel
    (scale max(|a|,|b|,1), proj/src/audit.cpp:146) of every library's final
    interior against the first one's, plus event-timed sweep ms.
"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [("sod_x", 2048, 200, "transmit", 0), ("random", 2048, 100, "transmit", 2106),
         ("corner_blast", 1024, 300, "reflect", 0)]

if len(sys.argv) > 2 and sys.argv[1] == "--run":
    sys.path.insert(0, ROOT)
    import paper_2106_13465_b200 as P
    out, math = sys.argv[2], sys.argv[3]
    for case, n, steps, bc, seed in CASES:
        with P.GpuGrid(n, n, 1.0 / n, 1.0 / n, P.GasModel(), bc, device=0, math=math) as g:
            g.init_case(case, seed)
            g.run(3)
            g.set_timing(True)
            g.run(steps - 3)
            t = g.kernel_times()
            planes = np.zeros((4, n + 4, n + 4))
            g.download(planes)
        np.save(f"{out}_{case}.npy", planes[:, 2:n + 2, 2:n + 2])
        print(f"{case}: ms/sweep x {t['ms_x'] / t['n_x']:.4f} y {t['ms_y'] / t['n_y']:.4f}", flush=True)
    sys.exit(0)

libs = sys.argv[1:]
for k, spec in enumerate(libs):
    lib, _, math = spec.partition(":")
    env = dict(os.environ, HYDRO_B200_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, __file__, "--run", f"/tmp/tol_{k}", math or "bitwise"], env=env,
                       capture_output=True, text=True)
    print(os.path.basename(spec), r.stdout.strip().replace("\n", " | "), r.stderr[-300:] if r.returncode else "")
    if k:
        for case, *_ in CASES:
            a = np.load(f"/tmp/tol_0_{case}.npy")
            b = np.load(f"/tmp/tol_{k}_{case}.npy")
            rel = np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)
            print(f"   {case}: max_rel {rel.max():.3e}  differing cells {np.count_nonzero(rel)} / {rel.size}")
