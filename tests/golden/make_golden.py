"""Generates the committed golden vectors from the UNMODIFIED reference.

Run in the build container (needs /root/reference compiled into
oracle/_ref/libhydro_ref.so by ``make -C oracle``):

    python tests/golden/make_golden.py            # golden.json (seconds)
    python tests/golden/make_golden.py --full     # golden_full.json (minutes)
    python tests/golden/make_golden.py --full --only cfg1_sod_x_2048_200_exact10  # ~15 min
    python tests/golden/make_golden.py --full --only cfg2_random_8192_50_exact10 \
        --out /tmp/cfg2.json     # ~1.5 h single-threaded; --out lets runs go in parallel

Every digest here is produced by the reference's own run_sequential /
run_coarse_grain (bitwise equal to each other, acceptance_tests.cpp:48-113)
through oracle/ref_shim.cpp; the only addition is the transmissive boundary
(link-time --wrap of apply_boundary) that BASELINE configs 1, 2 and 4 need.
The initial grids come from the C restatement's initialisers, which
tests/test_oracle.py pins against the reference's make_case.

BASELINE.json names no public dataset: configs 2 and 4 use the seeded
counter-based random field (splitmix64, seeds 2106 and 13465), the rest are
analytic initial conditions.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402

SEED_CFG2 = 2106
SEED_CFG4 = 13465

# (name, case, nx, ny, bc, steps, seed, provenance)
SMALL = [
    ("readme_48_blast_5", "blast", 48, 48, "reflect", 5, 0, "proj/README.md:98-101 (published)"),
    ("readme_64_blast_5", "blast", 64, 64, "reflect", 5, 0, "proj/README.md:104-109 (published)"),
    ("accept_64_blast_10", "blast", 64, 64, "reflect", 10, 0, "acceptance_tests.cpp:111-112"),
    ("accept_128x96_blast_10", "blast", 128, 96, "reflect", 10, 0, "acceptance_tests.cpp:111-112"),
    ("survey_256_blast_10", "blast", 256, 256, "reflect", 10, 0, "SURVEY.md Appendix B"),
    ("survey_256_blast_100", "blast", 256, 256, "reflect", 100, 0, "SURVEY.md Appendix B"),
    ("cfg0_corner_blast_256_100", "corner_blast", 256, 256, "reflect", 100, 0,
     "BASELINE config 0 at full size (HLLC flux)"),
    ("cfg1_sod_x_256_100", "sod_x", 256, 256, "transmit", 100, 0, "BASELINE config 1, reduced size"),
    ("cfg2_random_128_50", "random", 128, 128, "transmit", 50, SEED_CFG2, "BASELINE config 2, reduced"),
    ("cfg3_corner_blast_384_60", "corner_blast", 384, 384, "reflect", 60, 0,
     "BASELINE config 3, reduced"),
    ("cfg4_random_256x128_20", "random", 256, 128, "transmit", 20, SEED_CFG4,
     "BASELINE config 4 (P=2 shape), reduced"),
    ("odd_blast_37x53_23", "blast", 37, 53, "reflect", 23, 0, "ragged extents"),
    ("odd_sod_x_33x17_40", "sod_x", 33, 17, "transmit", 40, 0, "ragged extents"),
    ("tiny_blast_4x4_7", "blast", 4, 4, "reflect", 7, 0, "minimum grid (grid.cpp:11-14)"),
    ("tiny_random_5x4_9", "random", 5, 4, "transmit", 9, 11, "minimum grid, transmissive"),
    ("sod_j_4x64_30", "sod", 4, 64, "reflect", 30, 0, "reference Sod tube (cases.cpp:54-69)"),
    ("uniform_16x24_5", "uniform", 16, 24, "reflect", 5, 0, "fixed point"),
    ("random_reflect_96x80_25", "random", 96, 80, "reflect", 25, 5, "random field, reflective"),
    ("corner_transmit_128x64_40", "corner_blast", 128, 64, "transmit", 40, 0, "blast, transmissive"),
]

# Full BASELINE sizes (configs 1-4; config 0 is already full size above).
FULL = [
    ("cfg1_sod_x_2048_200", "sod_x", 2048, 2048, "transmit", 200, 0, "BASELINE config 1, full"),
    ("cfg2_random_8192_50", "random", 8192, 8192, "transmit", 50, SEED_CFG2, "BASELINE config 2, full"),
    ("cfg4_random_16384_20", "random", 16384, 16384, "transmit", 20, SEED_CFG4,
     "BASELINE config 4 at P=1, full"),
    ("cfg3_corner_blast_16384_50", "corner_blast", 16384, 16384, "reflect", 50, 0,
     "BASELINE config 3, full"),
]


# The exact-10 flux is not on the reference's hot path: its full-size digest
# comes from the oracle's C restatement (oracle/hydro_oracle.c, exact10),
# which tests/test_exact_flux.py pins within 1e-12 of the reference's own
# exact solver (proj/src/exact_riemann.cpp).
FULL_EXACT10 = [
    ("cfg0_corner_blast_256_100_exact10", "corner_blast", 256, 256, "reflect", 100, 0,
     "BASELINE config 0 with its stated exact Riemann solver (10 Newton iterations), full"),
    ("cfg1_sod_x_2048_200_exact10", "sod_x", 2048, 2048, "transmit", 200, 0,
     "BASELINE config 1 with its stated exact Riemann solver (10 Newton iterations), full"),
    ("cfg2_random_8192_50_exact10", "random", 8192, 8192, "transmit", 50, SEED_CFG2,
     "BASELINE config 2 with its stated exact Riemann solver (10 Newton iterations), full"),
    ("cfg3_corner_blast_16384_50_exact10", "corner_blast", 16384, 16384, "reflect", 50, 0,
     "BASELINE config 3 at P=1 with its stated exact Riemann solver, full"),
    ("cfg4_random_16384_20_exact10", "random", 16384, 16384, "transmit", 20, SEED_CFG4,
     "BASELINE config 4 at P=1 with its stated exact Riemann solver, full"),
    ("random_1024_20_exact10", "random", 1024, 1024, "transmit", 20, 7,
     "dense random states, exact-10: Newton cycle exits at scale"),
]


THREADS = 1


def run_oracle_exact10(entry):
    name, case, nx, ny, bc, steps, seed, prov = entry
    g = O.make_case(case, nx, ny, seed=seed)
    t0 = time.time()
    O.set_threads(THREADS)
    with O.flux_mode("exact10"):
        O.run_sequential(g, steps, bc)
    O.set_threads(1)
    secs = time.time() - t0
    rec = {"case": case, "nx": g.nx, "ny": g.ny, "bc": bc, "steps": steps, "seed": seed,
           "flux": "exact10", "digest": f"{O.digest(g):016x}", "provenance": prov,
           "generator": "oracle (C restatement, oracle_set_flux exact10), "
                        + ("single thread" if THREADS == 1 else
                           f"strip-parallel x{THREADS} (oracle_set_threads; equal to one thread)"),
           "ref_seconds": round(secs, 1)}
    print(f"{name}: {rec['digest']} ({secs:.1f}s)", flush=True)
    return name, rec


def run_case(entry, strategy, workers):
    name, case, nx, ny, bc, steps, seed, prov = entry
    g = O.make_case(case, nx, ny, seed=seed)
    t0 = time.time()
    secs = O.ref_run(g, steps, bc=bc, strategy=strategy, workers=workers)
    rec = {"case": case, "nx": g.nx, "ny": g.ny, "bc": bc, "steps": steps, "seed": seed,
           "digest": f"{O.ref_digest(g):016x}", "checksum_line": O.ref_checksum_line(g),
           "provenance": prov, "generator": f"reference {strategy} x{workers}",
           "ref_seconds": round(secs, 3)}
    print(f"{name}: {rec['digest']} ({time.time() - t0:.1f}s)", flush=True)
    return name, rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--only", default=None)
    ap.add_argument("--out", default=None, help="write to this file instead (parallel runs)")
    ap.add_argument("--threads", type=int, default=1,
                    help="strip-parallel oracle sweeps for the exact-10 entries")
    args = ap.parse_args()
    global THREADS
    THREADS = args.threads
    if not O.ref_available():
        sys.exit("oracle/_ref/libhydro_ref.so missing: make -C oracle")
    out_path = args.out or os.path.join(HERE, "golden_full.json" if args.full else "golden.json")
    table = FULL if args.full else SMALL
    result = {}
    if os.path.exists(out_path):
        result = json.load(open(out_path))
    workers = max(1, os.cpu_count() or 1)
    for entry in table:
        if args.only and entry[0] != args.only:
            continue
        if args.full:
            name, rec = run_case(entry, "coarse_grain", workers)
        else:
            name, rec = run_case(entry, "sequential", 1)
        result[name] = rec
        json.dump(result, open(out_path, "w"), indent=1, sort_keys=True)
    if args.full:
        for entry in FULL_EXACT10:
            if args.only and entry[0] != args.only:
                continue
            name, rec = run_oracle_exact10(entry)
            result[name] = rec
            json.dump(result, open(out_path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
