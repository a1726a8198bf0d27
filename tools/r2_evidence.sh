#!/bin/bash
# Evidence pass of round 2 (run under gpurun from the repo root): FP64 peak,
# ncu captures of the sweeps on configs 3 and 2, the launch list of the bench
# command, compute-sanitizer on small grids.
set -x
O=gpurun_out
tools/_fp64_peak > $O/r2_fp64_peak.json 2>&1
for m in tolerance bitwise; do
  ncu --set full --import-source on --clock-control none -k regex:sweep --launch-skip 6 --launch-count 2 \
      -o $O/r2_cfg3_$m python tools/profile_step.py --nx 16384 --case corner_blast --bc reflect --pre 3 --steps 1 --math $m > $O/r2_ncu_cfg3_$m.log 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:sweep --launch-skip 6 --launch-count 2 \
    -o $O/r2_cfg2_tolerance python tools/profile_step.py --nx 8192 --case random --seed 2106 --bc transmit --pre 3 --steps 1 --math tolerance > $O/r2_ncu_cfg2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/r2_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-variants --no-cpu-baseline > $O/r2_launches_bench.log 2>&1
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/profile_step.py --nx 96 --ny 160 --case random --bc transmit --pre 1 --steps 2 > $O/r2_san_${t}_bitwise.log 2>&1
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/profile_step.py --nx 96 --ny 160 --case random --bc transmit --pre 1 --steps 2 --math tolerance > $O/r2_san_${t}_tol.log 2>&1
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/profile_step.py --nx 64 --case sod_x --bc transmit --pre 1 --steps 2 --flux exact10 > $O/r2_san_${t}_exact10.log 2>&1
done
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "loopback or single_process_group_equals" > $O/r2_san_memcheck_loopback.log 2>&1
echo done
