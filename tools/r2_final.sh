#!/bin/bash
# Final measurement pass of round 2 (run under gpurun from the repo root):
# bench lines, the reference arm, ncu captures, the launch list.
O=gpurun_out/r2f
mkdir -p $O
tools/_fp64_peak > $O/fp64_peak.json 2>&1
python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "cfg4 rc=$?"
python bench.py --workload cfg2 --flux exact10 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg2_exact10.json 2> $O/bench_cfg2_exact10.err; echo "cfg2x rc=$?"
python bench.py --impl reference --steps 10 --warmup 3 > $O/reference_cfg3.json 2> $O/reference_cfg3.err; echo "ref rc=$?"
for m in tolerance bitwise; do
  ncu --set full --import-source on --clock-control none -k regex:sweep --launch-skip 6 --launch-count 2 \
      -o $O/cfg3_$m python tools/profile_step.py --nx 16384 --case corner_blast --bc reflect --pre 3 --steps 1 --math $m > $O/ncu_cfg3_$m.log 2>&1
  ncu --set full --import-source on --clock-control none -k regex:sweep --launch-skip 6 --launch-count 2 \
      -o $O/cfg2_$m python tools/profile_step.py --nx 8192 --case random --seed 2106 --bc transmit --pre 3 --steps 1 --math $m > $O/ncu_cfg2_$m.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-variants --no-cpu-baseline > $O/launches_bench.log 2>&1
echo done
