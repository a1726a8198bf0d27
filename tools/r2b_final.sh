#!/bin/bash
# Measurement pass after the tiled-state kernels (run under gpurun from the repo root):
# GPU tests, bench lines, ncu captures of both sweeps (configs 3 and 2), the launch list.
O=gpurun_out/r2g
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "cfg4 rc=$?"
for m in tolerance bitwise; do
  ncu --set full --import-source on --clock-control none -k regex:sweep --launch-skip 6 --launch-count 2 \
      -o $O/cfg3_$m python tools/profile_step.py --nx 16384 --case corner_blast --bc reflect --pre 3 --steps 1 --math $m > $O/ncu_cfg3_$m.log 2>&1
  ncu --set full --import-source on --clock-control none -k regex:sweep --launch-skip 6 --launch-count 2 \
      -o $O/cfg2_$m python tools/profile_step.py --nx 8192 --case random --seed 2106 --bc transmit --pre 3 --steps 1 --math $m > $O/ncu_cfg2_$m.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-variants --no-cpu-baseline > $O/launches_bench.log 2>&1
echo done
