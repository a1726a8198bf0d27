#!/bin/bash
# Measurement pass with the fused schedule as the default (run under gpurun from the repo root):
# GPU tests, the default bench line, fused-vs-split check, ncu captures of the fused step kernel.
O=gpurun_out/r2h
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $O/pytest_gpu.log
python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
timeout 900 python tools/fused_check.py --quick --time cfg3 cfg2 cfg4 cfg1 > $O/fused_check.log 2>&1; echo "fused_check rc=$?"
for m in tolerance bitwise; do
  ncu --set full --import-source on --clock-control none -k regex:sweep_xy --launch-skip 2 --launch-count 1 \
      -o $O/cfg3_fused_$m python tools/profile_step.py --nx 16384 --case corner_blast --bc reflect --pre 4 --steps 3 --math $m --schedule fused > $O/ncu_cfg3_$m.log 2>&1
  ncu --set full --import-source on --clock-control none -k regex:sweep_xy --launch-skip 2 --launch-count 1 \
      -o $O/cfg2_fused_$m python tools/profile_step.py --nx 8192 --case random --seed 2106 --bc transmit --pre 4 --steps 3 --math $m --schedule fused > $O/ncu_cfg2_$m.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-variants --no-cpu-baseline > $O/launches_bench.log 2>&1
echo done
