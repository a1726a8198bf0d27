#!/bin/bash
# Final measurement pass of round 2 (run under gpurun from the repo root), in parts so that
# each call's gpurun_out stays under the 64 MiB that is copied back:
#   tools/r2k_final.sh bench   GPU tests, the default bench line + the reference arm, config 4, launch list
#   tools/r2k_final.sh ncu3    ncu --set full of the fused step on config 3 (both arithmetics)
#   tools/r2k_final.sh ncu2    ncu --set full of the split sweeps on config 2 (both arithmetics)
O=gpurun_out/r2k
mkdir -p $O
case "$1" in
bench)
  nvidia-smi > $O/nvidia_smi.txt 2>&1
  timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
  python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
  python bench.py --impl reference --steps 5 --warmup 1 > $O/reference_cfg3.json 2> $O/reference_cfg3.err; echo "reference rc=$?"
  python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "cfg4 rc=$?"
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv \
      python bench.py --steps 1 --warmup 1 --no-variants --no-cpu-baseline > $O/launches_bench.log 2>&1
  ;;
ncu3)
  for m in tolerance bitwise; do
    ncu --set full --import-source on --clock-control none -k regex:sweep_xy --launch-skip 6 --launch-count 1 \
        -o $O/cfg3_fused_$m python tools/profile_step.py --nx 16384 --case corner_blast --bc reflect --pre 4 --steps 4 --math $m --schedule fused > $O/ncu_cfg3_$m.log 2>&1
  done
  ;;
ncu2)
  for m in tolerance bitwise; do
    ncu --set full --import-source on --clock-control none -k regex:sweep --launch-skip 6 --launch-count 2 \
        -o $O/cfg2_split_$m python tools/profile_step.py --nx 8192 --case random --seed 2106 --bc transmit --pre 3 --steps 1 --math $m --schedule split > $O/ncu_cfg2_$m.log 2>&1
  done
  ;;
esac
ls -la $O; echo done
