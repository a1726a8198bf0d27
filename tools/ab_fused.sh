#!/bin/bash
# A/B of fused-step builds (run under gpurun): tools/ab_fused.sh <out> <lib>...   (lib "tree" = in-tree)
O=$1; shift
mkdir -p $(dirname $O)
for lib in "$@"; do
  if [ "$lib" = tree ]; then unset HYDRO_B200_LIB; else export HYDRO_B200_LIB=$PWD/build_variants/$lib.so; fi
  echo "== $lib" >> $O
  timeout 600 python tools/fused_check.py --quick --time 2>&1 | grep -E "MISMATCH|mismatches" >> $O
  for m in tolerance bitwise; do
    echo "cfg3 $m: $(python tools/profile_step.py --nx 16384 --case corner_blast --bc reflect --pre 4 --steps 5 --math $m --schedule fused 2>&1 | grep fused)" >> $O
  done
  for m in tolerance bitwise; do
    echo "cfg2 $m: $(python tools/profile_step.py --nx 8192 --case random --seed 2106 --bc transmit --pre 4 --steps 5 --math $m --schedule fused 2>&1 | grep fused)" >> $O
  done
  echo "cfg1 tolerance: $(python tools/profile_step.py --nx 2048 --case sod_x --bc transmit --pre 50 --steps 21 --math tolerance --schedule fused 2>&1 | grep fused)" >> $O
done
cat $O
