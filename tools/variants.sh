#!/bin/bash
# Builds compile-time variants of libhydro_b200.so into build_variants/<name>.so
#   tools/variants.sh name "EXTRA nvcc flags" [name "flags" ...]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$ROOT/build_variants"
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  make -s -C "$ROOT/paper_2106_13465_b200/csrc" OUT="$ROOT/build_variants/$name.so" \
       OBJ="$ROOT/build_variants/obj_$name" EXTRA="$flags" >/dev/null
  regs=$(make -s -C "$ROOT/paper_2106_13465_b200/csrc" ptxas EXTRA="$flags" 2>&1 | grep -E "Used [0-9]+ registers" | tail -2 | sed -E 's/.*Used ([0-9]+) registers.*/\1/' | tr '\n' '/')
  spill=$(make -s -C "$ROOT/paper_2106_13465_b200/csrc" ptxas EXTRA="$flags" 2>&1 | grep -E "spill" | tail -2 | sed -E 's/.*, ([0-9]+) bytes spill stores.*/\1/' | tr '\n' '/')
  echo "$name: regs(y/x)=$regs spills=$spill"
done
