#!/bin/bash
# Builds the library of a git revision into build_variants/<name>.so for A/B timing
#   tools/ab_build.sh <rev> <name> ["EXTRA flags"]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rev=$1; name=$2; flags=${3:-}
wt=/tmp/ab_$name
rm -rf "$wt"; git -C "$ROOT" worktree prune
git -C "$ROOT" worktree add -f "$wt" "$rev" >/dev/null 2>&1
mkdir -p "$ROOT/build_variants"
make -s -C "$wt/paper_2106_13465_b200/csrc" OUT="$ROOT/build_variants/$name.so" OBJ="$wt/objab" EXTRA="$flags" >/dev/null 2>&1
git -C "$ROOT" worktree remove --force "$wt"
echo "built $name from $rev"
