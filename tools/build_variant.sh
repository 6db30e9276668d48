#!/bin/bash
# Build a variant of libsparsedrop_b200.so for in-process A/B (dev tool).
#   tools/build_variant.sh NAME REF [NVCC_DEFINES...]
# REF = a git ref (the sources as committed there) or "work" (the working tree).
# Output: paper_2411_01238_b200/lib/var_NAME.so (git-ignored; travels with gpurun).
set -e
NAME=$1; REF=$2; shift 2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
T=/tmp/sdvar_$NAME
rm -rf "$T"; mkdir -p "$T"
if [ "$REF" = work ]; then
  mkdir -p "$T/paper_2411_01238_b200"
  cp -r "$ROOT/paper_2411_01238_b200/csrc" "$T/paper_2411_01238_b200/"
  cp -r "$ROOT/include" "$T/"
else
  git -C "$ROOT" archive "$REF" paper_2411_01238_b200/csrc include | tar -x -C "$T"
fi
make -s -C "$T/paper_2411_01238_b200/csrc" -j8 NVCC="/usr/local/cuda/bin/nvcc $*" > "$T/build.log" 2>&1 || { tail -30 "$T/build.log"; exit 1; }
cp "$T/paper_2411_01238_b200/lib/libsparsedrop_b200.so" "$ROOT/paper_2411_01238_b200/lib/var_$NAME.so"
echo "built paper_2411_01238_b200/lib/var_$NAME.so ($REF $*)"
