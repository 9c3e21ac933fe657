#!/usr/bin/env bash
# Build an experiment variant of libtt_b200.so with extra nvcc flags (A/B measurements):
#   scripts/build_variant.sh TAG -DTT_PIPE_BLOCK=256 ...  ->  paper_2603_00538_b200/libtt_b200_TAG.so
# (load it with TT_LIB_PATH=...; the product build is paper_2603_00538_b200/_build.py)
set -euo pipefail
cd "$(dirname "$0")/.."
TAG=$1; shift
OUT=build/variant_$TAG
mkdir -p $OUT
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude"
for f in paper_2603_00538_b200/csrc/*.cu; do
  nvcc $FLAGS "$@" -c $f -o $OUT/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2603_00538_b200/libtt_b200_$TAG.so $OUT/*.o
echo paper_2603_00538_b200/libtt_b200_$TAG.so
