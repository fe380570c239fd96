#!/bin/bash
# Build librfk_<name>.so with extra nvcc flags for the sweep TU only (A/B):
#   scripts/build_variant.sh name -DRFK_SWEEP_SKIP=0 ...
# The other translation units are compiled once into build/ab/ and reused.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
CS=paper_2603_00035_b200/csrc
OUT=build/ab
mkdir -p $OUT
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden"
pids=()
for f in rfk_solve rfk_sweep_f32 rfk_backward rfk_project rfk_inverse rfk_capi rfk_capi_inverse; do
  if [ ! -f $OUT/$f.o ] || [ $CS/$f.cu -nt $OUT/$f.o ] || [ $CS/rfk_internal.h -nt $OUT/$f.o ]; then
    nvcc $FL -c $CS/$f.cu -o $OUT/$f.o & pids+=($!)
  fi
done
nvcc $FL "$@" -c $CS/rfk_sweep.cu -o $OUT/rfk_sweep_$name.o
for p in "${pids[@]}"; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2603_00035_b200/librfk_$name.so $OUT/rfk_sweep_$name.o \
  $OUT/rfk_solve.o $OUT/rfk_sweep_f32.o $OUT/rfk_backward.o $OUT/rfk_project.o $OUT/rfk_inverse.o $OUT/rfk_capi.o $OUT/rfk_capi_inverse.o
echo built paper_2603_00035_b200/librfk_$name.so
