#!/bin/bash
# A/B timing of prebuilt librfk_<v>.so variants on one box: scripts/ab.sh v1 v2 ...
mkdir -p gpurun_out
cp paper_2603_00035_b200/librfk.so /tmp/librfk_keep.so
for rep in 1 2; do
  for v in "$@"; do
    cp paper_2603_00035_b200/librfk_$v.so paper_2603_00035_b200/librfk.so
    echo "== $v" >> gpurun_out/ab.log
    timeout 60 python scripts/time_fwd.py ${AB_N:-4096} 3 >> gpurun_out/ab.log 2>&1
  done
done
cp /tmp/librfk_keep.so paper_2603_00035_b200/librfk.so
