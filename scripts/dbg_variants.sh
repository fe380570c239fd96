#!/bin/bash
# run scripts/dbg_hist.py against each prebuilt librfk_<v>.so variant
mkdir -p gpurun_out
cp paper_2603_00035_b200/librfk.so /tmp/librfk_main.so
for v in "$@"; do
  cp paper_2603_00035_b200/librfk_$v.so paper_2603_00035_b200/librfk.so
  echo "== $v" >> gpurun_out/variants.log
  timeout 200 python scripts/dbg_hist.py 2>&1 | grep bad >> gpurun_out/variants.log
done
cp /tmp/librfk_main.so paper_2603_00035_b200/librfk.so
