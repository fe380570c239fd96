#!/bin/bash
# A/B timing of prebuilt librfk_<v>.so variants with an optional CTA cap:
#   scripts/ab_env.sh v1[:ctas] v2[:ctas] ...   (AB_N grid size, AB_REPS rounds)
mkdir -p gpurun_out
cp paper_2603_00035_b200/librfk.so /tmp/librfk_keep.so
for rep in $(seq 1 ${AB_REPS:-2}); do
  for spec in "$@"; do
    v=${spec%%:*}; c=${spec#*:}; [ "$c" = "$spec" ] && c=""
    cp paper_2603_00035_b200/librfk_$v.so paper_2603_00035_b200/librfk.so
    echo "== $spec" >> gpurun_out/ab.log
    RFK_SWEEP_CTAS=$c timeout 60 python scripts/time_fwd.py ${AB_N:-4096} 3 >> gpurun_out/ab.log 2>&1
  done
done
cp /tmp/librfk_keep.so paper_2603_00035_b200/librfk.so
