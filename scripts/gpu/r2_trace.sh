# per-band traces of sweep variants (RFK_TRACE diagnostics)
for v in ${TR_VARIANTS:-s0 s1}; do
  cp paper_2603_00035_b200/librfk_$v.so paper_2603_00035_b200/librfk.so
  RFK_TRACE=1 timeout 300 python scripts/trace_sweep.py ${TR_N:-4096} all > gpurun_out/trace_$v.log 2>&1
done
