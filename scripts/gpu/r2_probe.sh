cp paper_2603_00035_b200/librfk_prb.so /tmp/prb.so
RFK_LIBRARY=/tmp/prb.so RFK_TRACE=1 timeout 300 python scripts/trace_sweep.py ${TR_N:-4096} > gpurun_out/trace_probe.log 2>&1
