# per-pass timeline of a 4096^2 solve (trace build)
mkdir -p gpurun_out
RFK_LIBRARY=$PWD/paper_2603_00035_b200/librfk_trace.so RFK_TRACE=1 timeout 600 python scripts/trace_sweep.py 4096 > gpurun_out/timeline.log 2>&1
