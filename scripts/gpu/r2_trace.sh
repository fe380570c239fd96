# per-band trace of the current build (instrumented instantiation, librfk_trace.so built by
# scripts/build_variant.sh trace -DRFK_SWEEP_TRACE_BUILD=1), 4096^2
mkdir -p gpurun_out
RFK_LIBRARY=$PWD/paper_2603_00035_b200/librfk_trace.so RFK_TRACE=1 timeout 600 python scripts/trace_sweep.py 4096 all > gpurun_out/trace.log 2>&1
