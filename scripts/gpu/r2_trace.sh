# per-band trace of the current build (instrumented instantiation), 4096^2
mkdir -p gpurun_out
RFK_TRACE=1 timeout 600 python scripts/trace_sweep.py 4096 all > gpurun_out/trace.log 2>&1
