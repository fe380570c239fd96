mkdir -p gpurun_out
timeout 900 python scripts/time_iters.py 4096 > gpurun_out/forward_vs_iterations.log 2>&1
