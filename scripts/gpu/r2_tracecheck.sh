# product build without the traced kernel: parity subset; trace build: per-band trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_bench_gpu.py -q -m gpu -x 2>&1 | tail -3 > gpurun_out/tracecheck_tests.log
bash scripts/gpu/r2_trace.sh
RFK_TRACE=1 timeout 300 python scripts/trace_sweep.py 256 > gpurun_out/trace_product.log 2>&1; echo "rc=$?" >> gpurun_out/trace_product.log
