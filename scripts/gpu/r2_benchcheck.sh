mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_bench_gpu.py -q -m gpu 2>&1 | tail -3 > gpurun_out/benchcheck.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_quick.jsonl 2>&1
