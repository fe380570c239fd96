# objective_and_grad reusing the solve's hoisted records: objective tests + inverse + e2e bench
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_objective.py tests/test_inverse.py tests/test_bench_gpu.py tests/test_fullsize_parity_gpu.py -q -m gpu 2>&1 | tail -3 > gpurun_out/objreuse_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_objreuse.jsonl 2>&1
