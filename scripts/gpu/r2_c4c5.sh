# C4 / C5 informational lines on the final build
mkdir -p gpurun_out
timeout 1200 python bench.py --workload c4 --scenes 16 --steps 2 --warmup 3 > gpurun_out/bench_c4.jsonl 2> gpurun_out/bench_c4.err
timeout 1200 python bench.py --workload c5 --steps 2 --warmup 3 > gpurun_out/bench_c5.jsonl 2> gpurun_out/bench_c5.err
