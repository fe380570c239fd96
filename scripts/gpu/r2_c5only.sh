mkdir -p gpurun_out
for i in 1 2; do timeout 1200 python bench.py --workload c5 --steps 2 --warmup 3 2>/dev/null | tail -1 >> gpurun_out/bench_c5_rep.jsonl; done
