# round-2 measurement: bench line, reference arm, ncu launch list + full sweep capture, C3 CPU reference
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.jsonl 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o gpurun_out/sweep_full python scripts/prof_solve.py 4096 > gpurun_out/ncu_full.log 2>&1
[ -n "$C3REF" ] && timeout 1500 python scripts/cpu_c3_reference.py 4096 gpurun_out/r02_cpu_c3_reference.json > gpurun_out/c3ref.log 2>&1
ls -la gpurun_out
