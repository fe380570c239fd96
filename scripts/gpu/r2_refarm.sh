# the reference arm at the driver's K/W, timed
mkdir -p gpurun_out
s=$(date +%s.%N)
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.jsonl 2> gpurun_out/bench_ref.err
echo "rc=$? wall_s=$(echo "$(date +%s.%N) - $s" | bc)" >> gpurun_out/bench_ref.err
nproc >> gpurun_out/bench_ref.err
