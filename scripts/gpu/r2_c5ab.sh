# C5 A/B: product vs the gather pass (nofp) vs identify_kernel (noih)
mkdir -p gpurun_out
cp paper_2603_00035_b200/librfk.so /tmp/keep.so
for v in base2 nofp noih base2; do
  cp paper_2603_00035_b200/librfk_$v.so paper_2603_00035_b200/librfk.so
  echo "== $v" >> gpurun_out/c5ab.log
  timeout 600 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['samples_per_s'], d['ms_per_step'])" >> gpurun_out/c5ab.log
done
cp /tmp/keep.so paper_2603_00035_b200/librfk.so
