# the adaptive dependents search (fused for >= 2048^2 grids): C5 and the 4096^2 backward vs the always-fused build; parity
mkdir -p gpurun_out
cp paper_2603_00035_b200/librfk.so /tmp/keep.so
for v in base2 adapt; do
  cp paper_2603_00035_b200/librfk_$v.so paper_2603_00035_b200/librfk.so
  echo "== $v" >> gpurun_out/adapt.log
  timeout 600 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', d['config']['samples_per_s'])" >> gpurun_out/adapt.log
  timeout 200 python scripts/time_backward.py 4096 2>&1 | head -4 | tail -1 >> gpurun_out/adapt.log
  timeout 200 python scripts/time_backward.py 1024 2>&1 | head -4 | tail -1 >> gpurun_out/adapt.log
done
cp paper_2603_00035_b200/librfk_adapt.so paper_2603_00035_b200/librfk.so
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity_gpu.py tests/test_edge_cases_gpu.py tests/test_fused_projection_gpu.py tests/test_fp32_mode.py tests/test_objective.py tests/test_inverse.py tests/test_torch_ops.py tests/test_training.py -q -m gpu 2>&1 | tail -3 > gpurun_out/adapt_tests.log
