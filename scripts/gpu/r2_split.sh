# A/B: adjoint order (keys/sort/rank) beside identify (bw1) vs serial (bw0); then backward parity with bw1
mkdir -p gpurun_out
for v in bw0 bw1 bw0 bw1; do
  cp paper_2603_00035_b200/librfk_$v.so paper_2603_00035_b200/librfk.so
  echo "== $v" >> gpurun_out/bwab.log
  timeout 200 python scripts/time_backward.py 4096 2>&1 | head -4 >> gpurun_out/bwab.log
done
cp paper_2603_00035_b200/librfk_bw1.so paper_2603_00035_b200/librfk.so
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity_gpu.py tests/test_edge_cases_gpu.py tests/test_fused_projection_gpu.py tests/test_fp32_mode.py tests/test_objective.py tests/test_inverse.py tests/test_torch_ops.py tests/test_multirank_gpu.py -q -m gpu 2>&1 | tail -5 > gpurun_out/split_tests.log
