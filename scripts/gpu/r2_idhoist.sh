# A/B: identify from hoisted records (ih1) vs the per-lane E/det/Q evaluation (ih0); backward parity with ih1
mkdir -p gpurun_out
for v in ih0 ih1 ih0 ih1; do
  cp paper_2603_00035_b200/librfk_$v.so paper_2603_00035_b200/librfk.so
  echo "== $v" >> gpurun_out/bwab.log
  timeout 200 python scripts/time_backward.py 4096 2>&1 | head -4 >> gpurun_out/bwab.log
done
cp paper_2603_00035_b200/librfk_ih1.so paper_2603_00035_b200/librfk.so
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity_gpu.py tests/test_edge_cases_gpu.py tests/test_fused_projection_gpu.py tests/test_fp32_mode.py tests/test_objective.py tests/test_inverse.py tests/test_torch_ops.py tests/test_reference_unit_suites.py tests/test_gradcheck.py -q -m gpu 2>&1 | tail -4 > gpurun_out/ih_tests.log
