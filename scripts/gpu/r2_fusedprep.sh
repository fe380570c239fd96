# A/B: the dataflow adjoint finds its dependents itself (fp1) vs the gather pass (fp0); backward parity with fp1
mkdir -p gpurun_out
for v in fp0 fp1 fp0 fp1; do
  cp paper_2603_00035_b200/librfk_$v.so paper_2603_00035_b200/librfk.so
  echo "== $v" >> gpurun_out/bwab.log
  timeout 200 python scripts/time_backward.py 4096 2>&1 | head -4 >> gpurun_out/bwab.log
done
cp paper_2603_00035_b200/librfk_fp1.so paper_2603_00035_b200/librfk.so
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity_gpu.py tests/test_edge_cases_gpu.py tests/test_fused_projection_gpu.py tests/test_fp32_mode.py tests/test_objective.py tests/test_inverse.py tests/test_torch_ops.py tests/test_reference_unit_suites.py -q -m gpu 2>&1 | tail -4 > gpurun_out/fp_tests.log
