# A/B of the backward (dataflow adjoint poll) variants
for v in dfo dfb dfo dfb; do
  cp paper_2603_00035_b200/librfk_$v.so paper_2603_00035_b200/librfk.so
  echo "== $v" >> gpurun_out/bwab.log
  timeout 200 python scripts/time_backward.py 4096 2>&1 | head -5 >> gpurun_out/bwab.log
done
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity_gpu.py -q -x 2>&1 | tail -1 >> gpurun_out/bwab.log
