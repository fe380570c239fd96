# A/B: the dirty vote consumed at the commit (vl1) vs gating the sqrt operands (vl0); parity with vl1
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh vl0 vl1
cp paper_2603_00035_b200/librfk_vl1.so paper_2603_00035_b200/librfk.so
timeout 1800 python -m pytest tests/test_fullsize_parity_gpu.py tests/test_gpu_parity.py tests/test_edge_cases_gpu.py tests/test_fp32_mode.py -q -m gpu 2>&1 | tail -3 > gpurun_out/vl_parity.log
