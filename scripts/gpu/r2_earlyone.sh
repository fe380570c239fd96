# A/B: one-point candidates and the NaN vote in the sqrt's shadow (eo1) vs after the two-point update (eo0)
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh eo0 eo1
cp paper_2603_00035_b200/librfk_eo1.so paper_2603_00035_b200/librfk.so
timeout 1800 python -m pytest tests/test_fullsize_parity_gpu.py tests/test_gpu_parity.py tests/test_edge_cases_gpu.py tests/test_fp32_mode.py -q -m gpu 2>&1 | tail -2 > gpurun_out/eo_parity.log
