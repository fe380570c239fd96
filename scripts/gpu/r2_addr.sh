# A/B: ring addresses one add from the step (ad1) and unconditional ring loads masked afterwards (ad2) vs HEAD (hd)
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh hd ad1 ad2
cp paper_2603_00035_b200/librfk_ad2.so paper_2603_00035_b200/librfk.so
timeout 1800 python -m pytest tests/test_fullsize_parity_gpu.py tests/test_gpu_parity.py tests/test_edge_cases_gpu.py -q -m gpu 2>&1 | tail -2 > gpurun_out/ad_parity.log
