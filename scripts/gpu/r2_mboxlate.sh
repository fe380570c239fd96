# A/B: the last line's mailbox store before (ml0, product) or after (ml1) the step barrier
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh ml0 ml1
cp paper_2603_00035_b200/librfk_ml1.so paper_2603_00035_b200/librfk.so
timeout 1800 python -m pytest tests/test_fullsize_parity_gpu.py tests/test_gpu_parity.py tests/test_edge_cases_gpu.py -q -m gpu 2>&1 | tail -2 > gpurun_out/ml_parity.log
