# A/B: next step's dirt read from ring stamps during the current step (ed1) vs vote-only entry (ed0)
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh ed0 ed1
cp paper_2603_00035_b200/librfk_ed1.so paper_2603_00035_b200/librfk.so
timeout 1800 python -m pytest tests/test_fullsize_parity_gpu.py tests/test_gpu_parity.py tests/test_edge_cases_gpu.py tests/test_fp32_mode.py -q -m gpu 2>&1 | tail -2 > gpurun_out/ed_parity.log
