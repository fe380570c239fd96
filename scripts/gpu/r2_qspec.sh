# A/B of the speculated validity test (qs1) against the previous chain (qs0), then parity with qs1
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh qs0 qs1
cp paper_2603_00035_b200/librfk_qs1.so paper_2603_00035_b200/librfk.so
timeout 1500 python -m pytest tests/test_fullsize_parity_gpu.py tests/test_gpu_parity.py tests/test_edge_cases_gpu.py -q -m gpu -x 2>&1 | tail -5 > gpurun_out/qspec_parity.log
