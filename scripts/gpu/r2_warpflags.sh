# A/B: per-warp progress flags (pw1) vs the compute warps' step barrier (pw0); then parity + stress with pw1
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh pw0 pw1
cp paper_2603_00035_b200/librfk_pw1.so paper_2603_00035_b200/librfk.so
timeout 900 python -m pytest tests/test_fullsize_parity_gpu.py tests/test_gpu_parity.py tests/test_edge_cases_gpu.py -q -m gpu -x 2>&1 | tail -2 > gpurun_out/pw_parity.log
REPS=10 timeout 900 python scripts/check_protocols.py > gpurun_out/pw_stress.log 2>&1; echo "rc=$?" >> gpurun_out/pw_stress.log
