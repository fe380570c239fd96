# the product build with 16-step TMA groups x 2: parity, protocol checker, fault control
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_fullsize_parity_gpu.py tests/test_gpu_parity.py tests/test_edge_cases_gpu.py tests/test_fp32_mode.py tests/test_fused_projection_gpu.py tests/test_protocol_checker_gpu.py -q -m gpu 2>&1 | tail -3 > gpurun_out/hg16_parity.log
RFK_LIBRARY=$PWD/paper_2603_00035_b200/librfk_chk.so timeout 1500 python scripts/check_protocols.py > gpurun_out/protocols_checked.log 2>&1; echo "rc=$?" >> gpurun_out/protocols_checked.log
