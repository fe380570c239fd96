# fp32 backward tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fp32_mode.py -k 4096 -q -m gpu -rA 2>&1 | grep -v "^PASSED" | tail -60 > gpurun_out/fp32_tests.log
