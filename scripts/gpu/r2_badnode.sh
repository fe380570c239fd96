mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "inconsistent" 2>&1 | tail -15 > gpurun_out/badnode.log
