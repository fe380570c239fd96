# A/B: writer role with a fence per lane before the progress release (wf1, current) vs the warp barrier only (wf0)
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh wf1 wf0
cp paper_2603_00035_b200/librfk_wf0.so paper_2603_00035_b200/librfk.so
timeout 1500 python -m pytest tests/test_fullsize_parity_gpu.py tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3 > gpurun_out/wf0_parity.log
