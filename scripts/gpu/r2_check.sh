# round-2 check: parity (goldens + full size), stress, A/B timing, trace
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_parity_gpu.py -x -q 2>&1 | tail -5
REPS=${REPS:-30} timeout 300 python scripts/dbg_hist.py 2>&1 | tail -8
AB_REPS=2 bash scripts/ab_env.sh ${AB_VARIANTS:-s0 s1 s2 s1w s0w}
cp paper_2603_00035_b200/librfk_s1.so paper_2603_00035_b200/librfk.so
RFK_TRACE=1 timeout 300 python scripts/trace_sweep.py 4096 all > gpurun_out/trace_s1.log 2>&1
