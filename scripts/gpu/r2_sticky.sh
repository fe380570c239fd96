# A/B: a warp enters the stencil body before its dirty vote when it was dirty in the last 1 (st1, product) / 2 / 4 steps
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh st1 st2 st4
