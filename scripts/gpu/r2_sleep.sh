# A/B: role-warp poll back-off multiplier (RFK_SWEEP_SLEEP 1 = product, 16, 32, 64)
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh sl1 sl16 sl32 sl64
AB_N=2048 bash scripts/ab.sh sl1 sl16 sl32
