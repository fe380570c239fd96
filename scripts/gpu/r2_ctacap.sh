# CTA cap sweep of the current build (is the forward CTA-bound?)
mkdir -p gpurun_out
AB_N=4096 AB_REPS=1 bash scripts/ab_env.sh cur:148 cur:136 cur:120 cur:100 cur:74
