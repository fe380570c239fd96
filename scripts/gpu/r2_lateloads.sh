# A/B: operand loads after the take decision (ll1) vs before the vote (ll0, product)
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh ll0 ll1
