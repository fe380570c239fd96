# A/B: next-step addresses computed ahead of the barrier (pp1: in the sqrt's shadow, pp2: after the operand loads) vs pp0
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh pp0 pp1 pp2
