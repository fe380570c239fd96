# sensitivity: +4 dependent DADDs after the fold (before relax) vs none
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh fe0 fe4
