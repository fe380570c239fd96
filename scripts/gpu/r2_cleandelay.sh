# sensitivity of the 4096^2 forward to the cost of a clean step (no warp of the band evaluates)
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh cs0 cs200 cs600
