# sensitivity of the 4096^2 forward to the producer's chunk publication latency
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh pd0 pd1000 pd3000
