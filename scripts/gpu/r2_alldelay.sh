# sensitivity of the 4096^2 forward to a delay added to every step (dirty or clean)
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh as0 as100 as300
