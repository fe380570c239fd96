# A/B: no sticky body entry (every step waits for the dirty vote) vs sticky (product)
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh ns0 ns1
