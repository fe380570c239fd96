# A/B: the writer waits for batches of 1 (product) / 8 / 32 columns
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh wb1 wb8 wb32
