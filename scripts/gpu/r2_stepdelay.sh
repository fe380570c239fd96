# sensitivity of the 4096^2 forward to the dirty-step latency (extra dependent DADDs on the stencil chain)
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh sd0 sd4 sd8
