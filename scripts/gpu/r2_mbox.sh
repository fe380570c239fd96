# sensitivity of the 4096^2 forward to the band-to-band hand-off latency (extra delay in the mailbox role)
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh md0 md500 md1000
