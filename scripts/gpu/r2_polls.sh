# A/B: sleeps in the compute warps' input poll (cp20/cp60 ns) and in the mailbox poll when nothing arrived (mp32/mp128 ns)
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh pp0 cp20 cp60 mp32 mp128
