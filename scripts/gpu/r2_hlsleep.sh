# A/B: TMA loader sleeps after an unfinished mbarrier try_wait (64 / 256 ns) vs none (product)
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh hl0 hl64 hl256
