# A/B: hoisted-record TMA groups: HG=8 x HB=4 (product), HG=16 x HB=2, HG=8 x HB=3
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh hb0 hg16 hb3
