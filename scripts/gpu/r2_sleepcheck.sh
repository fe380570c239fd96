# the product build with RFK_SWEEP_SLEEP 16 vs 1 at 1024^2 and 256^2; then the full suite/bench
mkdir -p gpurun_out
AB_N=1024 bash scripts/ab.sh sl1 sl16p
AB_N=256 bash scripts/ab.sh sl1 sl16p
cp paper_2603_00035_b200/librfk_sl16p.so paper_2603_00035_b200/librfk.so
rm -f paper_2603_00035_b200/librfk_sl*.so
bash scripts/gpu/r2_final2.sh
