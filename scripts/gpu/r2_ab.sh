# A/B of sweep variants + a trace of the current build (round 2)
AB_REPS=2 bash scripts/ab_env.sh ${AB_VARIANTS:-s0 s1 s2}
cp paper_2603_00035_b200/librfk_s1.so paper_2603_00035_b200/librfk.so
RFK_TRACE=1 timeout 300 python scripts/trace_sweep.py 4096 all > gpurun_out/trace.log 2>&1
