# delay-injection map (base: vote consumed at the commit): q1 +4 DADD on the step index
# before the address arithmetic, q2 +4 DADD on t1/t2 after their loads, q3 +4 DADD after the fold
mkdir -p gpurun_out
AB_N=4096 bash scripts/ab.sh q0 q1 q2 q3
