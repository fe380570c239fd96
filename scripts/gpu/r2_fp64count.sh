# absolute FP64 instruction counts of one C3 sweep launch (current build)
mkdir -p gpurun_out
timeout 900 ncu --metrics smsp__inst_executed_pipe_fp64.sum,smsp__inst_executed.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,gpu__time_duration.sum --clock-control none -k regex:sweep_kernel -c 1 --csv --log-file gpurun_out/sweep_fp64_inst.csv python scripts/prof_solve.py 4096 > gpurun_out/ncu_fp64.log 2>&1
