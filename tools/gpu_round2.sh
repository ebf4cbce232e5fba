#!/bin/bash
# Round profile set: launch list of the bench command, --set full of the top kernels at S = 1024
# (k_local, both TS K-passes, k_cr, k_gather), FP32 op counts of k_local.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-pile > gpurun_out/launches.out 2>&1; tail -1 gpurun_out/launches.out | head -c 300; echo
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_local|k_kpass_ts|k_cr|k_gather" -s 12 -c 6 -o gpurun_out/full_r01 -f \
  python tools/prof_batched.py 1024 1 > gpurun_out/full_r01.log 2>&1; tail -1 gpurun_out/full_r01.log
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__inst_executed_pipe_xu.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"k_local" -s 1 -c 2 --csv --log-file gpurun_out/local_ops.csv python tools/prof_batched.py 1024 1 > gpurun_out/local_ops.log 2>&1; tail -1 gpurun_out/local_ops.log
true
