#!/bin/bash
# Round-2 evidence: launch lists (cfg5 S = 1024 and the single cfg3 scene) with DRAM bytes, ncu --set
# full of the top kernels (paired local step, plane K-passes), and a summary of each.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv \
    python tools/prof_batched.py 1024 2 > gpurun_out/launches_cfg5.log 2>&1
python tools/launches.py gpurun_out/launches_cfg5.csv > gpurun_out/launches_cfg5.txt 2>&1
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_single.csv \
    python tools/prof_single.py 4 > gpurun_out/launches_single.log 2>&1
python tools/launches.py gpurun_out/launches_single.csv > gpurun_out/launches_single.txt 2>&1
for K in "k_local2<.int.0>" "k_kpass_pl<.int.1>" "k_kpass_pl<.int.2>"; do
  N=$(echo "$K" | tr -cd 'a-z0-9_')
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
      -k "regex:$K" -s 2 -c 1 -o gpurun_out/full_$N -f python tools/prof_batched.py 1024 1 > gpurun_out/full_$N.log 2>&1
  python tools/ncu_summary.py gpurun_out/full_$N.ncu-rep > gpurun_out/full_$N.txt 2>&1
  ncu -i gpurun_out/full_$N.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv, sys
rows = list(csv.reader(sys.stdin)); h = rows[0]; v = rows[2]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__sass_thread_inst_executed_op_ffma_pred_on.sum', 'sm__sass_thread_inst_executed_op_fmul_pred_on.sum', 'sm__sass_thread_inst_executed_op_fadd_pred_on.sum']
for i, n in enumerate(h):
    if n in want: print(n, v[i], rows[1][i])
" >> gpurun_out/full_$N.txt 2>&1
done
