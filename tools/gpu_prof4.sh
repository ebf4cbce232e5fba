#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_cfg4.csv python tools/prof_cfg4_min.py 2 > gpurun_out/launches_cfg4.out 2>&1; tail -2 gpurun_out/launches_cfg4.out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_kpass1|k_kpass2|k_gcr_gram|k_gcr_slot|k_gcr_row|k_local" -s 300 -c 6 -o gpurun_out/full_cfg4 -f \
  python tools/prof_cfg4_min.py 2 > gpurun_out/full_cfg4.log 2>&1; tail -2 gpurun_out/full_cfg4.log
true
