#!/bin/bash
# DRAM bytes and duration of the TS K-passes at S = 1024 (one frame after warm-up)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_kpass_ts" -s 8 -c 4 --csv \
  --log-file gpurun_out/kpass_traffic.csv python tools/prof_batched.py 1024 2 > gpurun_out/kpass_traffic.log 2>&1
python tools/launches.py gpurun_out/kpass_traffic.csv
