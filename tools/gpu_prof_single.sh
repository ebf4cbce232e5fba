#!/bin/bash
# single-scene cfg3: ncu launch list (2 frames after setup) and --set full of the two K-passes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_single.csv python tools/prof_frames.py 3 > gpurun_out/launches_single.out 2>&1; tail -1 gpurun_out/launches_single.out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_kpass1|k_kpass2|k_cr|k_local" -s 8 -c 4 -o gpurun_out/full_single -f \
  python tools/prof_frames.py 3 > gpurun_out/full_single.log 2>&1; tail -1 gpurun_out/full_single.log
true
