#!/bin/bash
# Launch list (ncu, serialised) of the single cfg3 scene with the contact set re-committed every frame.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_single.csv \
    python tools/prof_single.py 4 > gpurun_out/launches_single.log 2>&1
python tools/launches.py gpurun_out/launches_single.csv > gpurun_out/launches_single.txt 2>&1
true
