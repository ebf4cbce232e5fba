#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_frames.py 2 > gpurun_out/launches.out 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_kpass1|k_kpass2|k_local|k_scatter|k_chain_dot|k_cr" -s 12 -c 6 -o gpurun_out/prof1 python tools/prof_frames.py 2 > gpurun_out/prof1.out 2>&1
ls -la gpurun_out
