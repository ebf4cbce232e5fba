#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on --warp-sampling-interval 2 -k regex:"k_kpass1|k_kpass2" -s 4 -c 2 -o gpurun_out/prof5 python tools/prof_frames.py 1 > gpurun_out/prof5.out 2>&1
tail -2 gpurun_out/prof5.out
