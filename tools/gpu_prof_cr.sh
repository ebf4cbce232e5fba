#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:"k_cr" -s 3 -c 1 -o gpurun_out/prof_cr python tools/prof_frames.py 1 > gpurun_out/prof_cr.out 2>&1
tail -3 gpurun_out/prof_cr.out
