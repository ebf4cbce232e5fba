#!/bin/bash
# ncu --set full (with source) of the cluster CR on the single cfg3 scene.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/cr_timeline_single.py > gpurun_out/cr_timeline.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:k_cr<" -s 10 -c 1 -o gpurun_out/full_cr -f python tools/cr_timeline_single.py > gpurun_out/full_cr.log 2>&1
python tools/ncu_summary.py gpurun_out/full_cr.ncu-rep > gpurun_out/full_cr.txt 2>&1
ncu -i gpurun_out/full_cr.ncu-rep --page raw --csv > gpurun_out/full_cr_raw.csv 2>/dev/null
ncu -i gpurun_out/full_cr.ncu-rep --page source --csv --print-source sass > gpurun_out/full_cr_sass.csv 2>/dev/null
ncu -i gpurun_out/full_cr.ncu-rep --page source --csv --print-source cuda > gpurun_out/full_cr_cuda.csv 2>/dev/null
true
