#!/bin/bash
# ncu --set full (with source) of one k_local<0> launch at S = 1024, and the launch list of a frame
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:k_local<.int.0>" -s ${SKIP:-2} -c 1 -o gpurun_out/local_0 -f python tools/prof_batched.py 1024 1 > gpurun_out/ncu_local.log 2>&1
tail -2 gpurun_out/ncu_local.log
python tools/ncu_summary.py gpurun_out/local_0.ncu-rep > gpurun_out/ncu_local.txt 2>&1
