#!/bin/bash
# Round-2 (session 3): the full-size penetrating parity tests, the TMEM fold-interval accuracy
# sweep, and an ncu --set full capture (with source) of the paired local step.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batched.py -m gpu -q -x -s -k "penetrating" 2>&1 | tail -15 > gpurun_out/pen.log
timeout 600 python tools/drain_sweep.py 2 4 > gpurun_out/drain.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:k_local2<.int.0>" -s 2 -c 1 -o gpurun_out/full_local2 -f python tools/prof_batched.py 1024 1 > gpurun_out/full_local2.log 2>&1
python tools/ncu_summary.py gpurun_out/full_local2.ncu-rep > gpurun_out/full_local2.txt 2>&1
ncu -i gpurun_out/full_local2.ncu-rep --page raw --csv > gpurun_out/full_local2_raw.csv 2>/dev/null
ncu -i gpurun_out/full_local2.ncu-rep --page source --csv --print-source sass > gpurun_out/full_local2_sass.csv 2>/dev/null
true
