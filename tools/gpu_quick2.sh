#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/prof_kpass_exp.py > gpurun_out/quick.txt 2>&1
timeout 2000 python -m pytest tests -m gpu -q 2>&1 | tail -6 >> gpurun_out/quick.txt
true
