#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/diag2.py cfg3 > gpurun_out/diag2.log 2>&1; cat gpurun_out/diag2.log
timeout 900 python tools/diag2.py incline >> gpurun_out/diag2.log 2>&1; tail -12 gpurun_out/diag2.log
