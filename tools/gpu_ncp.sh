#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ncp_ablation.py -q -x 2>&1 | tail -30 > gpurun_out/pytest_ncp.log; tail -20 gpurun_out/pytest_ncp.log
timeout 900 python tools/fig11_ablation.py 100 > gpurun_out/fig11.log 2>&1; cat gpurun_out/fig11.log | tail -80
true
