#!/bin/bash
# quick check: cfg5 per-frame kernel times (in-graph events), batched + parity GPU tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/prof_kpass_exp.py > gpurun_out/quick.txt 2>&1
[ -z "$SKIP_TESTS" ] && timeout 1200 python -m pytest tests/test_gpu_batched.py tests/test_gpu_parity.py tests/test_gpu_grid_cr.py -m gpu -q -x 2>&1 | tail -3 >> gpurun_out/quick.txt
true
