#!/bin/bash
# K-pass variant check: per-frame kernel times at S = 1024, K-apply accuracy vs fold interval, batched GPU tests.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/prof_kpass_exp.py > gpurun_out/kp.txt 2>&1
timeout 600 python tools/drain_sweep.py 2 4 >> gpurun_out/kp.txt 2>&1
[ -z "$SKIP_TESTS" ] && timeout 1200 python -m pytest tests/test_gpu_batched.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -5 >> gpurun_out/kp.txt
true
