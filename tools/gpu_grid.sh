#!/bin/bash
# grid-CR / cfg4 GPU round trip: new tests first, then the whole GPU suite, then cfg4 frame timing
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_grid_cr.py -q -x 2>&1 | tail -30 > gpurun_out/pytest_grid.log; tail -25 gpurun_out/pytest_grid.log
[ -z "$SKIP_ALL" ] && { timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log; tail -6 gpurun_out/pytest_gpu.log; }
[ -n "$PROF4" ] && timeout 900 python tools/prof_cfg4.py > gpurun_out/cfg4.log 2>&1; tail -20 gpurun_out/cfg4.log
true
