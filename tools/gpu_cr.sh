#!/bin/bash
# CR work: timeline of the single scene, single-scene frame timing, GPU test suite.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/cr_timeline_single.py > gpurun_out/cr_timeline.txt 2>&1
timeout 300 python tools/prof_single.py 20 2>&1 | grep -v "^{" > gpurun_out/prof_single.txt
[ -z "$SKIP_TESTS" ] && timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
true
