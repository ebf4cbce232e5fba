#!/bin/bash
# GPU round trip used while developing: build check, the GPU tests (or a -k subset via
# TESTS_K), then optional extra commands from EXTRA.  Everything lands in gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
if [ -z "$SKIP_TESTS" ]; then
  if [ -n "$TESTS_K" ]; then
    timeout 1800 python -m pytest tests -m gpu -q --tb=line -p no:cacheprovider -k "$TESTS_K" 2>&1 > gpurun_out/pytest_gpu.log
  else
    timeout 1800 python -m pytest tests -m gpu -q --tb=line -p no:cacheprovider 2>&1 > gpurun_out/pytest_gpu.log
  fi
  tail -25 gpurun_out/pytest_gpu.log
fi
if [ -n "$EXTRA" ]; then bash -c "$EXTRA"; fi
true
