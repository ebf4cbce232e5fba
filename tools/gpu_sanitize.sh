#!/bin/bash
# compute-sanitizer memcheck / synccheck / racecheck / initcheck over tools/sanitize.py
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for T in memcheck synccheck racecheck initcheck; do
  echo "## $T" >> gpurun_out/sanitizer.txt
  timeout 1500 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize.py > gpurun_out/san_$T.log 2>&1
  grep -E "ERROR SUMMARY|sanitize run done" gpurun_out/san_$T.log >> gpurun_out/sanitizer.txt
done
