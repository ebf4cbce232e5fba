#!/bin/bash
# ncu --set full of one launch each of the plane-layout tensor-core K-passes at S = 1024
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for P in 1 2; do
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
      -k "regex:k_kpass_pl<.int.$P>" -s ${SKIP:-2} -c 1 -o gpurun_out/pl_$P -f python tools/prof_batched.py 1024 1 > gpurun_out/ncu_pl$P.log 2>&1
  tail -2 gpurun_out/ncu_pl$P.log
  python tools/ncu_summary.py gpurun_out/pl_$P.ncu-rep > gpurun_out/ncu_pl$P.txt 2>&1
done
