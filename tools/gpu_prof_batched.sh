#!/bin/bash
# ncu --set full of the batched hot kernels (S = 128 instances), one launch each
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/prof_batched.py 128 1
for K in k_local k_kpass_b k_scatter k_chain_dot k_cr k_gather; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$K -s 2 -c 1 -o gpurun_out/b_$K -f python tools/prof_batched.py 128 1 > gpurun_out/ncu_$K.log 2>&1
  tail -2 gpurun_out/ncu_$K.log
done
