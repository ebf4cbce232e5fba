cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for v in s128 s64 s32; do cp libsim_$v.so.alt paper_2503_15078_b200/libsim.so; echo "== $v"; timeout 300 python tools/prof_single.py 30 2>&1 | grep -v "^{" | sed -n 1,2p; done; done > gpurun_out/ab7.txt 2>&1
