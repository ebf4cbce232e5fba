cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for v in s35 s42; do cp libsim_$v.so.alt paper_2503_15078_b200/libsim.so; echo "== $v"; timeout 300 python tools/prof_kpass_exp.py 2>&1 | tail -1; done; done > gpurun_out/ab2.txt 2>&1
