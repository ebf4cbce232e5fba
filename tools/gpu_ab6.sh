cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for v in t64 t32; do cp libsim_$v.so.alt paper_2503_15078_b200/libsim.so; echo "== $v"; timeout 300 python tools/prof_kpass_exp.py 2>&1 | head -1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('local', d['local'])"; done; done > gpurun_out/ab6.txt 2>&1
