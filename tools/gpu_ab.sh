cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do timeout 300 python tools/prof_kpass_exp.py 2>&1 | tail -1; done > gpurun_out/ab.txt 2>&1
timeout 300 python tools/pl_timeline.py > gpurun_out/pl_timeline.txt 2>&1
