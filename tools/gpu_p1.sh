cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 1024 512 256 128; do echo "== SIM_P1_ITEM_COLS=$c"; SIM_P1_ITEM_COLS=$c timeout 300 python tools/prof_single.py 30 2>&1 | grep -v "^{" | head -3; done > gpurun_out/p1.txt 2>&1
