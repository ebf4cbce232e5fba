cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for u in 96 128 192; do echo "== SIM_PL_UNIT_TILES=$u"; SIM_PL_UNIT_TILES=$u timeout 300 python tools/prof_kpass_exp.py 2>&1 | tail -1; done > gpurun_out/ut.txt 2>&1
for u in 48 96 128; do echo "== SIM_PL_UNIT_TILES=$u"; SIM_PL_UNIT_TILES=$u timeout 600 python tools/drain_sweep.py 4 2>&1 | tail -1; done >> gpurun_out/ut.txt 2>&1
