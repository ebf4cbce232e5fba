cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for u in 2 1 4 8; do echo "== SIM_TS_CTAS_PER_SM=$u"; SIM_TS_CTAS_PER_SM=$u timeout 300 python tools/prof_kpass_exp.py 2>&1 | head -1 | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('chain', d['chain_dot'], 'scatter', d['scatter'])"; done; done > gpurun_out/ts.txt 2>&1
