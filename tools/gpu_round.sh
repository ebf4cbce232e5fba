#!/bin/bash
# Round measurement: GPU tests, smoke, default bench line, ncu launch list of the bench command,
# ncu --set full of the batched K-pass.  Everything lands in gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
[ -z "$SKIP_TESTS" ] && { timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.log; tail -4 gpurun_out/pytest_gpu.log; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; head -c 3000 gpurun_out/bench.json
[ -z "$SKIP_NCU" ] && {
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/launches.out 2>&1; tail -2 gpurun_out/launches.out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_kpass" -s 6 -c 2 -o gpurun_out/full_kpass -f \
  python tools/prof_batched.py 128 2 > gpurun_out/full_kpass.log 2>&1; tail -2 gpurun_out/full_kpass.log
}
true
