#!/bin/bash
# GPU round trip for the batched path: all GPU tests, single-scene bench, batched benches.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
[ -z "$SKIP_TESTS" ] && timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.log; tail -6 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -3 gpurun_out/bench1.err; cut -c1-600 gpurun_out/bench1.json
for S in ${BENCH_S:-128 1024}; do
  timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --instances $S > gpurun_out/bench_S$S.json 2> gpurun_out/bench_S$S.err
  tail -3 gpurun_out/bench_S$S.err; cut -c1-400 gpurun_out/bench_S$S.json; python -c "import json;d=json.load(open('gpurun_out/bench_S$S.json'));print(d['kernel_us_per_step']);print(d['roofline']);print(d['e2e']);print(d['breakdown'])"
done
