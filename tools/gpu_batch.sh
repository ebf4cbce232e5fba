#!/bin/bash
# GPU round trip: all GPU tests, the default bench line (cfg5, 1024 scenes + single-scene), extra S.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
[ -z "$SKIP_TESTS" ] && timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -40 > gpurun_out/pytest_gpu.log; tail -6 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print({k: d[k] for k in ("value", "ms_per_step", "scaling")}, d["single_scene"])
print({k: round(v) for k, v in d["kernel_us_per_step"].items()})
print(d["roofline"]); print(d["e2e"]); print(d["breakdown"]); print(d["cpu_baseline"]); print(d["clocks"])
PY
for S in ${BENCH_S:-}; do
  timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --instances $S > gpurun_out/bench_S$S.json 2> gpurun_out/bench_S$S.err
  tail -3 gpurun_out/bench_S$S.err; python -c "import json;d=json.load(open('gpurun_out/bench_S$S.json'));print('S=$S', d['value'], d['ms_per_step']);print({k: round(v) for k, v in d['kernel_us_per_step'].items()})"
done
