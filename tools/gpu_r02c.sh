#!/bin/bash
# CR phase timeline of the single scene, drop-tolerance table (cfg3, cfg4), single-scene launch list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/cr_timeline_single.py > gpurun_out/cr_timeline.txt 2>&1
timeout 600 python tools/drop_tolerance.py cfg3 > gpurun_out/drop_cfg3.txt 2>&1
timeout 900 python tools/drop_tolerance.py cfg4 > gpurun_out/drop_cfg4.txt 2>&1
true
