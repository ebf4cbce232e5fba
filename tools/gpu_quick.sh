#!/bin/bash
cd $GRAFT_REPO_ROOT
python tools/prof_frames.py 3 2>&1 | tail -3
