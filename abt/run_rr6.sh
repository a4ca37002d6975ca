#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_rr.py tests/test_gpu_solve.py -q -x -p no:cacheprovider 2>&1 | tail -2
python abt/dbg_rr2.py 2>&1 | tail -4
timeout 300 python tools/rr_timing.py 30000 3000
CHASE_TRD_UNFUSED=1 timeout 300 python tools/rr_timing.py 30000 3000
