#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_rr.py -q -x -p no:cacheprovider 2>&1 | tail -25
timeout 300 python tools/rr_timing.py 30000 3000
CHASE_RR_JACOBI=1 timeout 300 python tools/rr_timing.py 30000 3000
