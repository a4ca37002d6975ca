#!/bin/bash
cd "$GRAFT_REPO_ROOT"
python -m pytest tests/test_gpu_hhqr.py -q -x -p no:cacheprovider 2>&1 | tail -2
for g in 148 96 64 32; do CHASE_HH_GRID=$g python tools/qr_timing.py 30000 3000 complex 2 | tail -1 | sed "s/^/grid $g /"; done
