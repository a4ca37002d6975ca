#!/bin/bash
cd "$GRAFT_REPO_ROOT"
python -m pytest tests/test_gpu_hhqr.py tests/test_gpu_qr.py -q -x -p no:cacheprovider 2>&1 | tail -3
python tools/qr_timing.py 30000 3000 complex 2 | tail -1
CHASE_HH_PER_COLUMN=1 python tools/qr_timing.py 30000 3000 complex 2 | tail -1
python tools/qr_timing.py 60000 2500 real 2 | tail -1
