#!/bin/bash
cd "$GRAFT_REPO_ROOT"
python -m pytest tests/test_gpu_qr.py tests/test_gpu_hhqr.py tests/test_gpu_solve.py -q -x -p no:cacheprovider 2>&1 | tail -4
python tools/qr_timing.py 30000 3000
CHASE_TRSM_BLOCKED=1 CHASE_NO_GRAM_SPLIT=1 python tools/qr_timing.py 30000 3000
python tools/qr_timing.py 60000 1300
python tools/qr_timing.py 60000 2500 real
