#!/bin/bash
cd "$GRAFT_REPO_ROOT"
python -m pytest tests/test_gpu_qr.py tests/test_gpu_hhqr.py tests/test_gpu_solve.py tests/test_gpu_full.py -q -x -p no:cacheprovider 2>&1 | tail -2
python tools/qr_timing.py 30000 3000 complex 3 | head -1
python tools/qr_timing.py 60000 2500 real 3 | head -1
