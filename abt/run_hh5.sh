#!/bin/bash
cd "$GRAFT_REPO_ROOT"
python -m pytest tests/test_gpu_hhqr.py -q -x -p no:cacheprovider 2>&1 | tail -1
python tools/qr_timing.py 30000 3000 complex 2 2>&1 | tail -1
python tools/qr_timing.py 60000 2500 real 2 2>&1 | tail -1
