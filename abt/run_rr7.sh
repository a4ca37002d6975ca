#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_rr.py -q -x -p no:cacheprovider 2>&1 | tail -1
timeout 300 python tools/rr_timing.py 30000 3000
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rr_launches4.csv -c 20000 python tools/rr_timing.py 30000 3000 > /dev/null 2>&1
