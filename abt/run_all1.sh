#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_all1.log 2>&1; echo rc=$? >> gpurun_out/pytest_all1.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rr_launches2.csv -c 20000 python tools/rr_timing.py 30000 3000 > gpurun_out/rr_ncu3.log 2>&1
