#!/bin/bash
cd "$GRAFT_REPO_ROOT"
python tools/rr_timing.py 30000 3000 > gpurun_out/rr_timing.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rr_launches.csv -c 5000 python tools/rr_timing.py 30000 3000 > gpurun_out/rr_ncu.log 2>&1
echo rc=$?
