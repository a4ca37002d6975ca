#!/bin/bash
cd "$GRAFT_REPO_ROOT"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qr_launches.csv python tools/qr_timing.py 30000 3000 complex 1 > gpurun_out/qr_ncu.log 2>&1
echo rc=$?
