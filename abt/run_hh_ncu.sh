#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p /tmp/ncu
ncu --set full --clock-control none -k regex:"hh_reflect|hh_update" --launch-skip 200 -c 2 -o /tmp/ncu/hh --force-overwrite python tools/qr_timing.py 30000 3000 complex 1 > gpurun_out/hh_ncu.log 2>&1
ncu -i /tmp/ncu/hh.ncu-rep --page details --csv > gpurun_out/ncu_hh_details.csv 2>/dev/null
ncu -i /tmp/ncu/hh.ncu-rep --page source --csv > gpurun_out/ncu_hh_source.csv 2>/dev/null
