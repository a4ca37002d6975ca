#!/bin/bash
cd "$GRAFT_REPO_ROOT"
ncu --set full --import-source on --clock-control none -k regex:"potrf_diag|potrf_panel" -c 4 -o gpurun_out/ncu_potrf --force-overwrite python tools/qr_timing.py 30000 3000 complex 1 > gpurun_out/ncu_potrf.log 2>&1
echo rc=$?
