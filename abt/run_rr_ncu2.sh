#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p /tmp/ncu
ncu --set full --clock-control none --nvtx --nvtx-include "chase_rayleigh_ritz/other/" -k regex:zgemm_kernel --launch-skip 3 -c 6 -o /tmp/ncu/rr --force-overwrite python tools/rr_timing.py 30000 3000 > gpurun_out/rr_ncu2.log 2>&1
ncu -i /tmp/ncu/rr.ncu-rep --page details --csv > gpurun_out/ncu_rr_details.csv 2>/dev/null
ncu -i /tmp/ncu/rr.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,launch__grid_size,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio > gpurun_out/ncu_rr_raw.csv 2>/dev/null
