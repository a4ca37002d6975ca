#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
python bench.py --steps 3 --warmup 3 > gpurun_out/bench1.log 2>&1; echo rc=$? >> gpurun_out/bench1.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches_bench1.csv python bench.py --steps 1 --warmup 3 --no-extras --no-sub --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch_rc=$?
ncu --set full --clock-control none -k regex:zgemm_kernel -c 2 -o /tmp/ncu/hemm --force-overwrite python tools/profile_hemm.py 30000 3000 > gpurun_out/ncu_hemm.log 2>&1; echo ncu_hemm_rc=$?
ncu --set full --clock-control none --nvtx --nvtx-include "gram/" -c 1 -o /tmp/ncu/gram --force-overwrite python tools/qr_timing.py 30000 3000 complex 1 > gpurun_out/ncu_gram.log 2>&1; echo ncu_gram_rc=$?
ncu --set full --clock-control none --nvtx --nvtx-include "trsm/" -k regex:zgemm_kernel -c 14 -o /tmp/ncu/trsm --force-overwrite python tools/qr_timing.py 30000 3000 complex 1 > gpurun_out/ncu_trsm.log 2>&1; echo ncu_trsm_rc=$?
for r in hemm gram trsm; do
  ncu -i /tmp/ncu/$r.ncu-rep --page details --csv > gpurun_out/ncu_${r}_details.csv 2>/dev/null
  ncu -i /tmp/ncu/$r.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,launch__grid_size > gpurun_out/ncu_${r}_raw.csv 2>/dev/null
done
ls -la gpurun_out /tmp/ncu
