#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/final_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo rc=$? >> gpurun_out/final_smoke.log
python bench.py --steps 5 --warmup 3 > gpurun_out/final_bench1.log 2>&1; echo rc=$? >> gpurun_out/final_bench1.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/final_launches_bench1.csv python bench.py --steps 1 --warmup 3 --no-extras --no-sub --no-e2e --no-cpu-baseline > gpurun_out/final_ncu_launch.log 2>&1; echo ncu_launch_rc=$?
ncu --set full --clock-control none -k regex:zgemm_kernel -c 2 -o /tmp/ncu/hemm --force-overwrite python tools/profile_hemm.py 30000 3000 > gpurun_out/final_ncu_hemm.log 2>&1; echo ncu_hemm_rc=$?
ncu --set full --clock-control none -k regex:dgemm_kernel -c 2 -o /tmp/ncu/dhemm --force-overwrite python tools/profile_hemm.py 60000 2500 real > gpurun_out/final_ncu_dhemm.log 2>&1; echo ncu_dhemm_rc=$?
for r in hemm dhemm; do
  ncu -i /tmp/ncu/$r.ncu-rep --page details --csv > gpurun_out/final_ncu_${r}_details.csv 2>/dev/null
  ncu -i /tmp/ncu/$r.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,launch__grid_size,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,launch__registers_per_thread > gpurun_out/final_ncu_${r}_raw.csv 2>/dev/null
done
