# ncu --set full: plain dgemm_kernel vs fused-self dgemm_fused_kernel on the same even step
mkdir -p /tmp/ncu gpurun_out
M="gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_op_dmma.sum,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,launch__grid_size,smsp__warp_issue_stalled_barrier_per_warp_active.pct,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_wait_per_warp_active.pct,smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct,smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_membar_per_warp_active.pct,smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct,smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct,smsp__cycles_active.avg,sm__cycles_elapsed.avg,l1tex__t_bytes_pipe_lsu_mem_global_op_st.sum,l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum"
ncu --set full --clock-control none --import-source on -k regex:"dgemm_kernel" -s 1 -c 1 -o /tmp/ncu/plain python tools/hemm_timing.py 18944 1024 4 real > gpurun_out/ncu_fvp_plain.log 2>&1
FUSED_SELF=1 ncu --set full --clock-control none --import-source on -k regex:"dgemm_fused_kernel" -s 1 -c 1 -o /tmp/ncu/fused python tools/hemm_timing.py 18944 1024 4 real > gpurun_out/ncu_fvp_fused.log 2>&1
for r in plain fused; do
  ncu -i /tmp/ncu/$r.ncu-rep --page raw --csv --metrics $M > gpurun_out/ncu_fvp_${r}_raw.csv 2>&1
done
