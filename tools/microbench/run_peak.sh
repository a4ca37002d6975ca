#!/bin/bash
# FP64 peak microbenchmarks on one B200 with clocks sampled during the run.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 -i 0 > gpurun_out/peak_clocks.csv &
SMI=$!
./tools/microbench/fp64_peak > gpurun_out/fp64_peak.log 2>&1
python tools/microbench/torch_gemm.py > gpurun_out/torch_gemm.log 2>&1
kill $SMI
nproc > gpurun_out/host_info.txt; lscpu | head -20 >> gpurun_out/host_info.txt; free -g >> gpurun_out/host_info.txt
nvidia-smi topo -m >> gpurun_out/host_info.txt 2>&1
