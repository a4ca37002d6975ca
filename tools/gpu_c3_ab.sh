mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "full_size_grid and C3-grid0-fused" > gpurun_out/c3_tail.log 2>&1; echo rc=$? >> gpurun_out/c3_tail.log
timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q > gpurun_out/virt_push.log 2>&1; echo rc=$? >> gpurun_out/virt_push.log
