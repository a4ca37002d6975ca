mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q > gpurun_out/virt_stage.log 2>&1; echo rc=$? >> gpurun_out/virt_stage.log
TAG=fself FUSED_SELF=1 python tools/hemm_timing.py 60000 3000 20 real > gpurun_out/fself_stage.log 2>&1
TAG=plain python tools/hemm_timing.py 60000 3000 20 real >> gpurun_out/fself_stage.log 2>&1
TAG=fself18944 FUSED_SELF=1 python tools/hemm_timing.py 18944 1024 4 real >> gpurun_out/fself_stage.log 2>&1
TAG=plain18944 python tools/hemm_timing.py 18944 1024 4 real >> gpurun_out/fself_stage.log 2>&1
