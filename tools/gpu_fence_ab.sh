mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q > gpurun_out/virt_fence.log 2>&1; echo rc=$? >> gpurun_out/virt_fence.log
TAG=fself FUSED_SELF=1 python tools/hemm_timing.py 60000 3000 20 real > gpurun_out/fself_fence.log 2>&1
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config R --steps 2 --warmup 3 --no-extras --no-sub --no-e2e"
timeout 600 $B > gpurun_out/benchR2f.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi2_fence.log 2>&1; echo rc=$? >> gpurun_out/multi2_fence.log
