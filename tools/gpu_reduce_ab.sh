mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q > gpurun_out/virt_red.log 2>&1; echo rc=$? >> gpurun_out/virt_red.log
TAG=fself FUSED_SELF=1 python tools/hemm_timing.py 60000 3000 20 real > gpurun_out/fself_red.log 2>&1
TAG=fself18944 FUSED_SELF=1 python tools/hemm_timing.py 18944 1024 4 real >> gpurun_out/fself_red.log 2>&1
TAG=plain18944 python tools/hemm_timing.py 18944 1024 4 real >> gpurun_out/fself_red.log 2>&1
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --no-extras --no-sub --no-e2e"
timeout 600 $B --config R > gpurun_out/benchR2red.log 2>&1
timeout 600 $B --config R --comm nccl > gpurun_out/benchR2redn.log 2>&1
