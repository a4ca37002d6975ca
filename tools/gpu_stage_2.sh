mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi2_stage.log 2>&1; echo rc=$? >> gpurun_out/multi2_stage.log
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --no-extras --no-sub --no-e2e --no-cpu-baseline"
timeout 600 $B --config R > gpurun_out/benchR2stage.log 2>&1
timeout 600 $B --config R --comm nccl > gpurun_out/benchR2stagen.log 2>&1
