mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 4 --config R --steps 2 --warmup 3 --no-extras --no-sub --no-e2e --no-cpu-baseline"
timeout 140 $B > gpurun_out/benchR4_final_fused.log 2>&1
timeout 140 $B --comm nccl > gpurun_out/benchR4_final_nccl.log 2>&1
