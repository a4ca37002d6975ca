# complex W4 point on 2x2: fused HEMM + NVLink reduction vs HEMM + ncclAllReduce, same box
mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus 4 --steps 2 --warmup 3 --no-extras --no-sub --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/benchC4_fused.log 2>&1
timeout 600 $B --comm nccl > gpurun_out/benchC4_nccl.log 2>&1
