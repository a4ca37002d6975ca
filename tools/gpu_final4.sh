# 4-GPU evidence on the final code: multi-GPU suite (incl. full-size grids, fused + nccl), benches
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_multi.py -q -rs > gpurun_out/multi4_final.log 2>&1; echo rc=$? >> gpurun_out/multi4_final.log
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4"
timeout 1200 $B --steps 3 --warmup 3 > gpurun_out/bench4_final.log 2>&1
timeout 600 $B --config R --steps 2 --warmup 3 --no-extras --no-sub --no-e2e > gpurun_out/benchR4_fused.log 2>&1
timeout 600 $B --config R --steps 2 --warmup 3 --no-extras --no-sub --no-e2e --comm nccl > gpurun_out/benchR4_nccl.log 2>&1
