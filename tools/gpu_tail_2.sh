mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --no-extras --no-sub --no-e2e"
timeout 600 $B --config R > gpurun_out/benchR2t.log 2>&1
timeout 600 $B > gpurun_out/benchC2t.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi2_tail.log 2>&1; echo rc=$? >> gpurun_out/multi2_tail.log
