set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q > gpurun_out/virt_tail.log 2>&1; echo rc=$? >> gpurun_out/virt_tail.log
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config R --steps 2 --warmup 3 --no-extras --no-sub --no-e2e"
timeout 600 $B > gpurun_out/benchR2t.log 2>&1
CHASE_FUSED_NO_TAIL=1 timeout 600 $B > gpurun_out/benchR2nt.log 2>&1
