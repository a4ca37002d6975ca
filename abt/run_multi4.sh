#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo4.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py -k "not full_size" -q -p no:cacheprovider > gpurun_out/multi4_tests.log 2>&1; echo rc=$? >> gpurun_out/multi4_tests.log
timeout 1500 python bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench4.log 2>&1; echo rc=$? >> gpurun_out/bench4.log
timeout 1200 python bench.py --gpus 2 --steps 3 --warmup 3 --no-sub > gpurun_out/bench2.log 2>&1; echo rc=$? >> gpurun_out/bench2.log
