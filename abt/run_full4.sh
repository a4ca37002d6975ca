#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench4b.log 2>&1; echo rc=$? >> gpurun_out/bench4b.log
timeout 3000 python -m pytest tests/test_gpu_multi.py -k "full_size and not 2-4" -v -p no:cacheprovider > gpurun_out/full4.log 2>&1; echo rc=$? >> gpurun_out/full4.log
