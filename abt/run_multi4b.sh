#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -k "not full_size" -q -p no:cacheprovider > gpurun_out/multi4b_tests.log 2>&1; echo rc=$? >> gpurun_out/multi4b_tests.log
timeout 1500 python bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench4c.log 2>&1; echo rc=$? >> gpurun_out/bench4c.log
