#!/bin/bash
# final code on 2 GPUs: whole GPU suite (1-GPU cases + 2-GPU multi cases), smoke, 2-GPU bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/final2_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/final2_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2_smoke.log 2>&1; echo rc=$? >> gpurun_out/final2_smoke.log
timeout 1200 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/final2_bench2.log 2>&1; echo rc=$? >> gpurun_out/final2_bench2.log
