#!/bin/bash
# 1-GPU evidence on the final code: full GPU test suite, smoke, bench, launch list
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/final_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo rc=$? >> gpurun_out/final_smoke.log
python bench.py --steps 5 --warmup 3 > gpurun_out/final_bench1.log 2>&1; echo rc=$? >> gpurun_out/final_bench1.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/final_launches_bench1.csv python bench.py --steps 1 --warmup 3 --no-extras --no-sub --no-e2e --no-cpu-baseline > gpurun_out/final_ncu_launch.log 2>&1; echo ncu_launch_rc=$?
