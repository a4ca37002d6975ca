#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -m pytest tests/test_gpu_filter.py tests/test_gpu_virtual.py -q -x -p no:cacheprovider 2>&1 | tail -3
for v in narrow wide; do
  if [ $v = wide ]; then export CHASE_NO_NARROW=1; fi
  TAG=$v python tools/hemm_timing.py 60000 2500 4 real
  TAG=$v python tools/hemm_timing.py 60000 2500 ramp real
  TAG=$v python tools/hemm_timing.py 60000 1300 4
  TAG=$v python tools/hemm_timing.py 30000 3000 4
done
