#!/bin/bash
cd "$GRAFT_REPO_ROOT"
python -m pytest tests/test_gpu_qr.py tests/test_gpu_filter.py tests/test_gpu_virtual.py -q -x -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do
  TAG=old python abt/oldpkg/hemm_timing_old.py 30000 3000 20
  TAG=new python tools/hemm_timing.py 30000 3000 20
done
python tools/qr_timing.py 30000 3000
