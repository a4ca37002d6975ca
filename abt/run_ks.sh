#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for v in default ks2 ks2n16; do
  if [ $v = default ]; then L=""; else L="CHASE_LIB=$PWD/abt/libchase_$v.so"; fi
  env $L TAG=$v python tools/hemm_timing.py 60000 2500 4 real
  env $L TAG=$v python tools/hemm_timing.py 60000 2500 ramp real
  env $L TAG=$v python tools/hemm_timing.py 30000 2432 2 real
done
CHASE_LIB=$PWD/abt/libchase_ks2.so python -m pytest tests/test_gpu_filter.py tests/test_gpu_virtual.py tests/test_gpu_qr.py tests/test_gpu_hhqr.py -q -x -p no:cacheprovider 2>&1 | tail -3
