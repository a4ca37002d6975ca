#!/bin/bash
# A/B: real HEMM variants at a C5-recipe shape; ncu of the default real kernel
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for v in default bn64; do
  if [ $v = default ]; then L=""; else L="CHASE_LIB=$PWD/abt/libchase_$v.so"; fi
  env $L TAG=$v python tools/hemm_timing.py 60000 2500 4 real
  env $L TAG=$v python tools/hemm_timing.py 60000 1200 4 real
  env $L TAG=$v python tools/hemm_timing.py 60000 300 4 real
done
TAG=cplx python tools/hemm_timing.py 30000 3000 4
ncu --set full --clock-control none --import-source on -k regex:dgemm_kernel -c 2 -o gpurun_out/ncu_dgemm_r60k --force-overwrite python tools/profile_hemm.py 60000 2500 real > gpurun_out/ncu_dgemm.log 2>&1
echo ncu_rc=$?
