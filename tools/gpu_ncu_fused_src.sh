# source-level stall sampling of the even-step real fused kernel (m = 1) vs the plain kernel
mkdir -p /tmp/ncu gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"dgemm_kernel" -s 1 -c 1 -o /tmp/ncu/plain python tools/hemm_timing.py 18944 1024 4 real > /dev/null 2>&1
FUSED_SELF=1 ncu --set full --clock-control none --import-source on -k regex:"dgemm_fused_kernel" -s 1 -c 1 -o /tmp/ncu/fused python tools/hemm_timing.py 18944 1024 4 real > /dev/null 2>&1
for r in plain fused; do
  ncu -i /tmp/ncu/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_src_${r}.csv 2>&1
  ncu -i /tmp/ncu/$r.ncu-rep --page details --csv > gpurun_out/ncu_det_${r}.csv 2>&1
done
ls -la gpurun_out/ncu_src_* gpurun_out/ncu_det_*
