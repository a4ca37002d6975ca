# ncu --set full of one fused-self real HEMM launch (even step, dgemm_fused_kernel<false>)
mkdir -p /tmp/ncu gpurun_out
FUSED_SELF=1 ncu --set full --clock-control none --import-source on -k regex:dgemm_fused_kernel -s 1 -c 1 \
  -o /tmp/ncu/fself python tools/hemm_timing.py 30000 1500 4 real > gpurun_out/ncu_fself.log 2>&1
ncu -i /tmp/ncu/fself.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_fself_source.csv 2>&1
ncu -i /tmp/ncu/fself.ncu-rep --page raw --csv > gpurun_out/ncu_fself_raw.csv 2>&1
ncu -i /tmp/ncu/fself.ncu-rep --page details --csv > gpurun_out/ncu_fself_details.csv 2>&1
ls -la gpurun_out/ncu_fself*
