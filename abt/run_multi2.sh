#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi nvlink -gt d -i 0 > gpurun_out/nvlink_probe.txt 2>&1
python - >> gpurun_out/nvlink_probe.txt 2>&1 <<'PY'
import pynvml as nv
nv.nvmlInit(); h=nv.nvmlDeviceGetHandleByIndex(0)
for fid in (nv.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES, nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX):
    for scope in (0, 0xFFFFFFFF):
        try:
            v=nv.nvmlDeviceGetFieldValues(h,[(fid,scope)])
            print(fid, scope, v[0].nvmlReturn, v[0].value.ullVal)
        except Exception as e: print(fid, scope, 'exc', e)
PY
timeout 1500 python -m pytest tests/test_gpu_multi.py -k "not full_size" -q -p no:cacheprovider > gpurun_out/multi2_tests.log 2>&1; echo rc=$? >> gpurun_out/multi2_tests.log
timeout 1200 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench2b.log 2>&1; echo rc=$? >> gpurun_out/bench2b.log
