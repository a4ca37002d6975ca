python tools/tail_diag.py 8000 1300 4 2 1 40
python tools/tail_diag.py 20000 1300 6 2 1 74
python tools/tail_diag.py 20000 1300 4 2 1 74 real
timeout 900 python -m pytest tests/test_gpu_virtual.py -x -q > gpurun_out/virt_push.log 2>&1; echo rc=$? >> gpurun_out/virt_push.log
