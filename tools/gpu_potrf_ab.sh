timeout 900 python -m pytest tests/test_gpu_qr.py tests/test_gpu_solve.py -x -q 2>&1 | tail -3
for o in 64 256 512; do echo "outer $o"; CHASE_POTRF_OUTER=$o python tools/qr_timing.py 30000 3000 2>&1 | head -1; done
for o in 64 256 512; do echo "outer $o real"; CHASE_POTRF_OUTER=$o python tools/qr_timing.py 60000 2500 real 2>&1 | head -1; done
