# filter HEMM TF/s vs ragged remainder width (real 128-wide tiles; remainder in 32-wide tiles)
for k in 2048 2080 2112 2144 2176 2063 2100; do python tools/hemm_timing.py 60000 $k 6 real; done
for k in 2048 2080 2112; do python tools/hemm_timing.py 40000 $k 4; done
