"""Time chase_cholqr (CholeskyQR2) and chase_hhqr on an N x n Gaussian block; per-category
device time.  Usage: python tools/qr_timing.py N n [real] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import chase_inputs as ci
import paper_2309_15595_b200 as cb

N = int(sys.argv[1]); n = int(sys.argv[2]); real = len(sys.argv) > 3 and sys.argv[3] == "real"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
X0 = torch.from_numpy(np.ascontiguousarray(ci.gaussian_block(N, n, 7, not real).T)).cuda()
h = cb.Chase(cb.CHASE_R64 if real else cb.CHASE_C128, N, n)
for rep in range(reps):
    X = X0.clone()
    cb.chase_profile_enable(h.h, True)
    cb.chase_profile_read(h.h)
    r = h.cholqr(X.T, 1e3)
    ms, ln = cb.chase_profile_read(h.h)
print(f"N={N} n={n} {'real' if real else 'complex'} variant {r['variant']} passes {r['passes']}: "
      f"gram {ms['gram']:.2f} ms potrf {ms['potrf']:.2f} ms trsm {ms['trsm']:.2f} ms; launches {ln}", flush=True)
for rep in range(reps):
    X = X0.clone()
    cb.chase_profile_enable(h.h, True)
    cb.chase_profile_read(h.h)
    h.hhqr(X.T)
    ms, ln = cb.chase_profile_read(h.h)
print(f"hhqr {ms['hhqr']:.2f} ms, {ln['hhqr']} launches", flush=True)
