"""Time chase_rayleigh_ritz on an N x n orthonormal block (random subspace of a Uniform matrix).
Usage: python tools/rr_timing.py N n"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import chase_inputs as ci
import paper_2309_15595_b200 as cb

N = int(sys.argv[1]); n = int(sys.argv[2])
lam = ci.uniform_spectrum(N)
A = ci.dft_phase(lam, 2).block(0, N, 0, N, device="cuda").T
X = torch.from_numpy(np.ascontiguousarray(ci.gaussian_block(N, n, 5, True).T)).cuda().T
h = cb.Chase(cb.CHASE_C128, N, n)
h.cholqr(X, 1e3)
V = X.clone()
torch.cuda.synchronize()
t0 = time.perf_counter()
theta, sw = h.rayleigh_ritz(A, V)
torch.cuda.synchronize()
t = time.perf_counter() - t0
print(f"inner={os.environ.get('CHASE_JAC_INNER', 15)} N={N} n={n}: RR {t*1e3:.1f} ms, {sw} sweeps, ritz[0]={theta[0]:.6e}", flush=True)
