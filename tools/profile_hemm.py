"""Small driver for ncu: one chase_filter call with degree 2 on every column (one ConjTrans and
one NoTrans HEMM launch) at a chosen size.  Usage: python tools/profile_hemm.py [N] [n] [real]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import chase_inputs as ci
import paper_2309_15595_b200 as cb

N = int(sys.argv[1]) if len(sys.argv) > 1 else 30000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
real = len(sys.argv) > 3 and sys.argv[3] == "real"
lam = ci.uniform_spectrum(N)
gen = ci.hartley_sign(lam, 2) if real else ci.dft_phase(lam, 2)
A = gen.block(0, N, 0, N, device="cuda").T
V = torch.from_numpy(np.ascontiguousarray(ci.gaussian_block(N, n, 1002, not real).T)).cuda().T
b = ci.bounds_from_spectrum(lam, n)
h = cb.Chase(cb.CHASE_R64 if real else cb.CHASE_C128, N, n)
h.filter(A, V, [2] * n, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))
torch.cuda.synchronize()
print("ok")
