"""Time the filter HEMM kernels alone: chase_filter with uniform degree D on an N x n problem,
per-orientation device time from the library's profile events.
Usage: python tools/hemm_timing.py N n [D] [real]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import chase_inputs as ci
import paper_2309_15595_b200 as cb

N = int(sys.argv[1]); n = int(sys.argv[2]); D = int(sys.argv[3]) if len(sys.argv) > 3 else 4
real = len(sys.argv) > 4 and sys.argv[4] == "real"
lam = ci.uniform_spectrum(N)
gen = ci.hartley_sign(lam, 2) if real else ci.dft_phase(lam, 2)
A = gen.block(0, N, 0, N, device="cuda").T
V = torch.from_numpy(np.ascontiguousarray(ci.gaussian_block(N, n, 1002, not real).T)).cuda().T
b = ci.bounds_from_spectrum(lam, n)
h = cb.Chase(cb.CHASE_R64 if real else cb.CHASE_C128, N, n)
h.filter(A, V, [D] * n, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))
torch.cuda.synchronize()
cb.chase_profile_enable(h.h, True)
cb.chase_profile_read(h.h)
h.filter(A, V, [D] * n, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))
ms, ln = cb.chase_profile_read(h.h)
fl = (2.0 if real else 8.0) * N * N * n
tag = os.environ.get("TAG", "")
print(f"{tag} N={N} n={n} {'real' if real else 'complex'}: odd(A^H) {ms['hemm_odd']/ln['hemm_odd']:.2f} ms "
      f"{fl/(ms['hemm_odd']/ln['hemm_odd'])/1e9:.2f} TF | even(A) {ms['hemm_even']/ln['hemm_even']:.2f} ms "
      f"{fl/(ms['hemm_even']/ln['hemm_even'])/1e9:.2f} TF", flush=True)
