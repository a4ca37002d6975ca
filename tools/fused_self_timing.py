"""Diagnostic: the fused persistent HEMM kernel on one GPU (CHASE_FUSED_SELF=1, single-member
'communicator'), vs the standard kernel.  Usage: CHASE_FUSED_SELF=1 python tools/fused_self_timing.py N n"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import chase_inputs as ci
import paper_2309_15595_b200 as cb

N = int(sys.argv[1]); n = int(sys.argv[2])
lam = ci.uniform_spectrum(N)
A = ci.dft_phase(lam, 2).block(0, N, 0, N, device="cuda").T
V = torch.from_numpy(np.ascontiguousarray(ci.gaussian_block(N, n, 1002, True).T)).cuda().T
b = ci.bounds_from_spectrum(lam, n)
h = cb.Chase(cb.CHASE_C128, N, n)
if os.environ.get("CHASE_FUSED_SELF"):
    nb = cb.chase_fused_workspace_size(h.h)
    buf = torch.zeros(nb + 256, dtype=torch.uint8, device="cuda")
    base = (buf.data_ptr() + 255) // 256 * 256
    cb.chase_set_fused_workspace(h.h, base, [base])
for rep in range(2):
    cb.chase_profile_enable(h.h, True)
    cb.chase_profile_read(h.h)
    h.filter(A, V, [2] * n, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))
    ms, ln = cb.chase_profile_read(h.h)
fl = 8.0 * N * N * n
print(f"{'fused-self' if os.environ.get('CHASE_FUSED_SELF') else 'standard'} N={N} n={n}: odd {ms['hemm_odd']:.1f} ms {fl/ms['hemm_odd']/1e9:.2f} TF | even {ms['hemm_even']:.1f} ms {fl/ms['hemm_even']/1e9:.2f} TF", flush=True)
