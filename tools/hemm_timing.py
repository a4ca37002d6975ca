"""Time the filter HEMM kernels alone: one chase_filter call (after a warm-up call) with uniform
degree D (or the C5 ramp 10..36) on an N x n problem; device time per odd / even step from the
library's profile events, TFLOP/s from the algorithmic flops of those steps.
Usage: python tools/hemm_timing.py N n [D|ramp] [real]
FUSED_SELF=1: the 1x1 handle runs every step through the fused kernel (chase_set_fused_mode 1,
optional FUSED_BUDGET CTAs) -- the fused protocol's own cost without NVLink."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import chase_inputs as ci
import paper_2309_15595_b200 as cb

N = int(sys.argv[1]); n = int(sys.argv[2])
darg = sys.argv[3] if len(sys.argv) > 3 else "4"
real = len(sys.argv) > 4 and sys.argv[4] == "real"
degs = ci.ramp_degrees(n) if darg == "ramp" else ci.uniform_degrees(n, int(darg))
D = int(degs.max())
lam = ci.uniform_spectrum(N)
gen = ci.hartley_sign(lam, 2) if real else ci.dft_phase(lam, 2)
A = gen.block(0, N, 0, N, device="cuda").T
V = torch.from_numpy(np.ascontiguousarray(ci.gaussian_block(N, n, 1002, not real).T)).cuda().T
b = ci.bounds_from_spectrum(lam, n)
h = cb.Chase(cb.CHASE_R64 if real else cb.CHASE_C128, N, n)
if os.environ.get("FUSED_SELF"):
    region = torch.empty(cb.chase_fused_workspace_size(h.h), dtype=torch.uint8, device="cuda")
    cb.chase_set_fused_workspace(h.h, region.data_ptr(), [region.data_ptr()])
    cb.chase_set_fused_mode(h.h, 1, int(os.environ.get("FUSED_BUDGET", "0")))
h.filter(A, V, degs, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))
torch.cuda.synchronize()
cb.chase_profile_enable(h.h, True)
cb.chase_profile_read(h.h)
h.filter(A, V, degs, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))
ms, ln = cb.chase_profile_read(h.h)
per = (2.0 if real else 8.0) * N * N
f_odd = per * sum(int((degs >= s).sum()) for s in range(1, D + 1, 2))
f_even = per * sum(int((degs >= s).sum()) for s in range(2, D + 1, 2))
tag = os.environ.get("TAG", "")
print(f"{tag} N={N} n={n} D={darg} {'real' if real else 'complex'}: "
      f"odd(A^H) {ms['hemm_odd']:.1f} ms {f_odd / ms['hemm_odd'] / 1e9:.2f} TF | "
      f"even(A) {ms['hemm_even']:.1f} ms {f_even / ms['hemm_even'] / 1e9:.2f} TF | "
      f"all {(f_odd + f_even) / (ms['hemm_odd'] + ms['hemm_even']) / 1e9:.2f} TF ({ln['hemm']} launches)", flush=True)
