"""Small filter + CholeskyQR runs (complex and real, ragged degrees, odd sizes, padded ld) for
compute-sanitizer (memcheck / racecheck / synccheck, one tool per run)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import chase_inputs as ci
import paper_2309_15595_b200 as cb

for complex_ in (True, False):
    for N, degs in ((61, [2, 2, 4, 4, 6, 8, 8, 10, 12, 20]), (200, [4] * 3 + [10] * 40 + [20] * 27)):
        n = len(degs)
        lam = ci.uniform_spectrum(N)
        A = ci.dense_from_spectrum(lam, 3, complex_)
        V0 = ci.gaussian_block(N, n, 4, complex_)
        b = ci.bounds_from_spectrum(lam, n)
        ld = N + (N % 2) + 2
        Ab = np.zeros((N, ld), dtype=A.dtype); Ab[:, :N] = A.T
        Vb = np.zeros((n, ld), dtype=A.dtype); Vb[:, :N] = V0.T
        Ad = torch.from_numpy(Ab).cuda().T[:N]
        Vd = torch.from_numpy(Vb).cuda().T[:N]
        h = cb.Chase(cb.CHASE_C128 if complex_ else cb.CHASE_R64, N, n)
        h.filter(Ad, Vd, degs, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))
        est = cb.chase_cond_est(lam, b.c, b.e, degs, 0)
        r = h.cholqr(Vd, est)
        torch.cuda.synchronize()
        Q = Vd.T.cpu().numpy().T
        print(complex_, N, r, np.linalg.norm(Q.conj().T @ Q - np.eye(n)))
        h.close()
print("sanitize run ok")
