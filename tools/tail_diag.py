"""Diagnostic: the fused filter with its split-K wave tail (fused_tail.cuh) on a virtual p x q grid
(all ranks on this GPU) against the 1x1 plain filter on the same inputs; prints the largest
column error and, if any, the wrong (row-tile, column) blocks of rank 0.
Usage: python tools/tail_diag.py N n degree p q budget [real]"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch

import chase_inputs as ci
import paper_2309_15595_b200 as cb

N, n, D, p, q, budget = (int(x) for x in sys.argv[1:7])
real = len(sys.argv) > 7 and sys.argv[7] == "real"
lam = ci.uniform_spectrum(N)
gen = ci.hartley_sign(lam, 2) if real else ci.dft_phase(lam, 2)
A = gen.block(0, N, 0, N, device="cuda").T
V0 = torch.from_numpy(np.ascontiguousarray(ci.gaussian_block(N, n, 1002, not real).T)).cuda().T
b = ci.bounds_from_spectrum(lam, n)
degs = [D] * n
dt = cb.CHASE_R64 if real else cb.CHASE_C128
h1 = cb.Chase(dt, N, n)
Vr = V0.clone()
h1.filter(A, Vr, degs, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))
torch.cuda.synchronize()
ref = Vr.cpu().numpy()
h1.close()

world = p * q
hs = [cb.Chase(dt, N, n, p, q, r // q, r % q, None, 0, torch.cuda.Stream(), virtual=True) for r in range(world)]
size = cb.chase_fused_workspace_size(hs[0].h)
regions = [torch.empty(size, dtype=torch.uint8, device="cuda") for _ in hs]
ptrs = [t.data_ptr() for t in regions]
for h, t in zip(hs, regions):
    cb.chase_set_fused_workspace(h.h, t.data_ptr(), ptrs)
    cb.chase_set_fused_mode(h.h, 0, budget)
def colmajor(x):
    return x.T.contiguous().T


rows = [torch.as_tensor(h.rows, device="cuda") for h in hs]
cols = [torch.as_tensor(h.cols, device="cuda") for h in hs]
A_loc = [colmajor(A[rr][:, cc]) for rr, cc in zip(rows, cols)]
V_loc = [colmajor(V0[rr]) for rr in rows]
torch.cuda.synchronize()
errs = [None] * world


def work(r):
    try:
        hs[r].filter(A_loc[r], V_loc[r], degs, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))
        hs[r].stream.synchronize()
    except Exception as exc:
        errs[r] = exc


th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
for t in th:
    t.start()
for t in th:
    t.join(300)
print("errors:", errs)
worst = 0.0
for r, h in enumerate(hs):
    V = V_loc[r].cpu().numpy()
    R = ref[h.rows]
    col = np.linalg.norm(V - R, axis=0) / np.linalg.norm(R, axis=0)
    worst = max(worst, float(col.max()))
    if r == 0 and col.max() > 1e-10:
        bad = np.abs(V - R) > 1e-8 * np.abs(R).max()
        rt, cc = np.nonzero(bad)
        blocks = sorted(set(zip((rt // 128).tolist(), cc.tolist())))
        print("rank 0 bad blocks (row-tile, col):", blocks[:40], "... total", len(blocks))
print(f"N={N} n={n} D={D} grid={p}x{q} budget={budget} {'real' if real else 'complex'}: worst col err {worst:.3e}")
