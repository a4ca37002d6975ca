"""Oracle: the 2D block-distributed filter scheme of PAPER.md §3.1 (Alg.2 l.12),
simulated in one address space over a p x q grid.  Used to pin the distributed readings the
CUDA path implements (#6, #7), not to produce expected values for it.

Rank (i, j) owns A_ij = A[r0_i:r0_i+n_r, c0_j:c0_j+n_c], C_i = rows r0_i.. of the C-layout
block (replicated over the row communicator) and B_j = rows c0_j.. of the B-layout block
(replicated over the column communicator).

  odd step s  ("performs HC and stores the result in B"):
      partial_ij = alpha_s (A_ij^H C_i - c * band_ij(C_i)) + [i == 0] beta_s B_j
      B_j = sum_i partial_ij                            (AllReduce SUM over ccomm)
  even step s ("executes H^H B and writes the result to C"):
      partial_ij = alpha_s (A_ij B_j - c * band_ij(B_j)) + [j == 0] beta_s C_i
      C_i = sum_j partial_ij                            (AllReduce SUM over rcomm)

band_ij(X) keeps only the rows whose global index lies in [r0_i, r0_i+n_r) and
[c0_j, c0_j+n_c) -- the part of -cI that rank (i, j) owns -- so the shift is applied exactly
once per global row.  Reductions sum in ascending rank order.
"""
from __future__ import annotations

import numpy as np

from .filter import chebyshev_scalars, _check_degrees


def _part(N, P, k):
    b, rem = divmod(N, P)
    return b + (1 if k < rem else 0), k * b + min(k, rem)


def distributed_filter(A, V0, degrees, c, e, mu_1, p, q):
    d = _check_degrees(degrees)
    N, n = V0.shape
    D = max(d)
    alpha, beta, _ = chebyshev_scalars(c, e, mu_1, D)
    rows = [_part(N, p, i) for i in range(p)]     # (n_r, r0)
    cols = [_part(N, q, j) for j in range(q)]     # (n_c, c0)
    dtype = np.result_type(A.dtype, V0.dtype)
    C = [np.array(V0[r0:r0 + nr], dtype=dtype) for (nr, r0) in rows]     # C_i (per grid row)
    B = [np.zeros((nc, n), dtype=dtype) for (nc, c0) in cols]           # B_j (per grid column)
    for s in range(1, D + 1):
        k = sum(1 for dj in d if dj >= s)
        off = n - k
        if s % 2 == 1:
            for j, (nc, c0) in enumerate(cols):
                acc = None
                for i, (nr, r0) in enumerate(rows):
                    Aij = A[r0:r0 + nr, c0:c0 + nc]
                    Ci = C[i][:, off:]
                    part = Aij.conj().T @ Ci
                    lo, hi = max(r0, c0), min(r0 + nr, c0 + nc)
                    if lo < hi:
                        part[lo - c0:hi - c0] -= c * Ci[lo - r0:hi - r0]
                    part = alpha[s - 1] * part
                    if i == 0 and s > 1:
                        part = part + beta[s - 1] * B[j][:, off:]
                    acc = part if acc is None else acc + part
                B[j][:, off:] = acc
        else:
            for i, (nr, r0) in enumerate(rows):
                acc = None
                for j, (nc, c0) in enumerate(cols):
                    Aij = A[r0:r0 + nr, c0:c0 + nc]
                    Bj = B[j][:, off:]
                    part = Aij @ Bj
                    lo, hi = max(r0, c0), min(r0 + nr, c0 + nc)
                    if lo < hi:
                        part[lo - r0:hi - r0] -= c * Bj[lo - c0:hi - c0]
                    part = alpha[s - 1] * part
                    if j == 0:
                        part = part + beta[s - 1] * C[i][:, off:]
                    acc = part if acc is None else acc + part
                C[i][:, off:] = acc
    return np.concatenate(C, axis=0)
