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


def _owned(N, P, k, nb):
    """Global indices of grid row/column k: block distribution (nb == 0, remainder rule S:102) or
    block-cyclic with block nb."""
    if nb == 0:
        size, start = _part(N, P, k)
        return np.arange(start, start + size)
    g = np.arange(N)
    return g[(g // nb) % P == k]


def step_partial(A, X, Y_old, i, j, p, q, odd, alpha, beta, c, use_beta, nb=0):
    """The summand rank (i, j) contributes to the AllReduce of one filter step:
        odd:  alpha (A_ij^H X - c band_ij(X)) + [use_beta] beta Y_old     (X = C_i, Y = B_j)
        even: alpha (A_ij X  - c band_ij(X)) + [use_beta] beta Y_old      (X = B_j, Y = C_i)
    band_ij(X) = the rows of X whose global index is both a row of grid row i and a column of
    grid column j (reading #6), placed on the output rows of the same global index."""
    N = A.shape[0]
    ri, cj = _owned(N, p, i, nb), _owned(N, q, j, nb)
    Aij = A[np.ix_(ri, cj)]
    if odd:
        part = Aij.conj().T @ X
        # diagonal share: B rows (global cj) that are also local C rows (global ri)
        _, o_out, o_in = np.intersect1d(cj, ri, return_indices=True)
    else:
        part = Aij @ X
        _, o_out, o_in = np.intersect1d(ri, cj, return_indices=True)
    part[o_out] -= c * X[o_in]
    part = alpha * part
    if use_beta:
        part = part + beta * Y_old
    return part


def distributed_filter(A, V0, degrees, c, e, mu_1, p, q, nb=0):
    """nb > 0: block-cyclic distribution; the diagonal share of rank (i, j) is then the set of
    global indices owned both as a row (grid row i) and as a column (grid column j)."""
    d = _check_degrees(degrees)
    N, n = V0.shape
    D = max(d)
    alpha, beta, _ = chebyshev_scalars(c, e, mu_1, D)
    R = [_owned(N, p, i, nb) for i in range(p)]
    Cc = [_owned(N, q, j, nb) for j in range(q)]
    dtype = np.result_type(A.dtype, V0.dtype)
    C = [np.array(V0[ri], dtype=dtype) for ri in R]                      # C_i (per grid row)
    B = [np.zeros((len(cj), n), dtype=dtype) for cj in Cc]              # B_j (per grid column)
    for s in range(1, D + 1):
        k = sum(1 for dj in d if dj >= s)
        off = n - k
        if s % 2 == 1:
            for j, cj in enumerate(Cc):
                acc = None
                for i in range(p):
                    part = step_partial(A, C[i][:, off:], B[j][:, off:], i, j, p, q, True,
                                        alpha[s - 1], beta[s - 1], c, i == 0 and s > 1, nb)
                    acc = part if acc is None else acc + part
                B[j][:, off:] = acc
        else:
            for i, ri in enumerate(R):
                acc = None
                for j in range(q):
                    part = step_partial(A, B[j][:, off:], C[i][:, off:], i, j, p, q, False,
                                        alpha[s - 1], beta[s - 1], c, j == 0, nb)
                    acc = part if acc is None else acc + part
                C[i][:, off:] = acc
    out = np.empty((N, n), dtype=dtype)
    for i, ri in enumerate(R):
        out[ri] = C[i]
    return out
