"""Oracle: Chebyshev polynomial filter (Eq.(1); Alg.1 l.4, P:95;
Alg.2 l.12) with the scaled-recurrence scalars of SPEC S:362 (reading #1 in DESIGN.md).

    sigma_1 = e / (mu_1 - c)
    V_1     = (sigma_1 / e) (A - c I) V_0                       (first step, beta = 0)
    sigma_{s} = 1 / (2/sigma_1 - sigma_{s-1})                   (s >= 2)
    V_{s}   = 2 (sigma_s / e) (A - c I) V_{s-1} - sigma_{s-1} sigma_s V_{s-2}

i.e. Eq.(1) with gamma_i = c, alpha = 2 sigma_{i+1}/e, beta = -sigma_i sigma_{i+1}.
Column j stops after exactly d_j steps (reading #3): its output is V_{d_j}[:, j].
Degrees must be even ("ChASE enforces even-degree Chebyshev polynomials") and sorted
non-decreasing (Alg.1 l.12), so the active set is a contiguous suffix of columns.
"""
from __future__ import annotations

import numpy as np


def chebyshev_scalars(c: float, e: float, mu_1: float, D: int):
    """Return (alpha[1..D], beta[1..D], sigma[1..D]) as Python lists indexed 0..D-1 for steps 1..D.

    Step s computes V_s = alpha_s (A - cI) V_{s-1} + beta_s V_{s-2}  (Eq.(1)).
    """
    sigma_1 = e / (mu_1 - c)
    sig = [sigma_1]
    alpha = [sigma_1 / e]
    beta = [0.0]
    for s in range(2, D + 1):
        sigma_prev = sig[-1]
        sigma_s = 1.0 / (2.0 / sigma_1 - sigma_prev)
        sig.append(sigma_s)
        alpha.append(2.0 * sigma_s / e)
        beta.append(-sigma_prev * sigma_s)
    return alpha, beta, sig


def _check_degrees(degrees):
    d = [int(x) for x in degrees]
    for j, dj in enumerate(d):
        if dj < 2 or dj % 2 != 0:
            raise ValueError(f"degree {dj} of column {j} must be even and >= 2 (P:149)")
        if j > 0 and dj < d[j - 1]:
            raise ValueError("degrees must be sorted non-decreasing (Alg.1 l.12, P:103)")
    return d


def filter_schedule(degrees):
    """Per step s = 1..D: (k_s, off_s, comm_s) with k_s = #{j : d_j >= s}, off_s = n - k_s,
    comm_s = 'col' for odd s (H C -> B, AllReduce over ccomm) and 'row' for even s
    (H^H B -> C, AllReduce over rcomm)."""
    d = _check_degrees(degrees)
    n = len(d)
    D = max(d)
    steps = []
    for s in range(1, D + 1):
        k = sum(1 for dj in d if dj >= s)
        steps.append((k, n - k, "col" if s % 2 == 1 else "row"))
    return steps


def filter_record(degrees, n_r: int, n_c: int):
    """Bookkeeping record of one filter call on a rank owning an n_r x n_c block of A:
    per step (k_s, off_s, comm_s, message elements) where an odd step all-reduces the
    n_c x k_s block B and an even step the n_r x k_s block C (Alg.2); plus
    matvecs = sum_j d_j."""
    steps = filter_schedule(degrees)
    rec = []
    for s, (k, off, comm) in enumerate(steps, start=1):
        elems = (n_c if comm == "col" else n_r) * k
        rec.append((k, off, comm, elems))
    return rec, int(sum(int(x) for x in degrees))


def chebyshev_filter(A: np.ndarray, V0: np.ndarray, degrees, c: float, e: float, mu_1: float):
    """Apply p_{d_j}(A) to every column v_j of V0 by the three-term recurrence (Eq.(1)).

    A: N x N Hermitian (complex128) or symmetric (float64).  V0: N x n.  Returns (V, record)
    where V[:, j] = V_{d_j}[:, j] and record = filter_schedule(degrees) plus matvecs.
    The HEMM step A @ W uses numpy's matmul (a library primitive, as allowed); the shift,
    scaling and axpby follow the formula term by term.
    """
    d = _check_degrees(degrees)
    N, n = V0.shape
    if len(d) != n:
        raise ValueError("len(degrees) != number of columns")
    if not (e > 0):
        raise ValueError("e must be positive (S:332)")
    D = max(d)
    alpha, beta, _ = chebyshev_scalars(c, e, mu_1, D)
    dtype = np.result_type(A.dtype, V0.dtype)
    out = np.array(V0, dtype=dtype, copy=True)
    W_prev = np.array(V0, dtype=dtype, copy=True)     # V_{s-2}
    W = np.array(V0, dtype=dtype, copy=True)          # V_{s-1}
    for s in range(1, D + 1):
        act = [j for j in range(n) if d[j] >= s]      # contiguous suffix (sorted degrees)
        Wa = W[:, act]
        AW = A @ Wa                                   # HEMM
        new = alpha[s - 1] * (AW - c * Wa)
        if s > 1:
            new = new + beta[s - 1] * W_prev[:, act]
        W_next = W.copy()
        W_next[:, act] = new
        W_prev, W = W, W_next
        for j in act:
            if d[j] == s:
                out[:, j] = W[:, j]
    return out, filter_schedule(d)
