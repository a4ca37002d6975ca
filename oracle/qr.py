"""Oracle: communication-avoiding CholeskyQR family of PAPER.md §3.2.

  gram              Alg.3 l.3  "R <- SYRK(X)"          G = X^H X
  potrf_upper       Alg.3 l.5  "[R, info] <- POTRF(R)" G = R^H R, R upper
  trsm_right_upper  Alg.3 l.6  "X <- TRSM(X, R)"       X <- X R^{-1}
  cholesky_qr       Alg.3      repeated cholDegree times
  shift_value       Alg.4 l.6  s = 11 (m n + n (n + 1)) u norm
  caqr              Alg.4      condition-driven dispatch
  cond_est          Alg.5      condition estimate of the filtered block
  householder_qr    Alg.4 l.9 "X <- ScaLAPACK-HHQR(X, comm)": LAPACK-
                    convention Householder QR (xGEQR2 + xUNG2R, reflectors of xLARFG), Q
                    normalised so diag(R) is positive real (reading #33); also a CholeskyQR pin

Readings: u = 2^-53 (#10); m = global row count, n = columns QR'd (#11);
norm = squared Frobenius norm of X (#12); shifted path = 1 shifted pass + CholeskyQR2 (#13);
threshold ties est == 20 / est == 1e8 -> CholeskyQR2 (#9); a POTRF failure in the first pass
of CholeskyQR1/2 (X still untouched) escalates to the shifted path, any other failure is
reported as CHASE_ECHOL with the pivot (#14/#15).
"""
from __future__ import annotations

import cmath
import math

import numpy as np

U_ROUNDOFF = 2.0 ** -53          # unit round-off of IEEE double (reading #10)

CHOL1, CHOL2, SHIFTED, HOUSEHOLDER = 1, 2, 3, 4  # include/chase.h chase_qr_variant_t
OK, ECHOL = 0, 4


def gram(X: np.ndarray) -> np.ndarray:
    """G[a, b] = sum_r conj(X[r, a]) X[r, b]   (SYRK/HERK, Alg.3 l.3)."""
    return X.conj().T @ X


def frobenius_sq(X: np.ndarray) -> float:
    """||X||_F^2 = sum |x_rb|^2  (Alg.4 l.5 before the AllReduce)."""
    return float(np.sum(np.abs(X) ** 2))


def potrf_upper(G: np.ndarray):
    """Upper Cholesky G = R^H R (POTRF).  Returns (R, info); info = 0 on success, else the
    1-based index j of the first pivot whose radicand G[j,j] - sum_{k<j} |R[k,j]|^2 is not
    positive (or NaN), LAPACK convention."""
    n = G.shape[0]
    R = np.zeros_like(G)
    for j in range(n):
        rad = np.real(G[j, j]) - np.sum(np.abs(R[:j, j]) ** 2)
        if not (rad > 0.0):
            return R, j + 1
        rjj = math.sqrt(rad)
        R[j, j] = rjj
        if j + 1 < n:
            R[j, j + 1:] = (G[j, j + 1:] - R[:j, j].conj() @ R[:j, j + 1:]) / rjj
    return R, 0


def trsm_right_upper(X: np.ndarray, R: np.ndarray) -> np.ndarray:
    """Y = X R^{-1} for upper-triangular R, column by column:
    Y[:, l] = (X[:, l] - sum_{k<l} Y[:, k] R[k, l]) / R[l, l]."""
    n = R.shape[0]
    Y = np.zeros_like(X)
    for l in range(n):
        acc = X[:, l] - Y[:, :l] @ R[:l, l]
        Y[:, l] = acc / R[l, l]
    return Y


def shift_value(m: int, n: int, norm: float) -> float:
    """s = 11 (m n + n (n + 1)) u norm   (Alg.4 l.6)."""
    return 11.0 * float(m * n + n * (n + 1)) * U_ROUNDOFF * norm


def cholesky_qr(X: np.ndarray, chol_degree: int):
    """Alg.3: repeat chol_degree times {G = X^H X; R = POTRF(G); X = X R^{-1}}.
    Returns (Q, info, passes_done)."""
    for i in range(chol_degree):
        G = gram(X)
        R, info = potrf_upper(G)
        if info != 0:
            return X, info, i
        X = trsm_right_upper(X, R)
    return X, 0, chol_degree


def select_variant(est: float) -> int:
    """Alg.4 branch: est > 1e8 -> shifted CholeskyQR2; est < 20 -> CholeskyQR; else CholeskyQR2."""
    if est > 1e8:
        return SHIFTED
    if est < 20.0:
        return CHOL1
    return CHOL2


def _shifted(X: np.ndarray, m_global: int):
    """Alg.4 l.3-12: one shifted pass then CholeskyQR2; a failing shifted POTRF reverts to
    HHQR (l.8-9).  Returns (Q, info, passes, hhqr_used)."""
    n = X.shape[1]
    G = gram(X)
    norm = frobenius_sq(X)
    s = shift_value(m_global, n, norm)
    R, info = potrf_upper(G + s * np.eye(n, dtype=G.dtype))
    if info != 0:
        return householder_qr(X), info, 0, True          # Alg.4 l.9
    X = trsm_right_upper(X, R)
    Q, info2, p = cholesky_qr(X, 2)
    if info2 != 0:                  # reading #33: HHQR on the last successful pass output
        return householder_qr(Q), info2, 1 + p, True
    return Q, 0, 1 + p, False


def caqr(X: np.ndarray, est: float):
    """Alg.4 (1D-CAQR for ChASE) on the global N x n block X.

    Returns dict(Q, status, variant, passes, info): variant is the branch actually executed
    (escalation per reading #14; HOUSEHOLDER when the HHQR fallback ran, reading #33), passes
    the number of successful Cholesky passes, info the 1-based pivot of the last failed POTRF
    (0 if none failed)."""
    if not (est >= 1.0):
        raise ValueError("cond_est must be >= 1 (S:397)")
    m = X.shape[0]
    v = select_variant(est)
    if v != SHIFTED:
        deg = 1 if v == CHOL1 else 2
        Q, info, passes = cholesky_qr(X, deg)
        if info == 0:
            return dict(Q=Q, status=OK, variant=v, passes=passes, info=0)
        if passes > 0:              # reading #33: later failure -> HHQR on the current X
            return dict(Q=householder_qr(Q), status=OK, variant=HOUSEHOLDER, passes=passes,
                        info=info)
        # first POTRF failed, X untouched: escalate (reading #14)
    Q, info, passes, hh = _shifted(X, m)
    return dict(Q=Q, status=OK, variant=HOUSEHOLDER if hh else SHIFTED, passes=passes, info=info)


def cond_est(ritz, c: float, e: float, degs, locked: int) -> float:
    """Alg.5, literally, with the complex square root of t^2 - 1:
        t' = (Lambda[1] - c)/e,  t = (Lambda[locked+1] - c)/e
        |rho|  = max(|t  - sqrt(t^2 - 1)|,  |t  + sqrt(t^2 - 1)|)
        |rho'| = max(|t' - sqrt(t'^2 - 1)|, |t' + sqrt(t'^2 - 1)|)
        d = degs[locked+1], d_M = max(degs[locked+1:])
        cond = |rho|^d |rho'|^(d_M - d)
    (1-based indices of the paper mapped to 0-based: Lambda[1] -> ritz[0]).
    """
    tp = (ritz[0] - c) / e
    t = (ritz[locked] - c) / e

    def rho(x):
        r = cmath.sqrt(complex(x * x - 1.0, 0.0))
        return max(abs(x - r), abs(x + r))

    d = int(degs[locked])
    dM = int(max(int(v) for v in degs[locked:]))
    return rho(t) ** d * rho(tp) ** (dM - d)


def larfg(alpha, x: np.ndarray):
    """The elementary reflector of LAPACK xLARFG, which ScaLAPACK's HHQR applies:
        H^H (alpha; x) = (beta; 0),  H = I - tau v v^H,  v = (1; x / (alpha - beta)),
        beta = -sign(Re alpha) ||(alpha; x)||_2  (real),  tau = (beta - alpha) / beta;
    H = I (tau = 0, beta = alpha) when x = 0 and alpha is real.  Returns (tau, beta, v[1:])."""
    xnorm2 = float(np.vdot(x, x).real)
    a = complex(alpha)
    if xnorm2 == 0.0 and a.imag == 0.0:
        return 0.0, a.real, x.copy()
    beta = -math.copysign(math.sqrt(abs(a) ** 2 + xnorm2), a.real)
    tau = (beta - alpha) / beta
    return tau, beta, x / (alpha - beta)


def householder_factor(X: np.ndarray):
    """Unblocked Householder QR, LAPACK xGEQR2 then xUNG2R, column by column:
        k = 0..n-1: (tau_k, beta_k, v_k) = larfg(A[k, k], A[k+1:, k]);
                    A[k:, k+1:] <- H_k^H A[k:, k+1:]
        Q = H_0 H_1 ... H_{n-1} [I_n; 0]   (applied right to left).
    Returns (Q, beta): R = Q^H X is upper triangular with diagonal beta (real)."""
    A = np.array(X, dtype=np.result_type(X.dtype, np.float64), copy=True)
    m, n = A.shape
    taus, betas, vs = [], [], []
    for k in range(n):
        tau, beta, v = larfg(A[k, k], A[k + 1:, k])
        vf = np.concatenate([np.ones(1, dtype=A.dtype), v])
        A[k, k] = beta
        A[k + 1:, k] = v
        if k + 1 < n:
            w = vf.conj() @ A[k:, k + 1:]
            A[k:, k + 1:] -= np.conj(tau) * np.outer(vf, w)
        taus.append(tau)
        betas.append(beta)
        vs.append(vf)
    Q = np.zeros((m, n), dtype=A.dtype)
    Q[np.arange(n), np.arange(n)] = 1.0
    for k in reversed(range(n)):
        vf = vs[k]
        Q[k:, :] -= taus[k] * np.outer(vf, vf.conj() @ Q[k:, :])
    return Q, np.array(betas)


def householder_qr(X: np.ndarray) -> np.ndarray:
    """Alg.4 l.9 "X <- ScaLAPACK-HHQR(X, comm)": the thin Q of householder_factor with
    column k scaled by sign(beta_k) (+1 for beta_k = 0), so diag(R) is non-negative real and Q
    equals CholeskyQR's Q for full-rank X (reading #33).  Also a CholeskyQR pin."""
    Q, beta = householder_factor(X)
    sgn = np.where(beta < 0.0, -1.0, 1.0)
    return Q * sgn[None, :]
