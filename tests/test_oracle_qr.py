"""Pins of the oracle CholeskyQR family (oracle/qr.py): SPEC hand cases (tests/golden),
library special cases (LAPACK Cholesky / triangular solve / Householder QR), QR invariants,
the Alg.4 dispatch and the Alg.5 estimate.  CPU only."""
import math

import numpy as np
import pytest
import scipy.linalg as sla

import chase_inputs as ci
import oracle
from oracle import qr as oqr


def rows(x):
    return np.array(x, dtype=np.float64)


def test_gram_hand(golden):
    g = golden["herk_gram"]
    assert np.array_equal(oracle.gram(rows(g["X_rows"])), rows(g["G"]))


def test_potrf_hand(golden):
    g = golden["potrf_diag"]
    R, info = oracle.potrf_upper(rows(g["G"]))
    assert info == g["info"] and np.array_equal(R, rows(g["R"]))
    g = golden["potrf_indefinite"]
    _, info = oracle.potrf_upper(rows(g["G"]))
    assert info == g["info"]


def test_trsm_hand(golden):
    g = golden["trsm_right"]
    assert np.array_equal(oracle.trsm_right_upper(rows(g["X_rows"]), rows(g["R"])), rows(g["Y_rows"]))


def test_cholqr_hand(golden):
    g = golden["cholesky_qr_hand"]
    Q, info, passes = oracle.cholesky_qr(rows(g["X_rows"]), 1)
    assert info == 0 and passes == 1 and np.array_equal(Q, rows(g["Q_rows"]))


@pytest.mark.parametrize("complex_", [True, False])
def test_potrf_matches_lapack(complex_):
    X = ci.svd_synthesized(80, 30, 1e3, 3, complex_)
    G = X.conj().T @ X
    R, info = oracle.potrf_upper(G)
    assert info == 0
    L = np.linalg.cholesky(G)                       # LAPACK: G = L L^H, L = R^H
    assert np.allclose(R, L.conj().T, rtol=0, atol=1e-12 * np.abs(R).max())
    assert np.all(np.tril(R, -1) == 0)
    assert np.all(np.real(np.diag(R)) > 0) and np.all(np.imag(np.diag(R)) == 0)


@pytest.mark.parametrize("complex_", [True, False])
def test_trsm_matches_lapack(complex_):
    rng = np.random.default_rng(4)
    n = 25
    R = np.triu(rng.standard_normal((n, n))) + 4 * np.eye(n)
    X = rng.standard_normal((60, n))
    if complex_:
        R = R + 1j * np.triu(rng.standard_normal((n, n)), 1)
        X = X + 1j * rng.standard_normal((60, n))
    Y = oracle.trsm_right_upper(X, R)
    ref = sla.solve_triangular(R.T, X.T, lower=True).T    # Y R = X  <=>  R^T Y^T = X^T
    assert np.allclose(Y, ref, rtol=0, atol=1e-13 * np.abs(ref).max())


@pytest.mark.parametrize("complex_", [True, False])
@pytest.mark.parametrize("zero_col", [None, 4, 0, 19])
def test_householder_matches_lapack(complex_, zero_col):
    """householder_factor is xGEQR2 + xUNG2R: the same reflectors as LAPACK xGEQRF + xUNGQR
    (numpy.linalg.qr), so Q and diag(R) agree to rounding even for a rank-deficient X (an exact
    zero column), where Q is not determined by X alone."""
    X = ci.svd_synthesized(70, 20, 1e4, 5, complex_)
    if zero_col is not None:
        X[:, zero_col] = 0
    Qf, beta = oracle.householder_factor(X)
    Ql, Rl = np.linalg.qr(X)
    assert np.abs(Qf - Ql).max() <= 10 * 1e4 * 2.0 ** -53     # kappa u (different blocking)
    assert np.abs(beta - np.diag(Rl).real).max() <= 1e-12 * np.abs(X).max()
    assert np.abs(np.diag(Rl).imag).max() == 0.0
    Q = oracle.householder_qr(X)
    assert np.linalg.norm(Q.conj().T @ Q - np.eye(20)) <= 1e-13
    R = Q.conj().T @ X                                     # upper, non-negative real diagonal
    assert np.abs(np.tril(R, -1)).max() <= 1e-13 * np.abs(X).max()
    assert (np.diag(R).real >= -1e-13).all() and np.abs(np.diag(R).imag).max() <= 1e-13
    if zero_col is None:
        ph = np.diag(Rl) / np.abs(np.diag(Rl))
        assert np.allclose(Q, Ql * ph[None, :], rtol=0, atol=1e-12)


def test_larfg_definition():
    """H^H (alpha; x) = (beta; 0) with H = I - tau v v^H, v = (1; v'), beta real; |beta| = norm."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal(9) + 1j * rng.standard_normal(9)
    tau, beta, v = oracle.larfg(x[0], x[1:])
    vf = np.concatenate([[1.0], v])
    H = np.eye(9) - tau * np.outer(vf, vf.conj())
    y = H.conj().T @ x
    assert abs(y[0] - beta) <= 1e-14 * np.linalg.norm(x) and np.abs(y[1:]).max() <= 1e-14 * 4
    assert abs(abs(beta) - np.linalg.norm(x)) <= 1e-14 * np.linalg.norm(x)
    assert np.abs(H.conj().T @ H - np.eye(9)).max() <= 1e-14      # unitary
    assert oracle.larfg(2.5, np.zeros(3))[0] == 0.0                 # H = I


def test_shift_golden(golden):
    g = golden["shift"]
    s = oracle.shift_value(g["m"], g["n"], g["norm"])
    assert s == g["s_over_u"] * 2.0 ** -53          # 1.3555823e-12, exact


def test_frobenius_sq_complex_golden(golden):
    """Alg.4 l.5 on complex entries: |3+4i|^2 + |1-2i|^2 = 30 (a real-part-only or
    unsquared norm gives 10 / 7.24)."""
    g = golden["frobenius_sq_complex"]
    X = rows(g["X_re"]) + 1j * rows(g["X_im"])
    assert oracle.frobenius_sq(X) == g["norm"]
    assert oracle.frobenius_sq(rows(g["X_re"])) == 10.0          # real X: 9 + 1


def test_shift_complex_golden(golden):
    """The shift the shifted pass adds for the complex golden X: s = 3300 u (Alg.4 l.5-6)."""
    g, f = golden["shift_complex"], golden["frobenius_sq_complex"]
    X = rows(f["X_re"]) + 1j * rows(f["X_im"])
    s = oracle.shift_value(X.shape[0], X.shape[1], oracle.frobenius_sq(X))
    assert (g["m"], g["n"], g["norm"]) == (X.shape[0], X.shape[1], f["norm"])
    assert s == g["s_over_u"] * 2.0 ** -53


def test_cond_est_golden(golden):
    g = golden["cond_est_t3"]
    c, e = 0.0, 1.0
    ritz = [g["t"], g["t"]]
    est = oracle.cond_est(ritz, c, e, [g["d"], g["d"]], 0)
    ref = g["cond_a"] + g["cond_b_sqrt2"] * math.sqrt(2.0)
    assert abs(est - ref) <= 4e-15 * ref
    g = golden["cond_est_inside"]
    assert oracle.cond_est([g["tp"], g["t"]], 0.0, 1.0, [2, g["d"]], 1) == g["cond"]


def test_cond_est_degree_split():
    """d = degs[locked+1], d_M = max(degs[locked+1:]): cond = rho^d rho'^(d_M - d)."""
    c, e = 0.0, 1.0
    tp, t = -2.0, -1.5
    rp, r = 2.0 + math.sqrt(3.0), 1.5 + math.sqrt(1.25)
    est = oracle.cond_est([tp, -1.8, t, 0.0], c, e, [4, 4, 6, 10], 2)
    assert abs(est - r ** 6 * rp ** 4) <= 1e-13 * est


def test_dispatch_golden(golden):
    X = ci.svd_synthesized(60, 8, 10.0, 7, True)
    for est, variant, passes in golden["dispatch"]["cases"]:
        assert oracle.select_variant(est) == variant
        res = oracle.caqr(X, est)
        assert res["variant"] == variant and res["passes"] == passes and res["status"] == 0
    assert oracle.select_variant(math.nextafter(1e8, 2e8)) == oqr.SHIFTED
    with pytest.raises(ValueError):
        oracle.caqr(X, 0.5)


@pytest.mark.parametrize("kappa,variant,tol", [(1e3, 2, 1e-13), (1e6, 2, 1e-13), (1e12, 3, 1e-13), (1e14, 3, 1e-12)])
def test_orthogonality_ladder(kappa, variant, tol):
    """CholeskyQR2 <= 1e-12 for kappa <= 1e6; shifted <= 1e-11 for kappa <= 1e14."""
    X = ci.svd_synthesized(400, 40, kappa, 8, True)
    res = oracle.caqr(X, kappa if variant == 3 else 1e3)
    assert res["status"] == 0 and res["variant"] == variant
    Q = res["Q"]
    assert np.linalg.norm(Q.conj().T @ Q - np.eye(40)) <= tol * math.sqrt(40)
    # same column space and triangular relation: Q^H X upper with positive real diagonal
    Rx = Q.conj().T @ X
    assert np.linalg.norm(np.tril(Rx, -1)) <= 1e-10 * kappa * 1e-3 * np.linalg.norm(X) + 1e-12
    assert np.all(np.real(np.diag(Rx)) > 0)


def test_cholqr1_loses_orthogonality_like_kappa_squared():
    X = ci.svd_synthesized(300, 20, 1e4, 9, True)
    Q, info, _ = oracle.cholesky_qr(X, 1)
    orth = np.linalg.norm(Q.conj().T @ Q - np.eye(20))
    assert info == 0 and 1e-10 < orth < 1e-4          # ~ u kappa^2 = 1e-8


def test_cholqr2_equals_householder_within_kappa_u():
    kappa = 1e5
    X = ci.svd_synthesized(300, 30, kappa, 10, True)
    Q, info, _ = oracle.cholesky_qr(X, 2)
    Qh = oracle.householder_qr(X)
    assert info == 0
    assert np.linalg.norm(Q - Qh) / math.sqrt(30) <= 10 * kappa * 2.0 ** -53


def _filtered_c1(degree, N=512, n=60):
    lam = ci.uniform_spectrum(N)
    A = ci.dense_from_spectrum(lam, 1, True)
    V0 = ci.gaussian_block(N, n, 101, True)
    b = ci.bounds_from_spectrum(lam, n)
    X, _ = oracle.chebyshev_filter(A, V0, [degree] * n, b.c, b.e, b.mu_1)
    return X, lam, b


@pytest.mark.parametrize("degree,variant", [(2, 1), (20, 2), (36, 3)])
def test_variant_ladder_on_filtered_blocks(degree, variant):
    """C1 filtered blocks: Alg.5 on the exact spectrum selects CQR1 / CQR2 / shifted, the
    estimate bounds kappa from above, and the result is orthonormal."""
    X, lam, b = _filtered_c1(degree)
    est = oracle.cond_est(lam, b.c, b.e, [degree] * 60, 0)
    assert oracle.select_variant(est) == variant
    kappa = np.linalg.cond(X)
    assert est >= kappa
    res = oracle.caqr(X, est)
    assert res["status"] == 0 and res["variant"] == variant
    orth = np.linalg.norm(res["Q"].conj().T @ res["Q"] - np.eye(60))
    assert orth <= (1e-13 if variant > 1 else 1e-12)


def test_degree36_plain_cqr2_fails_and_escalates():
    X, lam, b = _filtered_c1(36)
    _, info, passes = oracle.cholesky_qr(X, 2)
    assert info > 0 and passes == 0
    res = oracle.caqr(X, 1e3)                   # force CQR2: first POTRF fails -> shifted
    assert res["status"] == 0 and res["variant"] == oqr.SHIFTED and res["passes"] == 3


def test_hhqr_fallback_paths():
    """Alg.4 l.8-9 and reading #33.  (a) X = 0: norm = 0 so s = 0 and the shifted
    POTRF fails at pivot 1 -> HHQR, whose reflectors are all identities: Q = [I; 0].
    (b) an exact zero column j: CQR2's first POTRF fails at j+1 (escalation, reading #14), the
    shifted pass succeeds and keeps column j exactly zero, the next POTRF fails at j+1 -> HHQR
    on that output: orthonormal Q spanning X, Q^H X upper triangular."""
    Z = np.zeros((40, 6), dtype=np.complex128)
    res = oracle.caqr(Z, 1e9)
    assert (res["status"], res["variant"], res["passes"], res["info"]) == (0, oqr.HOUSEHOLDER, 0, 1)
    assert np.array_equal(res["Q"], np.eye(40, 6))
    X = ci.svd_synthesized(300, 10, 10.0, 3, True)
    X[:, 4] = 0
    for est in (1e3, 1e9):
        res = oracle.caqr(X, est)
        assert (res["status"], res["variant"], res["passes"], res["info"]) == (0, oqr.HOUSEHOLDER, 1, 5)
        Q = res["Q"]
        assert np.linalg.norm(Q.conj().T @ Q - np.eye(10)) <= 1e-13
        R = Q.conj().T @ X
        assert np.abs(np.tril(R, -1)).max() <= 1e-13 * np.abs(X).max()
        assert np.linalg.norm(Q @ R - X) <= 1e-13 * np.linalg.norm(X)


def test_hhqr_row_permutation_invariance():
    """Reading #33(c): the GPU HHQR takes rows in the "virtual" order of the column communicator
    (rank 0's local rows, then rank 1's ...), a row permutation P of the block-cyclic global
    order.  With diag(R) >= 0 the thin Q of P X is P Q (X full rank), so the order does not change
    the result beyond rounding."""
    X = ci.svd_synthesized(90, 12, 1e3, 21, True)
    perm = np.concatenate([np.arange(k, 90, 3) for k in range(3)])      # cyclic-style dealing
    Q = oracle.householder_qr(X)
    Qp = oracle.householder_qr(X[perm])
    assert np.abs(Qp - Q[perm]).max() <= 100 * 1e3 * 2.0 ** -53
