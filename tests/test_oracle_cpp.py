"""Pins of the triple-loop C++ oracle (oracle/cpp/chase_oracle.cpp via oracle/cpp_oracle.py):
the same closed forms, golden hand cases, LAPACK special cases and QR invariants that pin the
numpy oracle -- each would fail on a dropped term, a wrong sign/index or a transposed operand.
CPU only."""
import math

import numpy as np
import pytest
import scipy.linalg as sla

import chase_inputs as ci
import oracle
from cheb_closed_form import apply_spectral, gain
from oracle import cpp_oracle as co

U = 2.0 ** -53


def relF(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def rows(x):
    return np.array(x, dtype=np.float64)


# ------------------------------------------------------------------------------------ filter
def test_one_by_one_degree_two():
    """1x1 A = [lam], degree 2: (2t^2 - 1) / (2 t1^2 - 1) written out."""
    lam, c, e, mu1 = 0.3, 0.6, 0.35, -0.1
    out = co.filter(np.array([[lam]]), np.array([[1.0]]), [2], c, e, mu1)
    t, t1 = (lam - c) / e, (mu1 - c) / e
    assert abs(out[0, 0] - (2 * t * t - 1) / (2 * t1 * t1 - 1)) <= 1e-15


@pytest.mark.parametrize("d", [2, 4, 8, 20, 36])
def test_diagonal_matrix_closed_form(d):
    """A = diag(lam): e_i scales by T_d(t_i) / T_d(t_1) (cos/cosh closed form)."""
    rng = np.random.default_rng(7)
    lam = np.sort(rng.uniform(-0.2, 1.0, 40))
    c, e, mu1 = 0.6, 0.4, lam[0]
    out = co.filter(np.diag(lam), np.eye(40)[:, :12], [d] * 12, c, e, mu1)
    ref = np.diag(gain(d, lam, c, e, mu1))[:, :12]
    assert relF(out, ref) <= 1e-13


@pytest.mark.parametrize("complex_", [True, False])
def test_haar_spectral_closed_form(complex_):
    """A = Q diag(lam) Q^H: column j = Q g_{d_j}(Lam) Q^H v_j, ragged degrees 2..36."""
    N, n = 96, 10
    lam = ci.uniform_spectrum(N)
    Q = ci.haar_unitary(N, 11, complex_)
    A = ci.dense_from_spectrum(lam, 11, complex_)
    V = ci.gaussian_block(N, n, 12, complex_)
    b = ci.bounds_from_spectrum(lam, n)
    degs = [2, 2, 4, 6, 8, 8, 12, 20, 30, 36]
    out = co.filter(A, V, degs, b.c, b.e, b.mu_1)
    ref = apply_spectral(Q, lam, V, degs, b.c, b.e, b.mu_1)
    for j in range(n):
        assert relF(out[:, j], ref[:, j]) <= 1e-12, j


def test_bruteforce_eigh_small():
    """N = 64 Clement spectrum: evaluation through numpy.linalg.eigh of the generated A."""
    N, n = 64, 6
    lam = ci.clement_spectrum(N)
    A = ci.dense_from_spectrum(lam, 5, True)
    V = ci.gaussian_block(N, n, 6, True)
    b = ci.bounds_from_spectrum(lam, n)
    w, Z = np.linalg.eigh(A)
    for d in (2, 10, 20):
        out = co.filter(A, V, [d] * n, b.c, b.e, b.mu_1)
        ref = Z @ (gain(d, w, b.c, b.e, b.mu_1)[:, None] * (Z.conj().T @ V))
        assert relF(out, ref) <= 1e-12


def test_matches_numpy_oracle():
    """Consistency with the numpy oracle on a C1-shaped problem (both pinned independently)."""
    N, n = 200, 17
    lam = ci.uniform_spectrum(N)
    A = ci.dense_from_spectrum(lam, 3, True)
    V = ci.gaussian_block(N, n, 4, True)
    b = ci.bounds_from_spectrum(lam, n)
    degs = [2, 2, 4, 4, 4, 6, 8, 8, 10, 10, 12, 12, 12, 14, 16, 18, 20]
    ref, _ = oracle.chebyshev_filter(A, V, degs, b.c, b.e, b.mu_1)
    out = co.filter(A, V, degs, b.c, b.e, b.mu_1)
    assert np.max(np.linalg.norm(out - ref, axis=0) / np.linalg.norm(ref, axis=0)) <= 1e-13


@pytest.mark.parametrize("bad", [[2, 3], [0, 2], [4, 2]])
def test_rejects_bad_degrees(bad):
    with pytest.raises(ValueError):
        co.filter(np.eye(2), np.ones((2, len(bad))), bad, 0.5, 0.5, -1.0)


# ------------------------------------------------------------------------------------ QR family
def test_gram_potrf_trsm_hand(golden):
    g = golden["herk_gram"]
    assert np.array_equal(co.gram(rows(g["X_rows"])), rows(g["G"]))
    g = golden["potrf_diag"]
    R, info = co.potrf(rows(g["G"]))
    assert info == g["info"] and np.array_equal(R, rows(g["R"]))
    assert co.potrf(rows(golden["potrf_indefinite"]["G"]))[1] == golden["potrf_indefinite"]["info"]
    g = golden["trsm_right"]
    assert np.array_equal(co.trsm(rows(g["X_rows"]), rows(g["R"])), rows(g["Y_rows"]))
    g = golden["cholesky_qr_hand"]
    r = co.caqr(rows(g["X_rows"]), 5.0)
    assert (r["variant"], r["passes"], r["info"]) == (1, 1, 0)
    assert np.array_equal(r["Q"], rows(g["Q_rows"]))


def test_shift_complex_golden(golden):
    """Alg.4 l.5-6 on X = [[3+4i, 0], [0, 1-2i]]: ||X||_F^2 = 30, s = 3300 u."""
    f = golden["frobenius_sq_complex"]
    X = rows(f["X_re"]) + 1j * rows(f["X_im"])
    assert co.shift(X) == golden["shift_complex"]["s_over_u"] * U
    g = golden["shift"]                                   # s(100, 10, ||X||^2 = 1) = 12210 u
    X = np.zeros((g["m"], g["n"]))
    X[0, 0] = 1.0
    assert co.shift(X) == g["s_over_u"] * U


@pytest.mark.parametrize("complex_", [True, False])
def test_potrf_trsm_match_lapack(complex_):
    X = ci.svd_synthesized(80, 30, 1e3, 3, complex_)
    G = X.conj().T @ X
    R, info = co.potrf(G)
    assert info == 0
    L = np.linalg.cholesky(G)                             # LAPACK: G = L L^H, R = L^H
    assert np.allclose(R, L.conj().T, rtol=0, atol=1e-12 * np.abs(R).max())
    Y = co.trsm(X, R)
    ref = sla.solve_triangular(R.T, X.T, lower=True, trans=0).T if not complex_ else \
        sla.solve_triangular(R, X.T, trans="T", lower=False).T
    assert relF(Y, ref) <= 1e-12
    assert relF(co.gram(X), G) <= 1e-14


@pytest.mark.parametrize("complex_", [True, False])
@pytest.mark.parametrize("degree,variant,passes", [(2, 1, 1), (20, 2, 2), (36, 3, 3)])
def test_variant_ladder_c1(complex_, degree, variant, passes):
    """Alg.4 on filtered C1 blocks: estimate -> CholeskyQR / CQR2 / shifted CQR2;
    Q orthonormal (CQR2, shifted) and spanning X; equal to the numpy oracle's Q within kappa u."""
    N, n = 512, 60
    lam = ci.uniform_spectrum(N)
    A = ci.dense_from_spectrum(lam, 1, complex_)
    V0 = ci.gaussian_block(N, n, 101, complex_)
    b = ci.bounds_from_spectrum(lam, n)
    X = co.filter(A, V0, [degree] * n, b.c, b.e, b.mu_1)
    est = oracle.cond_est(lam, b.c, b.e, [degree] * n, 0)
    r = co.caqr(X, est)
    assert (r["variant"], r["passes"], r["info"]) == (variant, passes, 0)
    Q = r["Q"]
    if variant >= 2:
        assert np.linalg.norm(Q.conj().T @ Q - np.eye(n)) <= 1e-12
    kappa = np.linalg.cond(X)
    ref = oracle.caqr(X, est)
    assert np.linalg.norm(Q - ref["Q"]) / math.sqrt(n) <= 100 * kappa * U + 1e-13
    if variant == 3:
        s_ref = oracle.shift_value(N, n, oracle.frobenius_sq(X))   # same sum, other order
        assert abs(r["shift"] - s_ref) <= 1e-13 * s_ref


def test_escalation_and_fallback_signal():
    """Reading #14: a failing first POTRF of CQR2 escalates to the shifted path; an exactly zero
    column makes a later Gram singular -> info > 0, variant 4 (the HHQR hand-off, reading #33)."""
    N, n = 512, 60
    lam = ci.uniform_spectrum(N)
    A = ci.dense_from_spectrum(lam, 1, True)
    V0 = ci.gaussian_block(N, n, 101, True)
    b = ci.bounds_from_spectrum(lam, n)
    X = co.filter(A, V0, [36] * n, b.c, b.e, b.mu_1)
    r = co.caqr(X, 1e3)
    ref = oracle.caqr(X, 1e3)
    assert (r["variant"], r["passes"]) == (ref["variant"], ref["passes"]) == (3, 3)
    Z = ci.svd_synthesized(300, 10, 10.0, 3, True)
    Z[:, 4] = 0
    r = co.caqr(Z, 1e9)
    ref = oracle.caqr(Z, 1e9)
    assert r["variant"] == ref["variant"] == 4 and r["info"] == ref["info"] and r["passes"] == ref["passes"]
