"""Pins of oracle.rayleigh_ritz (Alg.2 l.16-21): invariant subspaces give exact eigenpairs,
Cauchy interlacing, the one-column Rayleigh quotient, orthonormal Ritz vectors spanning C."""
import numpy as np

import chase_inputs as ci
import oracle


def test_invariant_subspace_gives_exact_eigenpairs():
    N, n = 80, 9
    lam = ci.uniform_spectrum(N, -1.0, 2.0)
    Q = ci.haar_unitary(N, 3, True)
    A = (Q * lam) @ Q.conj().T
    cols = [2, 5, 7, 11, 20, 33, 40, 61, 79]
    # a rotated basis of the invariant subspace
    M = ci.haar_unitary(n, 4, True)
    C = Q[:, cols] @ M
    theta, X = oracle.rayleigh_ritz(A, C)
    assert np.allclose(theta, lam[cols], atol=1e-13)
    for j, c in enumerate(cols):
        assert abs(abs(np.vdot(Q[:, c], X[:, j])) - 1.0) <= 1e-12


def test_cauchy_interlacing_and_orthonormal_ritz_vectors():
    N, n = 120, 15
    lam = ci.clement_spectrum(N)
    A = ci.dense_from_spectrum(lam, 5, True)
    C, _ = np.linalg.qr(ci.gaussian_block(N, n, 6, True))
    theta, X = oracle.rayleigh_ritz(A, C)
    lam = np.sort(lam)
    assert np.all(theta >= lam[:n] - 1e-10) and np.all(theta <= lam[N - n:] + 1e-10)
    assert np.linalg.norm(X.conj().T @ X - np.eye(n)) <= 1e-12
    P = C @ C.conj().T
    assert np.linalg.norm(P @ X - X) <= 1e-12


def test_one_column_rayleigh_quotient():
    N = 40
    A = ci.dense_from_spectrum(ci.uniform_spectrum(N), 8, True)
    v = ci.gaussian_block(N, 1, 9, True)
    v = v / np.linalg.norm(v)
    theta, X = oracle.rayleigh_ritz(A, v)
    assert abs(theta[0] - np.real(np.vdot(v[:, 0], A @ v[:, 0]))) <= 1e-14
