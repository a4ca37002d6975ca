"""Pins of oracle.residuals (Alg.2 l.24-28) by closed forms."""
import math

import numpy as np

import chase_inputs as ci
import oracle


def test_diagonal_closed_form():
    """A = diag(lam), v = e_i, theta: residual = |lam_i - theta| exactly."""
    lam = np.array([-1.5, 0.25, 2.0, 7.0])
    A = np.diag(lam)
    V = np.eye(4)[:, [0, 2, 3]]
    theta = [0.5, 2.0, -1.0]
    r = oracle.residuals(A, V, theta)
    assert np.array_equal(r, [2.0, 0.0, 8.0])


def test_two_eigenvector_mixture_closed_form():
    """v = cos(p) u1 + sin(p) u2 of a Hermitian A: ||A v - t v||^2 = cos^2 (l1-t)^2 + sin^2 (l2-t)^2."""
    N = 40
    lam = ci.uniform_spectrum(N, -1.0, 3.0)
    Q = ci.haar_unitary(N, 5, True)
    A = (Q * lam) @ Q.conj().T
    ph = 0.37
    v = math.cos(ph) * Q[:, 3] + math.sin(ph) * Q[:, 17]
    t = 0.8
    r = oracle.residuals(A, v[:, None], [t])[0]
    ref = math.sqrt(math.cos(ph) ** 2 * (lam[3] - t) ** 2 + math.sin(ph) ** 2 * (lam[17] - t) ** 2)
    assert abs(r - ref) <= 1e-13


def test_exact_eigenpairs_have_tiny_residual():
    N = 64
    lam = ci.clement_spectrum(N)
    Q = ci.haar_unitary(N, 7, True)
    A = (Q * lam) @ Q.conj().T
    r = oracle.residuals(A, Q[:, :10], lam[:10])
    assert np.all(r <= 1e-12 * np.max(np.abs(lam)))
