"""GPU parity of chase_rayleigh_ritz (Alg.2 l.16-22; own parallel block-Jacobi HEEVD) against
oracle.rayleigh_ritz: Ritz values to 1e-12 ||A||, Ritz vectors up to phase where the Ritz value
is separated, orthonormality, and the eigensolver alone (C = I: Ritz values = eigenvalues)."""
import numpy as np
import pytest

import chase_inputs as ci
import oracle
import paper_2309_15595_b200 as cb
from gpu_util import dev, host

pytestmark = pytest.mark.gpu


def gpu_rr(A, C, complex_):
    import torch
    N, n = C.shape
    h = cb.Chase(cb.CHASE_C128 if complex_ else cb.CHASE_R64, N, n)
    Ad, Cd = dev(A), dev(C)
    theta, sweeps = h.rayleigh_ritz(Ad, Cd)
    torch.cuda.synchronize()
    X = host(Cd)
    h.close()
    return theta, X, sweeps


def check(A, C, theta, X, tol_vec=1e-9):
    ref, Xr = oracle.rayleigh_ritz(A, C)
    scale = np.max(np.abs(ref)) + 1e-300
    assert np.max(np.abs(theta - ref)) <= 1e-12 * scale
    n = C.shape[1]
    assert np.linalg.norm(X.conj().T @ X - np.eye(n)) <= 1e-11
    gaps = np.full(n, np.inf)
    if n > 1:
        d = np.diff(ref)
        gaps[:-1] = np.minimum(gaps[:-1], d)
        gaps[1:] = np.minimum(gaps[1:], d)
    for j in range(n):
        if gaps[j] > 1e-3 * scale:
            ph = np.vdot(Xr[:, j], X[:, j])
            ph = ph / abs(ph)
            assert np.linalg.norm(X[:, j] - ph * Xr[:, j]) <= tol_vec


@pytest.mark.parametrize("complex_", [True, False])
@pytest.mark.parametrize("N,n", [(64, 1), (64, 7), (200, 60), (300, 64), (301, 65), (400, 129)])
def test_rr_random_subspace(complex_, N, n):
    lam = ci.uniform_spectrum(N, -2.0, 3.0)
    A = ci.dense_from_spectrum(lam, N + n, complex_)
    C, _ = np.linalg.qr(ci.gaussian_block(N, n, N + 1, complex_))
    theta, X, sweeps = gpu_rr(A, np.asfortranarray(C), complex_)
    assert sweeps >= 1
    check(A, C, theta, X)


@pytest.mark.parametrize("complex_", [True, False])
@pytest.mark.parametrize("n", [33, 96, 250])
def test_eigensolver_full_space(complex_, n):
    """C = I: the Ritz values are the eigenvalues of A (Clement spectrum, exactly known)."""
    lam = ci.clement_spectrum(n)
    A = ci.dense_from_spectrum(lam, 7 * n, complex_)
    C = np.eye(n, dtype=np.complex128 if complex_ else np.float64)
    theta, X, _ = gpu_rr(A, C, complex_)
    assert np.max(np.abs(theta - np.sort(lam))) <= 1e-12 * np.max(np.abs(lam))
    assert np.linalg.norm(A @ X - X * theta) <= 1e-11 * np.max(np.abs(lam)) * np.sqrt(n)


def test_rr_after_filter_and_qr_c1():
    """The ChASE sequence Filter -> CholeskyQR2 -> Rayleigh-Ritz on config C1: the Ritz values
    approach the lowest eigenvalues and match the oracle pipeline."""
    import torch
    N, n = 512, 60
    lam = ci.uniform_spectrum(N)
    A = ci.dense_from_spectrum(lam, 1, True)
    V0 = ci.gaussian_block(N, n, 101, True)
    b = ci.bounds_from_spectrum(lam, n)
    degs = [20] * n
    h = cb.Chase(cb.CHASE_C128, N, n)
    Ad, Vd = dev(A), dev(V0)
    h.filter(Ad, Vd, degs, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))
    est = cb.chase_cond_est(lam, b.c, b.e, degs, 0)
    h.cholqr(Vd, est)
    Q = host(Vd)
    theta, sweeps = h.rayleigh_ritz(Ad, Vd)
    X = host(Vd)
    resid = h.residuals(Ad, Vd, theta)
    torch.cuda.synchronize()
    h.close()
    check(A, Q, theta, X)
    ref_res = oracle.residuals(A, X, theta)
    assert np.max(np.abs(resid - ref_res)) <= 1e-10 * np.max(ref_res)
    assert np.all(theta[:20] - lam[:20] < 1e-6)      # the filter pushed the lowest 20 eigenpairs in
