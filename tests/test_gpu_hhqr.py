"""GPU parity of the Householder QR fallback (Alg.4 l.8-9; chase_hhqr, hhqr.cuh)
against the oracle (oracle.householder_qr: LAPACK xGEQR2/xUNG2R reflectors, diag(R) >= 0):
Q within C * kappa * u and orthonormal to 1e-12 on multi-panel ragged shapes; the same Q for a
rank-deficient X (same reflector convention); the caqr fallback paths (variant, passes, info)
equal to the oracle's; the HHQR mode of chase_cholqr."""
import math

import numpy as np
import pytest

import chase_inputs as ci
import oracle
import paper_2309_15595_b200 as cb
from gpu_util import dev, host

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


def orth(Q):
    return np.linalg.norm(Q.conj().T @ Q - np.eye(Q.shape[1]))


def gpu_hhqr(X, complex_=True):
    import torch
    N, n = X.shape
    h = cb.Chase(cb.CHASE_C128 if complex_ else cb.CHASE_R64, N, n)
    Xd = dev(X)
    h.hhqr(Xd)
    torch.cuda.synchronize()
    Q = host(Xd)
    h.close()
    return Q


@pytest.mark.parametrize("complex_", [True, False])
@pytest.mark.parametrize("m,n,kappa", [(300, 1, 1.0), (300, 31, 1e2), (700, 100, 1e3), (1000, 33, 1e6),
                                       (2000, 250, 1e4), (513, 64, 1e8), (65, 65, 1e3)])
def test_hhqr_matches_oracle(complex_, m, n, kappa):
    X = ci.svd_synthesized(m, n, kappa, int(3 * m + n), complex_)
    Q = gpu_hhqr(X, complex_)
    ref = oracle.householder_qr(X)
    assert orth(Q) <= 1e-12 * max(1.0, math.sqrt(n / 60))
    assert np.linalg.norm(Q - ref) / math.sqrt(n) <= 100 * kappa * U + 1e-13
    R = Q.conj().T @ X
    assert np.abs(np.tril(R, -1)).max() <= 1e-12 * np.abs(X).max() * max(1.0, kappa * U * 1e4)
    assert np.abs(np.diag(R).imag).max() <= 1e-12 and (np.diag(R).real > 0).all()


@pytest.mark.parametrize("complex_", [True, False])
def test_hhqr_rank_deficient(complex_):
    """exact zero columns (one inside a panel, one at a panel start): H_j = I there, and the
    completion columns follow from the same reflectors as the oracle's."""
    X = ci.svd_synthesized(400, 70, 10.0, 7, complex_)
    X[:, 5] = 0
    X[:, 32] = 0
    Q = gpu_hhqr(X, complex_)
    ref = oracle.householder_qr(X)
    assert orth(Q) <= 1e-12
    assert np.linalg.norm(Q - ref) / math.sqrt(70) <= 1e-12
    R = Q.conj().T @ X
    assert np.abs(np.tril(R, -1)).max() <= 1e-13 * np.abs(X).max()


def test_hhqr_zero_matrix():
    Q = gpu_hhqr(np.zeros((90, 40), dtype=np.complex128))
    assert np.array_equal(Q, np.eye(90, 40))


@pytest.mark.parametrize("complex_", [True, False])
@pytest.mark.parametrize("est", [1e3, 1e9])
def test_cholqr_falls_back_to_hhqr(complex_, est):
    """zero column: CQR2's first POTRF fails (escalation, reading #14) / the shifted path runs,
    the shifted pass keeps the column zero, the next POTRF fails -> HHQR (reading #33)."""
    import torch
    X = ci.svd_synthesized(300, 10, 10.0, 3, complex_)
    X[:, 4] = 0
    ref = oracle.caqr(X, est)
    h = cb.Chase(cb.CHASE_C128 if complex_ else cb.CHASE_R64, 300, 10)
    Xd = dev(X)
    res = h.cholqr(Xd, est, raise_on_error=False)
    torch.cuda.synchronize()
    Q = host(Xd)
    h.close()
    assert res["status"] == ref["status"] == 0
    assert (res["variant"], res["passes"], res["info"]) == (ref["variant"], ref["passes"], ref["info"]) == (4, 1, 5)
    assert orth(Q) <= 1e-12
    R = Q.conj().T @ X
    assert np.abs(np.tril(R, -1)).max() <= 1e-12 * np.abs(X).max()
    assert np.linalg.norm(Q @ R - X) <= 1e-12 * np.linalg.norm(X)


def test_cholqr_zero_matrix_shifted_potrf_fails():
    """X = 0: s = 0, the shifted POTRF fails at pivot 1 -> HHQR (Alg.4 l.9) -> Q = [I; 0]."""
    import torch
    Z = np.zeros((64, 8), dtype=np.complex128)
    ref = oracle.caqr(Z, 1e9)
    h = cb.Chase(cb.CHASE_C128, 64, 8)
    Zd = dev(Z)
    res = h.cholqr(Zd, 1e9, raise_on_error=False)
    torch.cuda.synchronize()
    Q = host(Zd)
    h.close()
    assert (res["status"], res["variant"], res["passes"], res["info"]) == (0, 4, 0, 1)
    assert (ref["status"], ref["variant"], ref["passes"], ref["info"]) == (0, 4, 0, 1)
    assert np.array_equal(Q, ref["Q"])


def test_qr_mode_householder():
    """chase_set_qr_mode(h, 1): every chase_cholqr call runs HHQR (the HHQR configuration of
    P:448, Table 3), whatever the estimate."""
    import torch
    X = ci.svd_synthesized(500, 48, 1e5, 11, True)
    h = cb.Chase(cb.CHASE_C128, 500, 48)
    h.set_qr_mode(1)
    Xd = dev(X)
    res = h.cholqr(Xd, 30.0)
    torch.cuda.synchronize()
    Q = host(Xd)
    h.close()
    assert (res["variant"], res["passes"]) == (4, 0)
    assert np.linalg.norm(Q - oracle.householder_qr(X)) / math.sqrt(48) <= 100 * 1e5 * U + 1e-13
