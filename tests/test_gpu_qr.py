"""GPU parity of chase_cholqr (Alg.3/Alg.4) against the oracle: same executed variant, passes
and POTRF info; ||Q^H Q - I||_F <= 1e-12 after CholeskyQR2 (north star); Q equal to the
oracle's Q within C * kappa * u."""
import math

import numpy as np
import pytest

import chase_inputs as ci
import oracle
import paper_2309_15595_b200 as cb
from gpu_util import dev, host

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


def gpu_qr(X, est, complex_=True):
    import torch
    N, n = X.shape
    h = cb.Chase(cb.CHASE_C128 if complex_ else cb.CHASE_R64, N, n)
    Xd = dev(X)
    res = h.cholqr(Xd, est, raise_on_error=False)
    torch.cuda.synchronize()
    Q = host(Xd)
    h.close()
    return Q, res


def orth(Q):
    return np.linalg.norm(Q.conj().T @ Q - np.eye(Q.shape[1]))


def filtered_c1(degree, complex_=True, N=512, n=60):
    lam = ci.uniform_spectrum(N)
    A = ci.dense_from_spectrum(lam, 1, complex_)
    V0 = ci.gaussian_block(N, n, 101, complex_)
    b = ci.bounds_from_spectrum(lam, n)
    X, _ = oracle.chebyshev_filter(A, V0, [degree] * n, b.c, b.e, b.mu_1)
    est = oracle.cond_est(lam, b.c, b.e, [degree] * n, 0)
    return X, est


@pytest.mark.parametrize("complex_", [True, False])
@pytest.mark.parametrize("degree,variant", [(2, 1), (20, 2), (36, 3)])
def test_variant_ladder_c1(complex_, degree, variant):
    X, est = filtered_c1(degree, complex_)
    ref = oracle.caqr(X, est)
    Q, res = gpu_qr(X, est, complex_)
    assert res["status"] == ref["status"] == 0
    assert res["variant"] == ref["variant"] == variant
    assert res["passes"] == ref["passes"]
    if variant >= 2:
        assert orth(Q) <= 1e-12
    kappa = np.linalg.cond(X)
    assert np.linalg.norm(Q - ref["Q"]) / math.sqrt(X.shape[1]) <= 100 * kappa * U + 1e-13


@pytest.mark.parametrize("complex_", [True, False])
@pytest.mark.parametrize("m,n,kappa,est", [(700, 100, 1e3, 1e3), (1000, 33, 1e6, 1e6),
                                           (600, 70, 1e12, 1e12), (2000, 250, 1e4, 1e4)])
def test_orthogonality_ladder(complex_, m, n, kappa, est):
    X = ci.svd_synthesized(m, n, kappa, int(m + n), complex_)
    ref = oracle.caqr(X, est)
    Q, res = gpu_qr(X, est, complex_)
    assert res["status"] == ref["status"] == 0
    assert (res["variant"], res["passes"]) == (ref["variant"], ref["passes"])
    assert orth(Q) <= 1e-12 * max(1.0, math.sqrt(n / 60))
    assert np.linalg.norm(Q - ref["Q"]) / math.sqrt(n) <= 100 * kappa * U + 1e-13


def test_hand_case(golden):
    g = golden["cholesky_qr_hand"]
    X = np.array(g["X_rows"], dtype=np.complex128)
    Q, res = gpu_qr(X, 5.0)
    assert res["variant"] == 1 and res["passes"] == 1
    assert np.allclose(Q, np.array(g["Q_rows"]), atol=1e-15)


def test_escalation_and_failure_match_oracle():
    # degree-36 block with a CholeskyQR2 request: first POTRF fails -> shifted path
    X, _ = filtered_c1(36)
    ref = oracle.caqr(X, 1e3)
    Q, res = gpu_qr(X, 1e3)
    assert ref["variant"] == 3 and res["variant"] == 3 and res["status"] == 0
    assert res["passes"] == ref["passes"] == 3
    assert orth(Q) <= 1e-12
    # an exactly zero column: the shifted pass succeeds, the next Gram is singular -> HHQR
    # fallback (reading #33; tests/test_gpu_hhqr.py checks the result)
    Z = ci.svd_synthesized(300, 10, 10.0, 3, True)
    Z[:, 4] = 0
    ref = oracle.caqr(Z, 1e9)
    _, res = gpu_qr(Z, 1e9)
    assert ref["status"] == 0 and res["status"] == 0
    assert (res["variant"], res["passes"], res["info"]) == (ref["variant"], ref["passes"], ref["info"])


def test_invalid_cond_est():
    X = ci.svd_synthesized(50, 5, 10.0, 4, True)
    for est in (0.5, float("nan")):
        _, res = gpu_qr(X, est)
        assert res["status"] == 1


@pytest.mark.parametrize("complex_", [True, False])
@pytest.mark.parametrize("case", ["c1_deg36", "svd_1e12"])
def test_applied_shift_matches_oracle(complex_, case):
    """The s of Alg.4 l.5-6 the library added to the Gram diagonal equals the
    oracle's shift_value(N, n, frobenius_sq(X)) within 1e-13 relative (the device takes
    ||X||_F^2 as Re tr G, reading #12: same quantity, different summation order)."""
    if case == "c1_deg36":
        X, est = filtered_c1(36, complex_)
        assert est > 1e8
    else:
        X, est = ci.svd_synthesized(600, 70, 1e12, 670, complex_), 1e12
    ref_s = oracle.shift_value(X.shape[0], X.shape[1], oracle.frobenius_sq(X))
    Q, res = gpu_qr(X, est, complex_)
    assert res["status"] == 0 and res["variant"] == 3
    assert abs(res["shift"] - ref_s) <= 1e-13 * ref_s
    # a non-shifted call reports no shift
    _, res2 = gpu_qr(X / np.linalg.norm(X), 1e3, complex_)
    assert res2["variant"] in (2, 3)
    if res2["variant"] == 2:
        assert res2["shift"] == 0.0
