"""The full ChASE iteration (chase_solve, Alg.2) on the GPU: converges to the lowest nev
eigenpairs of matrices with a prescribed spectrum; eigenvalues against the exact spectrum and
residuals/orthogonality recomputed independently on the host."""
import numpy as np
import pytest

import chase_inputs as ci
import oracle
import paper_2309_15595_b200 as cb
from gpu_util import dev, host

pytestmark = pytest.mark.gpu


def run(A, nev, nex, complex_, **kw):
    import torch
    N = A.shape[0]
    h = cb.Chase(cb.CHASE_C128 if complex_ else cb.CHASE_R64, N, nev + nex)
    Ad = dev(A)
    Vd = dev(np.zeros((N, nev + nex), dtype=A.dtype))
    out = h.solve(Ad, Vd, nev, nex, **kw)
    torch.cuda.synchronize()
    X = host(Vd)
    h.close()
    return out, X


@pytest.mark.parametrize("complex_", [True, False])
def test_diag_1_to_200(complex_):
    """diag(1..200) rotated by a Haar Q, nev = 20, nex = 10, tol 1e-10 ->
    Lambda = 1..20 to 1e-9, all residuals <= tol."""
    lam = np.arange(1, 201, dtype=np.float64)
    A = ci.dense_from_spectrum(lam, 3, complex_)
    out, X = run(A, 20, 10, complex_, tol=1e-10)
    assert out["status"] == 0, out
    L = out["lambda"][:20]
    assert np.max(np.abs(L - lam[:20])) <= 1e-9
    assert np.all(out["resid"][:20] <= 1e-10)
    scale = max(abs(out["stats"]["mu_1"]), abs(out["stats"]["b_sup"]))
    r = oracle.residuals(A, X[:, :20], L) / scale
    assert np.all(r <= 2e-10)
    assert np.linalg.norm(X[:, :20].conj().T @ X[:, :20] - np.eye(20)) <= 1e-11


@pytest.mark.parametrize("opt", [True, False])
def test_uniform_1000(opt):
    """Uniform spectrum on [0, 1], N = 1000, nev = 100, nex = 40 (SPEC S:622 protocol)."""
    N, nev, nex = 1000, 100, 40
    lam = ci.uniform_spectrum(N)
    A = ci.dense_from_spectrum(lam, 11, True)
    out, X = run(A, nev, nex, True, tol=1e-10, opt=opt, max_iter=30)
    assert out["status"] == 0, out
    assert np.max(np.abs(out["lambda"][:nev] - lam[:nev])) <= 1e-9
    scale = max(abs(out["stats"]["mu_1"]), abs(out["stats"]["b_sup"]))
    r = oracle.residuals(A, X[:, :nev], out["lambda"][:nev]) / scale
    assert np.all(r <= 2e-10)
    assert out["stats"]["b_sup"] >= lam[-1] - 1e-6          # Lanczos upper bound
    print(out["stats"])


def test_hhqr_mode_same_convergence():
    """"the usage of either HHQR or CholeskyQR results in the same convergence behaviour
    with the same number of MatVec operations and iterations" (Table 3).  chase_set_qr_mode(h, 1)
    runs Householder QR in every iteration; the run converges to the same eigenpairs in the same
    number of iterations and matvecs as the Alg.4 (CholeskyQR) run."""
    import torch
    N, nev, nex = 600, 40, 20
    lam = ci.uniform_spectrum(N)
    A = ci.dense_from_spectrum(lam, 5, True)
    res = {}
    for mode in (0, 1):
        h = cb.Chase(cb.CHASE_C128, N, nev + nex)
        h.set_qr_mode(mode)
        Ad = dev(A)
        Vd = dev(np.zeros((N, nev + nex), dtype=A.dtype))
        res[mode] = h.solve(Ad, Vd, nev, nex, tol=1e-10)
        torch.cuda.synchronize()
        h.close()
    for mode in (0, 1):
        assert res[mode]["status"] == 0, res[mode]
        assert np.max(np.abs(res[mode]["lambda"][:nev] - lam[:nev])) <= 1e-9
    assert res[0]["stats"]["iterations"] == res[1]["stats"]["iterations"]
    assert res[0]["stats"]["matvecs"] == res[1]["stats"]["matvecs"]


def test_clement_straddles_zero():
    """Clement spectrum lambda_k = -(N-1) + 2k (straddles 0, so Alg.5 with Lambda = 0 would give
    rho = 1 in iteration 1): the first QR must not be a single CholeskyQR pass (reading #31 --
    iteration 1 uses est = u^-1); converges with orthonormal eigenvectors."""
    N, nev, nex = 1000, 100, 40
    lam = ci.clement_spectrum(N)
    A = ci.dense_from_spectrum(lam, 13, True)
    out, X = run(A, nev, nex, True, tol=1e-10, max_iter=30)
    assert out["status"] == 0, out
    assert np.max(np.abs(out["lambda"][:nev] - lam[:nev])) <= 1e-7
    scale = max(abs(out["stats"]["mu_1"]), abs(out["stats"]["b_sup"]))
    r = oracle.residuals(A, X[:, :nev], out["lambda"][:nev]) / scale
    assert np.all(r <= 2e-10)
    assert np.linalg.norm(X[:, :nev].conj().T @ X[:, :nev] - np.eye(nev)) <= 1e-11
