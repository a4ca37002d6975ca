"""Multi-GPU parity (torchrun, one rank per GPU, NCCL over NVLink): the 2D-distributed filter
and the 1D-CAQR over the column communicator match the global oracle; replicas across the
row communicator are bitwise identical; bookkeeping equals the oracle's per-rank record.
Skipped when fewer than 2 GPUs are visible."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import chase_inputs as ci
import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def torchrun(nproc, script_args, timeout):
    """Launch a torchrun job on 127.0.0.1; retry on a rendezvous port collision."""
    for attempt in range(4):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), *script_args]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
        if r.returncode == 0 or "EADDRINUSE" not in (r.stdout + r.stderr):
            return r
    return r


GRIDS = [(2, 1), (1, 2), (2, 2), (4, 1), (1, 4)]


CASES = ([(c, g, 0, "nccl", 0) for c in (True, False) for g in GRIDS] +
         [(True, (1, 2), 6, "nccl", 0), (False, (1, 2), 5, "nccl", 0), (True, (2, 2), 6, "nccl", 0)] +
         [(True, g, 0, "fused", 0) for g in GRIDS] + [(True, (1, 2), 6, "fused", 0)] +
         [(True, (2, 1), 0, "nccl", 7), (False, (1, 2), 0, "nccl", 1), (True, (2, 2), 0, "nccl", 16),
          (True, (1, 2), 0, "fused", 5), (True, (2, 2), 0, "fused", 32), (False, (2, 2), 0, "nccl", 3)] +
         [(False, g, 0, "fused", 0) for g in GRIDS] + [(False, (1, 2), 5, "fused", 0), (False, (2, 2), 0, "fused", 3)])


@pytest.mark.parametrize("complex_,grid,pad,mode,nb", CASES)
def test_grid_matches_oracle(tmp_path, grid, complex_, pad, mode, nb):
    """pad > 0: leading dimensions larger than the local rows (strided AllReduce path).
    mode "fused": filter steps as one HEMM + NVLink peer-memory reduction kernel.
    nb > 0: block-cyclic distribution with block size nb."""
    p, q = grid
    if ngpus() < p * q:
        pytest.skip(f"needs {p * q} GPUs")
    N = 301
    out = str(tmp_path / "res.npz")
    r = torchrun(p * q, [os.path.join(ROOT, "tests", "mp_gpu_worker.py"), str(p), str(q), str(N),
                         "c" if complex_ else "r", out, str(pad), mode, str(nb)], 600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = np.load(out)
    degs = sorted([2, 2, 4, 4, 4, 6, 8, 8, 10, 10, 12, 12, 12, 14, 16, 18, 20] * 3)
    n = len(degs)
    lam = ci.uniform_spectrum(N)
    A = ci.dense_from_spectrum(lam, 77, complex_)
    V0 = ci.gaussian_block(N, n, 78, complex_)
    b = ci.bounds_from_spectrum(lam, n)
    ref, _ = oracle.chebyshev_filter(A, V0, degs, b.c, b.e, b.mu_1)
    V = res["V"]
    err = np.max(np.linalg.norm(V - ref, axis=0) / np.linalg.norm(ref, axis=0))
    assert err <= 1e-10
    assert float(res["replica"]) == 0.0                       # identical bits on all replicas
    assert np.all(res["repeat_equal"])                        # bitwise repeatable
    assert np.all(res["mv"] == sum(degs))
    for (i, j, n_r, n_c), recs in zip(res["ranks"], res["recs"]):
        if nb == 0:
            assert (n_r, n_c) == ci.block_dims(N, p, q, int(i), int(j))[:2]
        else:
            assert n_r == len(ci.cyclic_indices(N, p, int(i), nb))
            assert n_c == len(ci.cyclic_indices(N, q, int(j), nb))
        orec, _ = oracle.filter_record(degs, int(n_r), int(n_c))
        assert recs == str(orec)
    qref = oracle.caqr(ref, float(res["est"]))
    assert np.all(res["status"] == 0)
    assert np.all(res["variants"] == qref["variant"]) and np.all(res["passes"] == qref["passes"])
    Q = res["Q"]
    assert np.linalg.norm(Q.conj().T @ Q - np.eye(n)) <= 1e-12
    kappa = np.linalg.cond(ref)
    assert np.linalg.norm(Q - qref["Q"]) / np.sqrt(n) <= 100 * kappa * 2.0 ** -53 + 1e-13
    # Householder QR (Alg.4 l.9) over the column communicator: the oracle's HHQR Q
    Hq = res["H"]
    assert np.linalg.norm(Hq.conj().T @ Hq - np.eye(n)) <= 1e-12
    assert np.linalg.norm(Hq - oracle.householder_qr(ref)) / np.sqrt(n) <= 100 * kappa * 2.0 ** -53 + 1e-13
    # residuals (Alg.2 l.23-28): identical on every rank, equal to the oracle on the gathered Q
    rres = oracle.residuals(A, Q, res["ritz"])
    assert np.all(res["resid"] == res["resid"][0])
    assert np.max(np.abs(res["resid"][0] - rres) / rres) <= 1e-10
    # Rayleigh-Ritz (Alg.2 l.16-22): Ritz values identical on every rank and equal to the oracle's
    theta_ref, X_ref = oracle.rayleigh_ritz(A, Q)
    assert np.all(res["theta"] == res["theta"][0])
    assert np.max(np.abs(res["theta"][0] - theta_ref)) <= 1e-12 * np.max(np.abs(theta_ref))
    X = res["X"]
    assert np.linalg.norm(X.conj().T @ X - np.eye(n)) <= 1e-11


FULL = [(c, g, m) for c, g in [("C3", (2, 1)), ("C3", (2, 2)), ("C3", (2, 4)), ("C4", (2, 2)),
                                ("C4", (2, 4)), ("C5", (2, 2)), ("C5", (1, 4)), ("C5", (4, 1)),
                                ("C5", (2, 4))]
        for m in ("fused", "nccl")]


@pytest.mark.slow
@pytest.mark.parametrize("name,grid,mode", FULL)
def test_full_size_grid(tmp_path, name, grid, mode):
    """BASELINE configurations on the 2D grid: closed-form filter check of sampled columns on every
    rank, per-rank bookkeeping, Alg.4 variant and distributed orthogonality (tests/full_worker.py),
    with the filter steps as fused HEMM + NVLink reduction kernels or HEMM + ncclAllReduce."""
    import json
    p, q = grid
    if ngpus() < p * q:
        pytest.skip(f"needs {p * q} GPUs")
    out = str(tmp_path / "full.json")
    r = torchrun(p * q, [os.path.join(ROOT, "tests", "full_worker.py"), name, str(p), str(q), out,
                         mode], 1800)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    for res in json.load(open(out)):
        print(res)
        assert res["closed_form_col_err"] <= 1e-10, res
        assert res["record_equal"], res
        assert res["qr_variant"] == res["oracle_variant"], res
        assert res["orth"] <= 1e-12, res


@pytest.mark.parametrize("grid", [(1, 1), (2, 1), (1, 2), (2, 2)])
def test_solve_grid(tmp_path, grid):
    """the full ChASE loop on a p x q grid converges to the lowest nev
    eigenpairs of Uniform[0,1] (N = 400); identical eigenvalues on every rank."""
    p, q = grid
    if ngpus() < p * q:
        pytest.skip(f"needs {p * q} GPUs")
    N, nev, nex = 400, 40, 20
    out = str(tmp_path / "solve.npz")
    r = torchrun(p * q, [os.path.join(ROOT, "tests", "mp_solve_worker.py"), str(p), str(q), str(N),
                         str(nev), str(nex), out], 900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = np.load(out)
    lam = ci.uniform_spectrum(N)
    assert int(res["status"]) == 0 and bool(res["same"])
    assert np.max(np.abs(res["lam"][:nev] - lam[:nev])) <= 1e-9
    A = ci.dense_from_spectrum(lam, 21, True)
    X = res["X"][:, :nev]
    rr = oracle.residuals(A, X, res["lam"][:nev])
    assert np.max(rr) <= 1e-9


def test_spmd_check(tmp_path):
    """include/chase.h: collective calls need identical scalar arguments; with CHASE_SPMD_CHECK=1
    a disagreeing rank makes chase_filter return CHASE_EINVAL on every rank (hash min != max over
    the world communicator) before any device work."""
    import json
    if ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    out = str(tmp_path / "spmd.json")
    r = torchrun(2, [os.path.join(ROOT, "tests", "mp_spmd_worker.py"), out], 300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    for res in json.load(open(out)):
        assert res["mismatch_status"] == 1 and res["untouched"] and res["agree_status"] == 0, res
