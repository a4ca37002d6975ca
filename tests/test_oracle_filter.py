"""Pins of the oracle filter (oracle/filter.py, oracle/grid.py) against closed forms,
brute-force eigendecomposition and hand-counted bookkeeping.  CPU only."""
import numpy as np
import pytest

import chase_inputs as ci
import oracle
from cheb_closed_form import apply_spectral, cheb_T, dft_phase_closed_form, gain, hartley_closed_form


def relF(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("c,e,mu1", [(0.55, 0.45, 0.0), (1299.0, 58700.0, -59999.0), (0.5, 0.5, -0.2)])
def test_scalars_are_chebyshev_ratios(c, e, mu1):
    """sigma_s = T_{s-1}(t1) / T_s(t1) (damped scaling of S:362)."""
    alpha, beta, sig = oracle.chebyshev_scalars(c, e, mu1, 36)
    t1 = (mu1 - c) / e
    for s in range(1, 37):
        ref = cheb_T(s - 1, np.array([t1]))[0] / cheb_T(s, np.array([t1]))[0]
        assert abs(sig[s - 1] - ref) <= 1e-13 * abs(ref)
    assert beta[0] == 0.0
    assert alpha[0] == sig[0] / e


def test_one_by_one_degree_two():
    """A = [lam], deg 2: output = (2t^2 - 1)/(2 t1^2 - 1) (T_2 written out)."""
    lam, c, e, mu1 = 0.3, 0.6, 0.4, 0.05
    A = np.array([[lam]])
    V = np.array([[1.0]])
    out, _ = oracle.chebyshev_filter(A, V, [2], c, e, mu1)
    t, t1 = (lam - c) / e, (mu1 - c) / e
    assert abs(out[0, 0] - (2 * t * t - 1) / (2 * t1 * t1 - 1)) <= 1e-15


@pytest.mark.parametrize("d", [2, 4, 8, 20, 36])
def test_diagonal_matrix_closed_form(d):
    """A = diag(lam): e_i scales by T_d(t_i)/T_d(t1)."""
    rng = np.random.default_rng(7)
    lam = np.sort(rng.uniform(-0.2, 1.0, 40))
    c, e, mu1 = 0.6, 0.4, lam[0]
    A = np.diag(lam)
    V = np.eye(40)[:, :12]
    out, _ = oracle.chebyshev_filter(A, V, [d] * 12, c, e, mu1)
    ref = np.diag(gain(d, lam, c, e, mu1))[:, :12]
    assert relF(out, ref) <= 1e-13


def test_gain_at_mu1_is_one():
    lam = np.array([-0.3, 0.1, 0.5, 0.9])
    c, e = 0.5, 0.4
    out, _ = oracle.chebyshev_filter(np.diag(lam), np.eye(4)[:, :1], [20], c, e, lam[0])
    assert abs(out[0, 0] - 1.0) <= 1e-13
    assert np.all(out[1:, 0] == 0)


@pytest.mark.parametrize("complex_", [True, False])
def test_haar_spectral_closed_form(complex_):
    """A = Q diag(lam) Q^H: p(A) V = Q g(Lam) Q^H V; ragged degrees 2..36."""
    N, n = 96, 10
    lam = ci.uniform_spectrum(N)
    Q = ci.haar_unitary(N, 11, complex_)
    A = ci.dense_from_spectrum(lam, 11, complex_)
    V = ci.gaussian_block(N, n, 12, complex_)
    b = ci.bounds_from_spectrum(lam, n)
    degs = [2, 2, 4, 6, 8, 8, 12, 20, 30, 36]
    out, _ = oracle.chebyshev_filter(A, V, degs, b.c, b.e, b.mu_1)
    ref = apply_spectral(Q, lam, V, degs, b.c, b.e, b.mu_1)
    for j in range(n):
        assert relF(out[:, j], ref[:, j]) <= 1e-12, j


def test_bruteforce_eigh_small():
    """N <= 64: compare with evaluation through numpy.linalg.eigh of the generated A."""
    N, n = 64, 6
    lam = ci.clement_spectrum(N)
    A = ci.dense_from_spectrum(lam, 3, True)
    w, U = np.linalg.eigh(A)
    V = ci.gaussian_block(N, n, 4, True)
    b = ci.bounds_from_spectrum(lam, n)
    degs = [2, 4, 4, 10, 16, 20]
    out, _ = oracle.chebyshev_filter(A, V, degs, b.c, b.e, b.mu_1)
    ref = apply_spectral(U, w, V, degs, b.c, b.e, b.mu_1)
    assert relF(out, ref) <= 1e-11


def test_dft_phase_fft_closed_form():
    N, n = 256, 8
    lam = ci.uniform_spectrum(N)
    prm = ci.dft_phase(lam, 5)
    A = prm.block(0, N, 0, N).numpy().T       # (nc, nr) storage -> A[r, s]
    assert np.array_equal(A, A.conj().T)      # exactly Hermitian
    V = ci.gaussian_block(N, n, 6, True)
    b = ci.bounds_from_spectrum(lam, n)
    degs = [20] * n
    out, _ = oracle.chebyshev_filter(A, V, degs, b.c, b.e, b.mu_1)
    ref = dft_phase_closed_form(prm, V, degs, b.c, b.e, b.mu_1)
    assert relF(out, ref) <= 1e-12


def test_hartley_fft_closed_form():
    N, n = 200, 5
    lam = ci.clement_spectrum(N)
    prm = ci.hartley_sign(lam, 8)
    A = prm.block(0, N, 0, N).numpy().T
    assert np.array_equal(A, A.T)
    V = ci.gaussian_block(N, n, 9, False)
    b = ci.bounds_from_spectrum(lam, n)
    degs = [10, 12, 14, 20, 36]
    out, _ = oracle.chebyshev_filter(A, V, degs, b.c, b.e, b.mu_1)
    ref = hartley_closed_form(prm, V, degs, b.c, b.e, b.mu_1)
    assert relF(out, ref) <= 1e-11


def test_ragged_column_equals_its_uniform_run():
    N = 50
    lam = ci.uniform_spectrum(N)
    A = ci.dense_from_spectrum(lam, 21, True)
    V = ci.gaussian_block(N, 4, 22, True)
    degs = [2, 6, 6, 14]
    out, _ = oracle.chebyshev_filter(A, V, degs, 0.6, 0.4, 0.0)
    for j, d in enumerate(degs):
        single, _ = oracle.chebyshev_filter(A, V[:, j:j + 1], [d], 0.6, 0.4, 0.0)
        assert np.allclose(out[:, j], single[:, 0], rtol=0, atol=1e-14 * np.abs(single).max())


def test_linearity():
    N = 40
    A = ci.dense_from_spectrum(ci.uniform_spectrum(N), 31, True)
    x = ci.gaussian_block(N, 1, 32, True)
    y = ci.gaussian_block(N, 1, 33, True)
    a, bb = 0.7 - 0.2j, -1.3 + 0.5j
    f = lambda v: oracle.chebyshev_filter(A, v, [8], 0.6, 0.4, 0.0)[0]
    assert relF(f(a * x + bb * y), a * f(x) + bb * f(y)) <= 1e-13


def test_schedule_matches_hand_count(golden):
    g = golden["widths"]
    steps = oracle.filter_schedule(g["degrees"])
    assert [k for (k, off, comm) in steps] == g["k"]
    n = len(g["degrees"])
    assert [off for (k, off, comm) in steps] == [n - k for k in g["k"]]
    assert [comm for (_, _, comm) in steps] == ["col" if s % 2 else "row" for s in range(1, 21)]
    rec, mv = oracle.filter_record(g["degrees"], 7, 5)
    assert mv == g["matvecs"]
    assert [el for (*_, el) in rec] == [(5 if s % 2 else 7) * k for s, k in enumerate(g["k"], 1)]


@pytest.mark.parametrize("bad", [[2, 3], [0, 2], [4, 2], [1]])
def test_rejects_bad_degrees(bad):
    with pytest.raises(ValueError):
        oracle.filter_schedule(bad)


@pytest.mark.parametrize("grid", [(1, 1), (2, 1), (1, 2), (2, 2), (2, 3), (3, 2), (2, 4)])
def test_grid_scheme_equals_global(grid):
    """Band-restricted shift + designated-rank beta (readings #6, #7) reproduce the global
    recurrence on every grid."""
    N = 61
    lam = ci.uniform_spectrum(N)
    A = ci.dense_from_spectrum(lam, 41, True)
    degs = [2, 2, 4, 4, 4, 6, 8, 8, 10, 10, 12, 12, 12, 14, 16, 18, 20]
    V = ci.gaussian_block(N, len(degs), 42, True)
    b = ci.bounds_from_spectrum(lam, len(degs))
    ref, _ = oracle.chebyshev_filter(A, V, degs, b.c, b.e, b.mu_1)
    got = oracle.distributed_filter(A, V, degs, b.c, b.e, b.mu_1, *grid)
    assert relF(got, ref) <= 1e-13


@pytest.mark.parametrize("grid,nb", [((2, 1), 1), ((1, 2), 3), ((2, 2), 4), ((2, 3), 5), ((3, 2), 16)])
def test_block_cyclic_scheme_equals_global(grid, nb):
    """Block-cyclic distribution: same recurrence, diagonal share = rows owned in
    both index sets."""
    N = 61
    lam = ci.uniform_spectrum(N)
    A = ci.dense_from_spectrum(lam, 43, True)
    degs = [2, 4, 4, 8, 12, 20]
    V = ci.gaussian_block(N, len(degs), 44, True)
    b = ci.bounds_from_spectrum(lam, len(degs))
    ref, _ = oracle.chebyshev_filter(A, V, degs, b.c, b.e, b.mu_1)
    got = oracle.distributed_filter(A, V, degs, b.c, b.e, b.mu_1, *grid, nb=nb)
    assert relF(got, ref) <= 1e-13


@pytest.mark.parametrize("grid,nb", [((2, 2), 0), ((2, 3), 0), ((3, 2), 4), ((2, 4), 3)])
@pytest.mark.parametrize("odd", [True, False])
def test_step_partials_sum_to_global_step(grid, nb, odd):
    """oracle.step_partial: the partials of a reducing communicator sum to the global step
    alpha (A - cI) X + beta Y restricted to that communicator's output rows, with beta
    added by exactly one member and the -cI shift applied exactly once per global row."""
    p, q = grid
    N, k = 53, 5
    rng = np.random.default_rng(7)
    A = ci.dense_from_spectrum(ci.uniform_spectrum(N), 45, True)
    X = rng.standard_normal((N, k)) + 1j * rng.standard_normal((N, k))
    Y = rng.standard_normal((N, k)) + 1j * rng.standard_normal((N, k))
    alpha, beta, c = 1.7, -0.3, 0.45
    glob = alpha * (A @ X - c * X) + beta * Y            # A Hermitian: A^H = A
    owned = oracle.grid._owned
    for a in range(q if odd else p):                      # one communicator per output block
        out_rows = owned(N, q, a, nb) if odd else owned(N, p, a, nb)
        acc = 0
        for b in range(p if odd else q):
            i, j = (b, a) if odd else (a, b)
            in_rows = owned(N, p, i, nb) if odd else owned(N, q, j, nb)
            acc = acc + oracle.step_partial(A, X[in_rows], Y[out_rows], i, j, p, q, odd,
                                            alpha, beta, c, b == 0, nb)
        assert relF(acc, glob[out_rows]) <= 1e-14
