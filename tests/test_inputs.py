"""Input generators (chase_inputs): exact spectra, exact Hermitian symmetry, grid-invariant
block slicing, remainder rule.  CPU only."""
import numpy as np
import pytest

import chase_inputs as ci


def test_spectra():
    assert np.array_equal(ci.uniform_spectrum(5), [0, 0.25, 0.5, 0.75, 1.0])
    lam = ci.clement_spectrum(50)
    T = np.diag(np.sqrt(np.arange(1, 50) * np.arange(49, 0, -1)), 1)
    assert np.allclose(np.linalg.eigvalsh(T + T.T), lam, atol=1e-12)
    w = ci.wilkinson_spectrum(21)
    d = np.abs(np.arange(21) - 10.0)
    W = np.diag(d) + np.diag(np.ones(20), 1) + np.diag(np.ones(20), -1)
    assert np.allclose(np.linalg.eigvalsh(W), w, atol=1e-12)


def test_dense_from_spectrum():
    lam = ci.uniform_spectrum(64)
    A = ci.dense_from_spectrum(lam, 3, True)
    assert np.array_equal(A, A.conj().T)
    assert np.allclose(np.linalg.eigvalsh(A), lam, atol=1e-13)


@pytest.mark.parametrize("N", [97, 128])
def test_dft_phase_blocks(N):
    lam = ci.uniform_spectrum(N)
    prm = ci.dft_phase(lam, 4)
    A = prm.block(0, N, 0, N).numpy().T
    assert np.array_equal(A, A.conj().T)
    assert np.allclose(np.linalg.eigvalsh(A), lam, atol=1e-13)
    for (p, q) in [(2, 3), (3, 2)]:
        for i in range(p):
            for j in range(q):
                nr, nc, r0, c0 = ci.block_dims(N, p, q, i, j)
                B = prm.block(r0, nr, c0, nc).numpy().T
                assert np.array_equal(B, A[r0:r0 + nr, c0:c0 + nc])


def test_hartley_blocks():
    N = 90
    lam = ci.clement_spectrum(N)
    prm = ci.hartley_sign(lam, 6)
    A = prm.block(0, N, 0, N).numpy().T
    assert np.array_equal(A, A.T)
    assert np.allclose(np.linalg.eigvalsh(A), lam, atol=1e-11)
    B = prm.block(10, 30, 45, 40).numpy().T
    assert np.array_equal(B, A[10:40, 45:85])


def test_block_dims_remainder_rule():
    dims = [ci.block_dims(10, 3, 4, i, 0) for i in range(3)]
    assert [d[0] for d in dims] == [4, 3, 3] and [d[2] for d in dims] == [0, 4, 7]
    dims = [ci.block_dims(10, 3, 4, 0, j) for j in range(4)]
    assert [d[1] for d in dims] == [3, 3, 2, 2] and [d[3] for d in dims] == [0, 3, 6, 8]


def test_gaussian_block_is_global():
    V = ci.gaussian_block(50, 4, 9, True)
    V2 = ci.gaussian_block(50, 4, 9, True)
    assert np.array_equal(V, V2)
    assert V.flags["F_CONTIGUOUS"]
    assert abs(np.mean(np.abs(V) ** 2) - 2.0) < 0.3


def test_ramp_degrees_c5():
    d = ci.ramp_degrees(2500)
    assert d[0] == 10 and d[-1] == 36 and d.sum() == 57488
    assert np.all(np.diff(d) >= 0) and np.all(d % 2 == 0)
