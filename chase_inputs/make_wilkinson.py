"""Precompute the W+_N spectrum for large N (config C5, N = 200000) with LAPACK dsterf.

W+_N = tridiag(1, |i - (N-1)/2|, 1) is persymmetric, so for even N = 2m its eigenvectors are
symmetric [u; Ju] or skew [u; -Ju] and the spectrum is the union of the spectra of the two
m x m tridiagonals diag(d_0..d_{m-1}) with the last diagonal entry d_{m-1} +- 1 (off-diagonal
ones).  Each half costs O(m^2) in dsterf; the two run in parallel.  The result is stored as
chase_inputs/data/wilkinson_<N>.npy and loaded by chase_inputs.wilkinson_spectrum.
Usage: python -m chase_inputs.make_wilkinson 200000
"""
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np


def half(args):
    N, sign = args
    from scipy.linalg import eigvalsh_tridiagonal
    m = N // 2
    d = np.abs(np.arange(m, dtype=np.float64) - (N - 1) / 2.0)
    d[-1] += sign
    return eigvalsh_tridiagonal(d, np.ones(m - 1), lapack_driver="sterf")


def main(N: int):
    assert N % 2 == 0
    with ProcessPoolExecutor(2) as ex:
        a, b = ex.map(half, [(N, 1.0), (N, -1.0)])
    lam = np.sort(np.concatenate([a, b]))
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", f"wilkinson_{N}.npy")
    np.save(out, lam)
    print(out, lam[:2], lam[2499], lam[-1])


if __name__ == "__main__":
    main(int(sys.argv[1]))
