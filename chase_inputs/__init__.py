"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no Chebyshev recurrence, no Gram/Cholesky/TRSM,
no condition estimate).  It only builds test matrices with a prescribed spectrum, random
starting vectors, spectral bounds and degree vectors -- the workloads of PAPER.md §4.1.2
("Artificial Matrices") and the BASELINE.json configurations.

Recipes (stated again in DESIGN.md "Input recipe"):

* Spectra ("eigenvalues ... distributed uniformly within an interval"; BASELINE adds
  Clement and Wilkinson):
    uniform   lam_k = lo + k (hi - lo)/(N - 1), k = 0..N-1          (SPEC S:251 reading)
    clement   lam_k = -(N - 1) + 2k                                 (textbook closed form)
    wilkinson eigenvalues of tridiag(1, |i - (N-1)/2|, 1)           (W+_N, via LAPACK stebz)
* Small N (<= 4096): A = Q diag(lam) Q^H with Q the Q factor of the QR factorisation of a
  seeded Gaussian matrix, phases fixed so diag(R) > 0 (Haar).  A is then made exactly
  Hermitian by mirroring the upper triangle (real diagonal), SPEC S:246/S:249 reading.
* Large N: closed-form "DFT-phase" Hermitian matrix with the exact spectrum:
    A_rs = phi_r * conj(phi_s) * a[(r - s) mod N],   a = ifft(lam[perm])
  whose eigenvectors are Phi F (F the unitary DFT).  Every element is O(1) to compute, so each
  rank fills its own block with no communication.  Entries with r > s are the conjugate of
  the (s, r) formula, so A is exactly Hermitian.  Real analogue ("Hartley-sign") for the real
  double configuration.
* Starting vectors V0: i.i.d. N(0,1) (complex: independent real and imaginary parts) from
  numpy Generator(Philox(seed)) in global column-major order; a rank takes its row slice, so
  inputs are grid-invariant (fixes the per-rank seeding P:339-348 flags).
* Bounds (Alg.1 l.2): mu_1 = lam_min, mu_ne = lam_(n), b_sup = lam_max of the exact
  spectrum; c = (b_sup + mu_ne)/2, e = (b_sup - mu_ne)/2 (Alg.2 l.3).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "uniform_spectrum", "clement_spectrum", "wilkinson_spectrum", "haar_unitary",
    "dense_from_spectrum", "DftPhase", "dft_phase", "HartleySign", "hartley_sign",
    "gaussian_block", "Bounds", "bounds_from_spectrum", "block_dims", "uniform_degrees",
    "ramp_degrees", "CONFIGS", "Config", "svd_synthesized", "cyclic_indices",
]


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


# ----------------------------------------------------------------------------- spectra
def uniform_spectrum(N: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    k = np.arange(N, dtype=np.float64)
    return lo + k * (hi - lo) / (N - 1) if N > 1 else np.array([lo], dtype=np.float64)


def clement_spectrum(N: int) -> np.ndarray:
    return -(N - 1) + 2.0 * np.arange(N, dtype=np.float64)


def wilkinson_spectrum(N: int) -> np.ndarray:
    """Eigenvalues of W+_N = tridiag(1, |i - (N-1)/2|, 1), ascending.  N = 200000 (config C5)
    is precomputed by chase_inputs/make_wilkinson.py (LAPACK dsterf on the two persymmetric
    halves) and loaded from chase_inputs/data; other N are computed here."""
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", f"wilkinson_{N}.npy")
    if os.path.exists(path):
        return np.load(path)
    from scipy.linalg import eigvalsh_tridiagonal

    d = np.abs(np.arange(N, dtype=np.float64) - (N - 1) / 2.0)
    off = np.ones(N - 1, dtype=np.float64)
    return np.sort(eigvalsh_tridiagonal(d, off, lapack_driver="sterf" if N > 2000 else "stebz"))


# ----------------------------------------------------------------------------- small dense A
def haar_unitary(N: int, seed: int, complex_: bool = True) -> np.ndarray:
    rng = _rng(seed)
    if complex_:
        Z = rng.standard_normal((N, N)) + 1j * rng.standard_normal((N, N))
    else:
        Z = rng.standard_normal((N, N))
    Q, R = np.linalg.qr(Z)
    d = np.diagonal(R)
    ph = d / np.abs(d)
    return Q * ph[None, :]


def _mirror_hermitian(A: np.ndarray) -> np.ndarray:
    """Upper triangle kept, lower := conj(upper)^T, diagonal real: exactly Hermitian."""
    U = np.triu(A, 1)
    H = U + U.conj().T
    H[np.diag_indices_from(H)] = np.real(np.diagonal(A))
    return np.asfortranarray(H)


def dense_from_spectrum(lam: np.ndarray, seed: int, complex_: bool = True) -> np.ndarray:
    """A = Q diag(lam) Q^H, Haar Q, mirrored to exact Hermitian, column-major."""
    Q = haar_unitary(lam.shape[0], seed, complex_)
    A = (Q * lam[None, :]) @ Q.conj().T
    return _mirror_hermitian(A)


# ----------------------------------------------------------------------------- large closed-form A
@dataclass
class DftPhase:
    """Parameters of A = Phi F diag(lam[perm]) F^H Phi^H (complex Hermitian, exact spectrum)."""
    N: int
    lam: np.ndarray       # spectrum, ascending
    perm: np.ndarray      # mu = lam[perm] is the DFT-ordered spectrum
    phi: np.ndarray       # unit-modulus phases, length N (complex128)
    a: np.ndarray         # first column of the circulant: a = ifft(mu), a[N-m] = conj(a[m])

    @property
    def mu(self) -> np.ndarray:
        return self.lam[self.perm]

    def block(self, r0: int, nr: int, c0: int, nc: int, device="cpu", chunk_cols: int = 2048):
        """Fill A[r0:r0+nr, c0:c0+nc] as a column-major torch.complex128 tensor on `device`.

        Returns a tensor T of shape (nc, nr) (row-major storage of the transpose) so that
        T.data_ptr() is the column-major block with leading dimension nr.
        """
        return self.block_idx(np.arange(r0, r0 + nr), np.arange(c0, c0 + nc), device, chunk_cols)

    def block_idx(self, rows, cols, device="cpu", chunk_cols: int = 2048):
        """A[rows][:, cols] for arbitrary global index arrays (block-cyclic blocks), same layout."""
        import torch

        dev = torch.device(device)
        pr = torch.from_numpy(np.ascontiguousarray(self.phi.real)).to(dev)
        pi = torch.from_numpy(np.ascontiguousarray(self.phi.imag)).to(dev)
        ar = torch.from_numpy(np.ascontiguousarray(self.a.real)).to(dev)
        ai = torch.from_numpy(np.ascontiguousarray(self.a.imag)).to(dev)
        rows_t = torch.as_tensor(np.asarray(rows, dtype=np.int64), device=dev)
        cols_t = torch.as_tensor(np.asarray(cols, dtype=np.int64), device=dev)
        nr, nc = rows_t.numel(), cols_t.numel()
        out = torch.empty((nc, nr), dtype=torch.complex128, device=dev)
        ov = torch.view_as_real(out)
        r = rows_t
        N = self.N
        for j0 in range(0, nc, chunk_cols):
            j1 = min(nc, j0 + chunk_cols)
            s = cols_t[j0:j1]
            R = r[None, :]            # (1, nr)
            S = s[:, None]            # (cols, 1)
            # canonical pair (lo, hi) = (min, max): value = phi_lo conj(phi_hi) a[(lo-hi) mod N],
            # conjugated when r > s.  Real arithmetic, one rounding per torch op, so the value
            # is bitwise independent of position, chunking and device (exact Hermitian A).
            lo = torch.minimum(R, S)
            hi = torch.maximum(R, S)
            tr = pr[lo] * pr[hi] + pi[lo] * pi[hi]
            ti = pi[lo] * pr[hi] - pr[lo] * pi[hi]
            k = torch.remainder(lo - hi, N)
            vr = tr * ar[k] - ti * ai[k]
            vi = tr * ai[k] + ti * ar[k]
            vi = torch.where(R > S, -vi, vi)
            vi = torch.where(R == S, torch.zeros_like(vi), vi)
            ov[j0:j1, :, 0] = vr
            ov[j0:j1, :, 1] = vi
            del lo, hi, tr, ti, k, vr, vi
        return out


def dft_phase(lam: np.ndarray, seed: int) -> DftPhase:
    N = lam.shape[0]
    rng = _rng(seed)
    perm = rng.permutation(N)
    phi = np.exp(2j * np.pi * rng.random(N))
    mu = lam[perm]
    a = np.fft.ifft(mu.astype(np.complex128))
    # enforce exact conjugate symmetry (mu real) and a real a[0]
    a[0] = a[0].real
    m = np.arange(1, (N + 1) // 2)
    a[N - m] = np.conj(a[m])
    if N % 2 == 0:
        a[N // 2] = a[N // 2].real
    return DftPhase(N=N, lam=lam, perm=perm, phi=phi, a=a)


@dataclass
class HartleySign:
    """Real symmetric A = S H diag(lam[perm]) H S (H the normalised Hartley matrix, S = diag(+-1))."""
    N: int
    lam: np.ndarray
    perm: np.ndarray
    sign: np.ndarray      # +-1, length N
    ac: np.ndarray        # (1/N) sum_k mu_k cos(2 pi m k / N), mirrored: ac[N-m] = ac[m]
    as_: np.ndarray       # (1/N) sum_k mu_k sin(2 pi m k / N)

    @property
    def mu(self) -> np.ndarray:
        return self.lam[self.perm]

    def block(self, r0: int, nr: int, c0: int, nc: int, device="cpu", chunk_cols: int = 4096):
        """A[r0:r0+nr, c0:c0+nc] as torch.float64 (nc, nr) tensor (column-major block, ld nr).

        cas(x) = cos x + sin x; (H diag(mu) H)_rs = (1/N) sum_k mu_k cas(2pi rk/N) cas(2pi sk/N)
        = ac[(r-s) mod N] + as_[(r+s) mod N]  (product-to-sum identity).  Symmetric in (r, s)
        by construction because ac is mirrored and (r+s) is symmetric.
        """
        return self.block_idx(np.arange(r0, r0 + nr), np.arange(c0, c0 + nc), device, chunk_cols)

    def block_idx(self, rows, cols, device="cpu", chunk_cols: int = 4096):
        """A[rows][:, cols] for arbitrary global index arrays (block-cyclic blocks)."""
        import torch

        dev = torch.device(device)
        sg = torch.from_numpy(self.sign).to(dev)
        ac = torch.from_numpy(self.ac).to(dev)
        as_ = torch.from_numpy(self.as_).to(dev)
        r = torch.as_tensor(np.asarray(rows, dtype=np.int64), device=dev)
        cols_t = torch.as_tensor(np.asarray(cols, dtype=np.int64), device=dev)
        nr, nc = r.numel(), cols_t.numel()
        out = torch.empty((nc, nr), dtype=torch.float64, device=dev)
        N = self.N
        for j0 in range(0, nc, chunk_cols):
            j1 = min(nc, j0 + chunk_cols)
            s = cols_t[j0:j1]
            R = r[None, :]
            S = s[:, None]
            val = ac[torch.remainder(R - S, N)] + as_[torch.remainder(R + S, N)]
            out[j0:j1] = sg[R] * sg[S] * val
        return out


def hartley_sign(lam: np.ndarray, seed: int) -> HartleySign:
    N = lam.shape[0]
    rng = _rng(seed)
    perm = rng.permutation(N)
    sign = np.where(rng.random(N) < 0.5, -1.0, 1.0)
    mu = lam[perm]
    F = np.fft.fft(mu)            # sum_k mu_k e^{-2 pi i m k / N}
    ac = F.real / N               # (1/N) sum mu_k cos
    as_ = -F.imag / N             # (1/N) sum mu_k sin
    m = np.arange(1, (N + 1) // 2)
    ac[N - m] = ac[m]
    return HartleySign(N=N, lam=lam, perm=perm, sign=sign, ac=ac, as_=as_)


# ----------------------------------------------------------------------------- vectors, bounds
def gaussian_block(N: int, n: int, seed: int, complex_: bool = True) -> np.ndarray:
    """N x n standard normal block, column-major, drawn in global column-major order."""
    rng = _rng(seed)
    if complex_:
        # draw (re, im) pairs element by element in column-major order
        x = rng.standard_normal(2 * N * n).view(np.complex128)
    else:
        x = rng.standard_normal(N * n)
    return x.reshape(n, N).T  # Fortran-ordered view (column-major)


def svd_synthesized(m: int, n: int, kappa: float, seed: int, complex_: bool = True) -> np.ndarray:
    """X = U diag(s) W^H with singular values geometrically spaced in [1/kappa, 1]."""
    rng = _rng(seed)
    if complex_:
        G1 = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
        G2 = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    else:
        G1 = rng.standard_normal((m, n))
        G2 = rng.standard_normal((n, n))
    U, _ = np.linalg.qr(G1)
    W, _ = np.linalg.qr(G2)
    s = np.logspace(0.0, -math.log10(kappa), n)
    return np.asfortranarray((U * s[None, :]) @ W.conj().T)


@dataclass
class Bounds:
    mu_1: float
    mu_ne: float
    b_sup: float

    @property
    def c(self) -> float:
        return (self.b_sup + self.mu_ne) / 2.0

    @property
    def e(self) -> float:
        return (self.b_sup - self.mu_ne) / 2.0


def bounds_from_spectrum(lam: np.ndarray, n: int) -> Bounds:
    lam = np.sort(lam)
    return Bounds(mu_1=float(lam[0]), mu_ne=float(lam[n - 1]), b_sup=float(lam[-1]))


def block_dims(N: int, p: int, q: int, i: int, j: int):
    """Block distribution with the remainder rule of SPEC S:102: the first N mod p grid rows
    get ceil(N/p) rows.  Returns (n_r, n_c, r0, c0)."""
    def part(N, P, k):
        b, rem = divmod(N, P)
        size = b + (1 if k < rem else 0)
        start = k * b + min(k, rem)
        return size, start
    n_r, r0 = part(N, p, i)
    n_c, c0 = part(N, q, j)
    return n_r, n_c, r0, c0


def cyclic_indices(N: int, P: int, k: int, nb: int) -> np.ndarray:
    """Global indices owned by grid row/column k of P under the block-cyclic distribution with
    block size nb: g with (g // nb) % P == k, increasing."""
    g = np.arange(N)
    return g[(g // nb) % P == k]


def uniform_degrees(n: int, d: int) -> np.ndarray:
    return np.full(n, d, dtype=np.int32)


def ramp_degrees(n: int, lo: int = 10, hi: int = 36) -> np.ndarray:
    """d_j = lo + 2 floor(((hi - lo)/2 + 1) j / n): non-decreasing even ramp lo..hi (config C5,
    SURVEY §8(d): d_j = 10 + 2 floor(14 j / 2500), sum 57,488)."""
    j = np.arange(n, dtype=np.int64)
    steps = (hi - lo) // 2 + 1
    return (lo + 2 * ((steps * j) // n)).astype(np.int32)


# ----------------------------------------------------------------------------- BASELINE configs
@dataclass
class Config:
    name: str
    N: int
    nev: int
    nex: int
    complex_: bool
    spectrum: str
    seed: int
    degree: int | None     # uniform degree, or None for the ramp
    grid: tuple            # default (p, q)

    @property
    def n(self) -> int:
        return self.nev + self.nex

    def spectrum_values(self) -> np.ndarray:
        if self.spectrum == "uniform":
            return uniform_spectrum(self.N)
        if self.spectrum == "clement":
            return clement_spectrum(self.N)
        if self.spectrum == "wilkinson":
            return wilkinson_spectrum(self.N)
        raise ValueError(self.spectrum)

    def degrees(self) -> np.ndarray:
        return uniform_degrees(self.n, self.degree) if self.degree else ramp_degrees(self.n)


CONFIGS = {
    "C1": Config("C1", 512, 40, 20, True, "uniform", 1, 20, (1, 1)),
    "C2": Config("C2", 30000, 2250, 750, True, "uniform", 2, 20, (1, 1)),
    "C3": Config("C3", 60000, 1000, 300, True, "clement", 3, 20, (1, 1)),
    "C4": Config("C4", 120000, 1200, 400, True, "uniform", 4, 20, (2, 4)),
    "C5": Config("C5", 200000, 2000, 500, False, "wilkinson", 5, None, (2, 4)),
}
