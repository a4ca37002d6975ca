"""Closed-form Chebyshev values used as independent pins (not the recurrence).

T_k(t) = cos(k arccos t)               |t| <= 1
       = cosh(k arccosh t)             t >= 1
       = (-1)^k cosh(k arccosh(-t))    t <= -1
The scaled filter of degree d maps eigenvalue lam to g_d(lam) = T_d((lam-c)/e) / T_d(t1),
t1 = (mu_1 - c)/e  (the damped polynomial of SPEC S:362; P:118-122 leaves scalars symbolic).
"""
import numpy as np


def cheb_T(k, t):
    t = np.asarray(t, dtype=np.float64)
    out = np.empty_like(t)
    inside = np.abs(t) <= 1.0
    out[inside] = np.cos(k * np.arccos(t[inside]))
    pos = t > 1.0
    out[pos] = np.cosh(k * np.arccosh(t[pos]))
    neg = t < -1.0
    out[neg] = (-1.0) ** k * np.cosh(k * np.arccosh(-t[neg]))
    return out


def gain(d, lam, c, e, mu_1):
    t1 = np.array([(mu_1 - c) / e])
    return cheb_T(d, (np.asarray(lam) - c) / e) / cheb_T(d, t1)[0]


def apply_spectral(U, lam, V, degrees, c, e, mu_1):
    """Column j of the result = U diag(g_{d_j}(lam)) U^H V[:, j]."""
    W = U.conj().T @ V
    out = np.empty_like(W)
    for j, d in enumerate(degrees):
        out[:, j] = gain(int(d), lam, c, e, mu_1) * W[:, j]
    return U @ out


def dft_phase_closed_form(params, V, degrees, c, e, mu_1):
    """p(A) V for A = Phi F diag(mu) F^H Phi^H via FFT, all columns, O(N n log N):
    p(A) V = Phi ifft(g(mu) * fft(conj(Phi) V))."""
    phi = params.phi[:, None]
    Y = np.fft.fft(np.conj(phi) * V, axis=0)
    out = np.empty_like(Y)
    mu = params.mu
    for j, d in enumerate(degrees):
        out[:, j] = gain(int(d), mu, c, e, mu_1) * Y[:, j]
    return phi * np.fft.ifft(out, axis=0)


def hartley_closed_form(params, V, degrees, c, e, mu_1):
    """p(A) V for real A = S H diag(mu) H S, H the normalised Hartley matrix:
    H x = (Re fft(x) - Im fft(x)) / sqrt(N)."""
    N = params.N
    s = params.sign[:, None]

    def hart(X):
        F = np.fft.fft(X, axis=0)
        return (F.real - F.imag) / np.sqrt(N)

    Y = hart(s * V)
    out = np.empty_like(Y)
    mu = params.mu
    for j, d in enumerate(degrees):
        out[:, j] = gain(int(d), mu, c, e, mu_1) * Y[:, j]
    return s * hart(out)
