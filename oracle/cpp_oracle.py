"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY: ctypes binding of the plain triple-loop C++ oracle
(oracle/cpp/chase_oracle.cpp, C++17 + OpenMP) -- the "plain, slow CPU filter and CholeskyQR
with triple loops" of the BASELINE north star.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may use it; it shares no code with csrc/.

Functions mirror oracle/filter.py and oracle/qr.py (same readings, same notation):
  filter(A, V0, degrees, c, e, mu_1)   Eq.(1) with the S:362 scalars
  gram(X), potrf(G), trsm(X, R)        Alg.3 l.3 / l.5 / l.6
  shift(X)                             Alg.4 l.5-6, s = 11 (mn + n(n+1)) u ||X||_F^2
  caqr(X, est)                         Alg.4 dispatch, readings #9 #13 #14
Pinned by tests/test_oracle_cpp.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp")
SRC = os.path.join(_DIR, "chase_oracle.cpp")
LIB = os.path.join(_DIR, "liboracle.so")
FLAGS = ["-O2", "-std=c++17", "-fopenmp", "-fno-fast-math", "-ffp-contract=off", "-fcx-limited-range",
         "-shared", "-fPIC"]
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["g++", *FLAGS, SRC, "-o", LIB + ".tmp"], check=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


def load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        I64, I32, D, P = ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p
        lib.oracle_cpp_filter.argtypes = [I64, I64, I32, P, I64, P, I64, P, D, D, D]
        lib.oracle_cpp_filter.restype = None
        lib.oracle_cpp_gram.argtypes = [I64, I64, I32, P, I64, P]
        lib.oracle_cpp_gram.restype = None
        lib.oracle_cpp_potrf.argtypes = [I64, I32, P, P]
        lib.oracle_cpp_potrf.restype = I32
        lib.oracle_cpp_trsm.argtypes = [I64, I64, I32, P, I64, P]
        lib.oracle_cpp_trsm.restype = None
        lib.oracle_cpp_shift.argtypes = [I64, I64, I32, P, I64]
        lib.oracle_cpp_shift.restype = D
        lib.oracle_cpp_caqr.argtypes = [I64, I64, I32, P, I64, D, ctypes.POINTER(I32),
                                        ctypes.POINTER(I32), ctypes.POINTER(D)]
        lib.oracle_cpp_caqr.restype = I32
        _lib = lib
    return _lib


def _f(a, dtype):
    """Column-major contiguous copy (Fortran order) of the given dtype."""
    return np.array(a, dtype=dtype, order="F", copy=True)


def _dt(*arrs):
    return np.complex128 if any(np.iscomplexobj(a) for a in arrs) else np.float64


def filter(A, V0, degrees, c, e, mu_1):
    d = [int(x) for x in degrees]
    for j, dj in enumerate(d):
        if dj < 2 or dj % 2 or (j and dj < d[j - 1]):
            raise ValueError("degrees must be even, >= 2 and non-decreasing (P:149, P:103)")
    dt = _dt(A, V0)
    Af, V = np.asfortranarray(A, dtype=dt), _f(V0, dt)        # A read only: no copy if F-ordered
    N, n = V.shape
    deg = np.ascontiguousarray(d, dtype=np.int32)
    load().oracle_cpp_filter(N, n, int(dt == np.complex128), Af.ctypes.data, N, V.ctypes.data, N,
                             deg.ctypes.data, float(c), float(e), float(mu_1))
    return V


def gram(X):
    dt = _dt(X)
    Xf = _f(X, dt)
    m, n = Xf.shape
    G = np.zeros((n, n), dtype=dt, order="F")
    load().oracle_cpp_gram(m, n, int(dt == np.complex128), Xf.ctypes.data, m, G.ctypes.data)
    return G


def potrf(G):
    dt = _dt(G)
    Gf = _f(G, dt)
    n = Gf.shape[0]
    R = np.zeros((n, n), dtype=dt, order="F")
    info = load().oracle_cpp_potrf(n, int(dt == np.complex128), Gf.ctypes.data, R.ctypes.data)
    return R, int(info)


def trsm(X, R):
    dt = _dt(X, R)
    Xf, Rf = _f(X, dt), _f(R, dt)
    m, n = Xf.shape
    load().oracle_cpp_trsm(m, n, int(dt == np.complex128), Xf.ctypes.data, m, Rf.ctypes.data)
    return Xf


def shift(X):
    dt = _dt(X)
    Xf = _f(X, dt)
    m, n = Xf.shape
    return float(load().oracle_cpp_shift(m, n, int(dt == np.complex128), Xf.ctypes.data, m))


def caqr(X, est):
    """Returns dict(Q, variant, passes, info, shift); info != 0 (variant 4) means the Cholesky
    path failed and Alg.4 l.9 hands X to Householder QR (not part of this oracle)."""
    if not (est >= 1.0):
        raise ValueError("cond_est must be >= 1 (S:397)")
    dt = _dt(X)
    Xf = _f(X, dt)
    m, n = Xf.shape
    v, p, s = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_double()
    info = load().oracle_cpp_caqr(m, n, int(dt == np.complex128), Xf.ctypes.data, m, float(est),
                                  ctypes.byref(v), ctypes.byref(p), ctypes.byref(s))
    return dict(Q=Xf, variant=v.value, passes=p.value, info=int(info), shift=s.value)
