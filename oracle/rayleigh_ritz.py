"""Oracle: Rayleigh-Ritz projection, Alg.2 l.16-21 and P:208-212:

    B  <- H C                  (l.17)
    A  <- B2^H B               (l.18, B2 = C redistributed, so A = C^H H C)
    Lambda, A <- HE(SY)EVD(A)  (l.20; numpy.linalg.eigh, LAPACK, as the library step)
    C  <- C2 A                 (l.21)

Global (single address space).  Returns (Lambda ascending, C).
"""
from __future__ import annotations

import numpy as np


def rayleigh_ritz(A: np.ndarray, C: np.ndarray):
    B = A @ C                        # l.17
    Arr = C.conj().T @ B             # l.18-19
    lam, Y = np.linalg.eigh(Arr)     # l.20
    return lam, C @ Y                # l.21
