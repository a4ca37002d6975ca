"""Oracle: Ritz-pair residual norms, Alg.2 l.24-28 and P:214 ("the
Euclidean norm of each column of C Lambda - H C"):

    B    <- H C                      (l.24)
    B    <- B - ritzv B2             (l.25, B2 = C redistributed, so B - ritzv C)
    nrm  <- SquaredNorm(B)           (l.26, per column)
    resd <- sqrt(nrm)                (l.28)

Global (single address space); the AllReduces of l.27 are sums over row blocks.
"""
from __future__ import annotations

import math

import numpy as np


def residuals(A: np.ndarray, V: np.ndarray, ritz) -> np.ndarray:
    B = A @ V                                          # l.24 (library matmul as the HEMM step)
    out = np.empty(V.shape[1])
    for j in range(V.shape[1]):
        r = B[:, j] - ritz[j] * V[:, j]                # l.25
        nrm = float(np.sum(np.abs(r) ** 2))            # l.26
        out[j] = math.sqrt(nrm)                        # l.28
    return out
