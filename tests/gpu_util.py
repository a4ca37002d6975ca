"""Helpers for the GPU parity tests: host (numpy, column-major) <-> device (torch column-major
views) without any arithmetic."""
import numpy as np


def dev(a: np.ndarray, ld: int | None = None):
    """numpy (rows, cols) -> CUDA column-major view with leading dimension ld (>= rows)."""
    import torch
    rows, cols = a.shape
    ld = rows if ld is None else ld
    if a.dtype == np.float64 and ld % 2:
        ld += 1                      # 16-byte column pitch (TMA) for real double
    buf = np.zeros((cols, ld), dtype=a.dtype)
    buf[:, :rows] = a.T
    t = torch.from_numpy(buf).cuda()
    return t.T[:rows, :]


def host(t) -> np.ndarray:
    """CUDA column-major view -> numpy (rows, cols)."""
    return t.T.cpu().numpy().T.copy()


def relF(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def colwise_rel(a, b):
    return float(np.max(np.linalg.norm(a - b, axis=0) / np.linalg.norm(b, axis=0)))
