"""B200-native ChASE hot path (arXiv 2309.15595): the 2D-distributed Chebyshev filter and the
condition-driven CholeskyQR family, behind the C-ABI of include/chase.h (libchase.so).

This module is argument marshalling only (ctypes): every step of the path runs in the CUDA
kernels and NCCL collectives of libchase.so.  There is no CPU fallback -- if the library is
missing or a call fails, an exception is raised.

Matrices are column-major.  From PyTorch pass a 2-D tensor with shape (rows, cols) and
strides (1, ld) -- e.g. ``colmajor_empty(rows, cols)`` or ``t.T`` of a contiguous (cols, rows)
tensor; its leading dimension is ``stride(1)``.
"""
from __future__ import annotations

import ctypes
import os
from typing import Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CHASE_LIB") or os.path.join(_PKG, "libchase.so")   # CHASE_LIB: A/B builds

CHASE_R64, CHASE_C128 = 1, 2
CHASE_QR_CHOL1, CHASE_QR_CHOL2, CHASE_QR_SHIFTED, CHASE_QR_HOUSEHOLDER = 1, 2, 3, 4
STATUS = {0: "CHASE_OK", 1: "CHASE_EINVAL", 2: "CHASE_EDEGREE", 3: "CHASE_EBOUNDS",
          4: "CHASE_ECHOL", 5: "CHASE_ECUDA", 6: "CHASE_ENCCL", 7: "CHASE_ENOMEM",
          8: "CHASE_ESTATE", 9: "CHASE_ENOCONV"}
PROFILE_CATEGORIES = ("hemm_odd", "hemm_even", "allreduce", "gram", "potrf", "trsm", "other", "hhqr")

# every symbol include/chase.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "chase_get_unique_id", "chase_create", "chase_set_stream", "chase_local_dims",
    "chase_block_dims", "chase_workspace_size", "chase_set_workspace", "chase_filter",
    "chase_filter_record", "chase_filter_schedule", "chase_cholqr", "chase_cond_est",
    "chase_shift_value", "chase_profile_enable", "chase_profile_read", "chase_destroy",
    "chase_status_string", "chase_residuals", "chase_fused_workspace_size",
    "chase_set_fused_workspace", "chase_create_cyclic", "chase_local_indices",
    "chase_cyclic_indices", "chase_rayleigh_ritz", "chase_solve", "chase_hhqr",
    "chase_set_qr_mode", "chase_create_virtual", "chase_set_fused_mode", "chase_filter_step",
)


class ChaseError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {STATUS.get(status, status)} ({_status_string(status)})")


class chase_bounds_t(ctypes.Structure):
    _fields_ = [("mu_1", ctypes.c_double), ("mu_ne", ctypes.c_double), ("b_sup", ctypes.c_double)]


class chase_stats_t(ctypes.Structure):
    _fields_ = [("matvecs", ctypes.c_int64), ("steps", ctypes.c_int32),
                ("qr_variant", ctypes.c_int32), ("qr_passes", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("shift", ctypes.c_double)]


class chase_solve_stats_t(ctypes.Structure):
    _fields_ = [("matvecs", ctypes.c_int64), ("iterations", ctypes.c_int32), ("locked", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("b_sup", ctypes.c_double), ("mu_1", ctypes.c_double),
                ("mu_ne", ctypes.c_double)]


class chase_step_record_t(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("off", ctypes.c_int32), ("comm", ctypes.c_int32),
                ("use_beta", ctypes.c_int32), ("elems", ctypes.c_int64),
                ("band_lo", ctypes.c_int32), ("band_hi", ctypes.c_int32)]


_lib = None


def load() -> ctypes.CDLL:
    """Load libchase.so (built in-tree by build.py).  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2309_15595_b200.build`")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    c_i64p = ctypes.POINTER(ctypes.c_int64)
    V, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    sig = {
        "chase_get_unique_id": (I32, [ctypes.c_char_p]),
        "chase_create": (I32, [ctypes.POINTER(V), I32, I64, I64, I32, I32, I32, I32, ctypes.c_char_p, I32, V]),
        "chase_set_stream": (I32, [V, V]),
        "chase_create_cyclic": (I32, [ctypes.POINTER(V), I32, I64, I64, I32, I32, I32, I32, I64, ctypes.c_char_p, I32, V]),
        "chase_create_virtual": (I32, [ctypes.POINTER(V), I32, I64, I64, I32, I32, I32, I32, I64, I32, V]),
        "chase_set_fused_mode": (I32, [V, I32, I32]),
        "chase_filter_step": (I32, [V, V, I64, V, I64, V, I64, I64, I32, D, D, D, I32]),
        "chase_local_indices": (I32, [V, c_i64p, c_i64p]),
        "chase_cyclic_indices": (I32, [I64, I32, I32, I64, c_i64p, c_i64p]),
        "chase_local_dims": (I32, [V, c_i64p, c_i64p, c_i64p, c_i64p]),
        "chase_block_dims": (I32, [I64, I32, I32, I32, I32, c_i64p, c_i64p, c_i64p, c_i64p]),
        "chase_workspace_size": (I32, [V, ctypes.POINTER(ctypes.c_size_t)]),
        "chase_set_workspace": (I32, [V, V, ctypes.c_size_t]),
        "chase_filter": (I32, [V, V, I64, V, I64, I64, ctypes.POINTER(I32), D, D,
                               ctypes.POINTER(chase_bounds_t), ctypes.POINTER(chase_stats_t)]),
        "chase_filter_record": (I32, [V, I32, ctypes.POINTER(chase_step_record_t), ctypes.POINTER(I32), c_i64p]),
        "chase_filter_schedule": (I32, [I64, I32, I32, I32, I32, I64, ctypes.POINTER(I32), I32,
                                        ctypes.POINTER(chase_step_record_t), ctypes.POINTER(I32), c_i64p]),
        "chase_cholqr": (I32, [V, V, I64, I64, D, ctypes.POINTER(chase_stats_t), ctypes.POINTER(I32)]),
        "chase_hhqr": (I32, [V, V, I64, I64]),
        "chase_set_qr_mode": (I32, [V, I32]),
        "chase_cond_est": (D, [ctypes.POINTER(D), I64, D, D, ctypes.POINTER(I32), I64]),
        "chase_residuals": (I32, [V, V, I64, V, I64, I64, ctypes.POINTER(D), ctypes.POINTER(D)]),
        "chase_fused_workspace_size": (I32, [V, ctypes.POINTER(ctypes.c_size_t)]),
        "chase_rayleigh_ritz": (I32, [V, V, I64, V, I64, I64, ctypes.POINTER(D), ctypes.POINTER(I32)]),
        "chase_solve": (I32, [V, V, I64, V, I64, I64, I64, D, I32, I32, I32, I32, ctypes.c_uint64, I32,
                              ctypes.POINTER(D), ctypes.POINTER(D), ctypes.POINTER(chase_solve_stats_t)]),
        "chase_set_fused_workspace": (I32, [V, V, ctypes.POINTER(ctypes.c_uint64), I32]),
        "chase_shift_value": (D, [I64, I64, D]),
        "chase_profile_enable": (I32, [V, I32]),
        "chase_profile_read": (I32, [V, ctypes.POINTER(D), c_i64p]),
        "chase_destroy": (I32, [V]),
        "chase_status_string": (ctypes.c_char_p, [I32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _status_string(s: int) -> str:
    try:
        return load().chase_status_string(s).decode()
    except Exception:
        return "?"


def _check(status: int, where: str):
    if status != 0:
        raise ChaseError(status, where)


def _i32_array(values: Sequence[int]):
    arr = np.ascontiguousarray(np.asarray(values, dtype=np.int32))
    return arr, arr.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def _colmajor(t, name: str):
    """(pointer, ld) of a column-major 2-D CUDA tensor view (stride(0) == 1)."""
    if t.dim() != 2 or t.stride(0) != 1:
        raise ValueError(f"{name} must be a column-major 2-D tensor view (stride(0) == 1)")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path)")
    return t.data_ptr(), max(t.stride(1), t.shape[0])


def colmajor_empty(rows: int, cols: int, dtype=None, device="cuda"):
    import torch
    dtype = dtype or torch.complex128
    return torch.empty((cols, rows), dtype=dtype, device=device).T


# ------------------------------------------------------------------------------ C-ABI wrappers
def chase_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().chase_get_unique_id(buf), "chase_get_unique_id")
    return buf.raw


def chase_create(dtype: int, N: int, n_max: int, p: int = 1, q: int = 1, myrow: int = 0,
                 mycol: int = 0, uid: bytes | None = None, device: int = 0, stream: int = 0,
                 nb: int = 0, virtual: bool = False):
    """nb > 0: block-cyclic distribution with block size nb (chase_create_cyclic).
    virtual: a rank of a grid living in this process on one device (chase_create_virtual)."""
    h = ctypes.c_void_p()
    if virtual:
        _check(load().chase_create_virtual(ctypes.byref(h), dtype, N, n_max, p, q, myrow, mycol, nb,
                                           device, ctypes.c_void_p(stream)), "chase_create_virtual")
    elif nb:
        _check(load().chase_create_cyclic(ctypes.byref(h), dtype, N, n_max, p, q, myrow, mycol, nb,
                                          uid, device, ctypes.c_void_p(stream)), "chase_create_cyclic")
    else:
        _check(load().chase_create(ctypes.byref(h), dtype, N, n_max, p, q, myrow, mycol, uid, device,
                                   ctypes.c_void_p(stream)), "chase_create")
    return h


def chase_local_indices(h, n_r: int, n_c: int):
    rows = np.empty(n_r, dtype=np.int64)
    cols = np.empty(n_c, dtype=np.int64)
    _check(load().chase_local_indices(h, rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                      cols.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))),
           "chase_local_indices")
    return rows, cols


def chase_cyclic_indices(N: int, P: int, k: int, nb: int):
    cnt = ctypes.c_int64()
    _check(load().chase_cyclic_indices(N, P, k, nb, None, ctypes.byref(cnt)), "chase_cyclic_indices")
    idx = np.empty(cnt.value, dtype=np.int64)
    _check(load().chase_cyclic_indices(N, P, k, nb, idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                       ctypes.byref(cnt)), "chase_cyclic_indices")
    return idx


def chase_set_stream(h, stream: int):
    _check(load().chase_set_stream(h, ctypes.c_void_p(stream)), "chase_set_stream")


def chase_local_dims(h):
    v = [ctypes.c_int64() for _ in range(4)]
    _check(load().chase_local_dims(h, *[ctypes.byref(x) for x in v]), "chase_local_dims")
    return tuple(x.value for x in v)


def chase_block_dims(N: int, p: int, q: int, i: int, j: int):
    v = [ctypes.c_int64() for _ in range(4)]
    _check(load().chase_block_dims(N, p, q, i, j, *[ctypes.byref(x) for x in v]), "chase_block_dims")
    return tuple(x.value for x in v)


def chase_workspace_size(h) -> int:
    b = ctypes.c_size_t()
    _check(load().chase_workspace_size(h, ctypes.byref(b)), "chase_workspace_size")
    return b.value


def chase_set_workspace(h, ws):
    """ws: a CUDA tensor of at least chase_workspace_size(h) bytes (kept alive by the caller)."""
    _check(load().chase_set_workspace(h, ctypes.c_void_p(ws.data_ptr()),
                                      ws.numel() * ws.element_size()), "chase_set_workspace")


def chase_fused_workspace_size(h) -> int:
    b = ctypes.c_size_t()
    _check(load().chase_fused_workspace_size(h, ctypes.byref(b)), "chase_fused_workspace_size")
    return b.value


def chase_set_fused_workspace(h, local_ptr: int | None, peer_ptrs=None):
    """peer_ptrs[r] = address of world rank r's symmetric region mapped in this process."""
    if not local_ptr:
        _check(load().chase_set_fused_workspace(h, None, None, 0), "chase_set_fused_workspace")
        return
    arr = (ctypes.c_uint64 * len(peer_ptrs))(*[int(x) for x in peer_ptrs])
    _check(load().chase_set_fused_workspace(h, ctypes.c_void_p(local_ptr), arr, len(peer_ptrs)),
           "chase_set_fused_workspace")


def chase_set_fused_mode(h, mode: int, sm_budget: int = 0):
    """mode 1: every filter step runs the fused kernel (also single-member communicators);
    sm_budget > 0: cap on the persistent fused grid (include/chase.h)."""
    _check(load().chase_set_fused_mode(h, int(mode), int(sm_budget)), "chase_set_fused_mode")


def chase_filter_step(h, A_local, X, Y, odd: bool, alpha: float, beta: float, c: float,
                      use_beta: bool, k: int | None = None):
    """This rank's partial of one filter step into Y, no reduction (include/chase.h)."""
    a_ptr, lda = _colmajor(A_local, "A_local")
    x_ptr, ldx = _colmajor(X, "X")
    y_ptr, ldy = _colmajor(Y, "Y")
    k = X.shape[1] if k is None else k
    _check(load().chase_filter_step(h, a_ptr, lda, x_ptr, ldx, y_ptr, ldy, k, 1 if odd else 0,
                                    float(alpha), float(beta), float(c), 1 if use_beta else 0),
           "chase_filter_step")


def chase_filter(h, A_local, V, degrees, c: float, e: float, bounds, ncols: int | None = None):
    """Chebyshev filter in place on V (see include/chase.h).  bounds = (mu_1, mu_ne, b_sup)."""
    a_ptr, lda = _colmajor(A_local, "A_local")
    v_ptr, ldv = _colmajor(V, "V")
    ncols = V.shape[1] if ncols is None else ncols
    arr, dp = _i32_array(degrees)
    if arr.shape[0] < ncols:
        raise ValueError("degrees shorter than ncols")
    b = chase_bounds_t(*[float(x) for x in bounds])
    st = chase_stats_t()
    _check(load().chase_filter(h, a_ptr, lda, v_ptr, ldv, ncols, dp, float(c), float(e),
                               ctypes.byref(b), ctypes.byref(st)), "chase_filter")
    return {"matvecs": st.matvecs, "steps": st.steps}


def _records(n, rec, full: bool = False):
    """(k, off, comm, elems) per step, the oracle's record schema; full=True appends
    (use_beta, band_lo, band_hi)."""
    out = []
    for i in range(n):
        r = rec[i]
        t = (r.k, r.off, "col" if r.comm == 0 else "row", r.elems)
        out.append(t + (r.use_beta, r.band_lo, r.band_hi) if full else t)
    return out


def chase_filter_record(h, full: bool = False):
    ns, mv = ctypes.c_int32(), ctypes.c_int64()
    _check(load().chase_filter_record(h, 0, None, ctypes.byref(ns), ctypes.byref(mv)), "chase_filter_record")
    rec = (chase_step_record_t * max(1, ns.value))()
    _check(load().chase_filter_record(h, ns.value, rec, ctypes.byref(ns), ctypes.byref(mv)), "chase_filter_record")
    return _records(ns.value, rec, full), mv.value


def chase_filter_schedule(N: int, p: int, q: int, myrow: int, mycol: int, degrees, full: bool = False):
    arr, dp = _i32_array(degrees)
    ns, mv = ctypes.c_int32(), ctypes.c_int64()
    _check(load().chase_filter_schedule(N, p, q, myrow, mycol, arr.shape[0], dp, 0, None,
                                        ctypes.byref(ns), ctypes.byref(mv)), "chase_filter_schedule")
    rec = (chase_step_record_t * max(1, ns.value))()
    _check(load().chase_filter_schedule(N, p, q, myrow, mycol, arr.shape[0], dp, ns.value, rec,
                                        ctypes.byref(ns), ctypes.byref(mv)), "chase_filter_schedule")
    return _records(ns.value, rec, full), mv.value


def chase_cholqr(h, V, cond_est: float, ncols: int | None = None, raise_on_error: bool = True):
    """1D-CAQR (Alg.4) in place on V.  Returns dict(status, variant, passes, info)."""
    v_ptr, ldv = _colmajor(V, "V")
    ncols = V.shape[1] if ncols is None else ncols
    st = chase_stats_t()
    info = ctypes.c_int32()
    s = load().chase_cholqr(h, v_ptr, ldv, ncols, float(cond_est), ctypes.byref(st), ctypes.byref(info))
    if raise_on_error:
        _check(s, "chase_cholqr")
    return {"status": s, "variant": st.qr_variant, "passes": st.qr_passes, "info": info.value,
            "shift": st.shift}


def chase_hhqr(h, V, ncols: int | None = None):
    """Householder QR (Alg.4 l.9) in place on V: V <- Q with diag(R) >= 0."""
    v_ptr, ldv = _colmajor(V, "V")
    ncols = V.shape[1] if ncols is None else ncols
    _check(load().chase_hhqr(h, v_ptr, ldv, ncols), "chase_hhqr")


def chase_set_qr_mode(h, mode: int):
    """0: Alg.4 dispatch; 1: Householder QR in every chase_cholqr call."""
    _check(load().chase_set_qr_mode(h, int(mode)), "chase_set_qr_mode")


def chase_residuals(h, A_local, V, ritz, ncols: int | None = None):
    """Residual norms ||A v_j - ritz_j v_j|| (Alg.2 l.23-28) of the columns of V."""
    a_ptr, lda = _colmajor(A_local, "A_local")
    v_ptr, ldv = _colmajor(V, "V")
    ncols = V.shape[1] if ncols is None else ncols
    r = np.ascontiguousarray(np.asarray(ritz, dtype=np.float64)[:ncols])
    out = np.empty(ncols, dtype=np.float64)
    _check(load().chase_residuals(h, a_ptr, lda, v_ptr, ldv, ncols,
                                  r.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                  out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))), "chase_residuals")
    return out


def chase_rayleigh_ritz(h, A_local, V, ncols: int | None = None):
    """Rayleigh-Ritz (Alg.2 l.16-22) in place on V; returns (ritz values ascending, sweeps)."""
    a_ptr, lda = _colmajor(A_local, "A_local")
    v_ptr, ldv = _colmajor(V, "V")
    ncols = V.shape[1] if ncols is None else ncols
    out = np.empty(ncols, dtype=np.float64)
    sw = ctypes.c_int32()
    _check(load().chase_rayleigh_ritz(h, a_ptr, lda, v_ptr, ldv, ncols,
                                      out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                      ctypes.byref(sw)), "chase_rayleigh_ritz")
    return out, sw.value


def chase_solve(h, A_local, V, nev: int, nex: int, tol: float = 1e-10, deg: int = 20,
                deg_max: int = 36, max_iter: int = 25, opt: bool = True, seed: int = 0,
                init_random: bool = True, raise_on_error: bool = True):
    """Full ChASE iteration (Alg.2).  V: C-layout n_r x (nev+nex) device block (in: initial
    vectors unless init_random; out: eigenvectors).  Returns dict(status, lambda, resid, stats)."""
    a_ptr, lda = _colmajor(A_local, "A_local")
    v_ptr, ldv = _colmajor(V, "V")
    ne = nev + nex
    lam = np.empty(ne, dtype=np.float64)
    res = np.empty(ne, dtype=np.float64)
    st = chase_solve_stats_t()
    s = load().chase_solve(h, a_ptr, lda, v_ptr, ldv, nev, nex, float(tol), deg, deg_max, max_iter,
                           1 if opt else 0, seed, 1 if init_random else 0,
                           lam.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                           res.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(st))
    if raise_on_error and s not in (0, 9):
        _check(s, "chase_solve")
    return {"status": s, "lambda": lam, "resid": res,
            "stats": {"matvecs": st.matvecs, "iterations": st.iterations, "locked": st.locked,
                      "b_sup": st.b_sup, "mu_1": st.mu_1, "mu_ne": st.mu_ne}}


def chase_cond_est(ritz, c: float, e: float, degrees, locked: int = 0) -> float:
    """Alg.5 over the n = len(degrees) vectors; ritz needs at least n values (ascending)."""
    r = np.ascontiguousarray(np.asarray(ritz, dtype=np.float64))
    arr, dp = _i32_array(degrees)
    n = arr.shape[0]
    if r.shape[0] < n:
        raise ValueError("need at least len(degrees) Ritz values")
    return load().chase_cond_est(r.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n,
                                 float(c), float(e), dp, int(locked))


def chase_shift_value(m: int, n: int, norm: float) -> float:
    return load().chase_shift_value(m, n, float(norm))


def chase_profile_enable(h, enable: bool = True):
    _check(load().chase_profile_enable(h, 1 if enable else 0), "chase_profile_enable")


def chase_profile_read(h):
    ms = (ctypes.c_double * 8)()
    ln = (ctypes.c_int64 * 8)()
    _check(load().chase_profile_read(h, ms, ln), "chase_profile_read")
    ms_d = {k: ms[i] for i, k in enumerate(PROFILE_CATEGORIES)}
    ln_d = {k: ln[i] for i, k in enumerate(PROFILE_CATEGORIES)}
    ms_d["hemm"] = ms_d["hemm_odd"] + ms_d["hemm_even"]
    ln_d["hemm"] = ln_d["hemm_odd"] + ln_d["hemm_even"]
    return ms_d, ln_d


def chase_destroy(h):
    _check(load().chase_destroy(h), "chase_destroy")


def chase_status_string(s: int) -> str:
    return _status_string(s)


# ------------------------------------------------------------------------------ convenience
class Chase:
    """One handle + its torch-owned workspace (a rank of the p x q grid, one GPU)."""

    def __init__(self, dtype: int, N: int, n_max: int, p: int = 1, q: int = 1, myrow: int = 0,
                 mycol: int = 0, uid: bytes | None = None, device: int = 0, stream=None, nb: int = 0,
                 virtual: bool = False):
        import torch
        self.device = torch.device("cuda", device)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.stream = s
        self.h = chase_create(dtype, N, n_max, p, q, myrow, mycol, uid, device, s.cuda_stream, nb,
                              virtual)
        self.n_r, self.n_c, self.r0, self.c0 = chase_local_dims(self.h)
        self.rows, self.cols = chase_local_indices(self.h, self.n_r, self.n_c)
        nbytes = chase_workspace_size(self.h)
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        chase_set_workspace(self.h, self.ws)
        self.dtype, self.N, self.n_max, self.p, self.q, self.nb = dtype, N, n_max, p, q, nb

    def filter(self, A_local, V, degrees, c, e, bounds, ncols=None):
        return chase_filter(self.h, A_local, V, degrees, c, e, bounds, ncols)

    def filter_step(self, A_local, X, Y, odd, alpha, beta, c, use_beta, k=None):
        return chase_filter_step(self.h, A_local, X, Y, odd, alpha, beta, c, use_beta, k)

    def cholqr(self, V, cond_est, ncols=None, raise_on_error=True):
        return chase_cholqr(self.h, V, cond_est, ncols, raise_on_error)

    def hhqr(self, V, ncols=None):
        return chase_hhqr(self.h, V, ncols)

    def set_qr_mode(self, mode):
        return chase_set_qr_mode(self.h, mode)

    def solve(self, A_local, V, nev, nex, **kw):
        return chase_solve(self.h, A_local, V, nev, nex, **kw)

    def rayleigh_ritz(self, A_local, V, ncols=None):
        return chase_rayleigh_ritz(self.h, A_local, V, ncols)

    def residuals(self, A_local, V, ritz, ncols=None):
        return chase_residuals(self.h, A_local, V, ritz, ncols)

    def record(self):
        return chase_filter_record(self.h)

    def close(self):
        if self.h is not None:
            chase_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
