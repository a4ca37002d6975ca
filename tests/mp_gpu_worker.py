"""torchrun worker for tests/test_gpu_multi.py: one rank per GPU, p x q grid, NCCL (or fused
peer-memory reduction).  Runs chase_filter (twice: bitwise repeat check), chase_cholqr, chase_hhqr,
chase_residuals, chase_rayleigh_ritz through the C-ABI on a seeded problem and writes the gathered result to
<out>.npz on rank 0.
argv: p q N c|r out [pad] [nccl|fused] [nb]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import torch.distributed as dist

import chase_inputs as ci
import paper_2309_15595_b200 as cb
from paper_2309_15595_b200 import dist as cdist


def main():
    p, q, N, complex_, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4] == "c", sys.argv[5]
    pad = int(sys.argv[6]) if len(sys.argv) > 6 else 0        # extra leading-dimension rows
    fused = len(sys.argv) > 7 and sys.argv[7] == "fused"      # fused HEMM + NVLink reduction
    nb = int(sys.argv[8]) if len(sys.argv) > 8 else 0         # block-cyclic block size (0: block)
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    assert world == p * q
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    myrow, mycol = cdist.grid_coords(rank, p, q)
    uid = cdist.share_unique_id(cb.chase_get_unique_id)
    degs = sorted([2, 2, 4, 4, 4, 6, 8, 8, 10, 10, 12, 12, 12, 14, 16, 18, 20] * 3)
    n = len(degs)
    lam = ci.uniform_spectrum(N)
    A = ci.dense_from_spectrum(lam, 77, complex_)
    V0 = ci.gaussian_block(N, n, 78, complex_)
    b = ci.bounds_from_spectrum(lam, n)
    h = cb.Chase(cb.CHASE_C128 if complex_ else cb.CHASE_R64, N, n, p, q, myrow, mycol, uid, local, nb=nb)
    n_r, n_c = h.n_r, h.n_c
    rows, cols = h.rows, h.cols
    dt = A.dtype
    if fused:
        cdist.enable_fused_comm(h)

    def dev(a):
        nrow, ncol = a.shape
        ld = nrow + pad
        ld += (ld % 2 if not complex_ else 0)
        buf = np.zeros((ncol, ld), dtype=dt)
        buf[:, :nrow] = a.T
        return torch.from_numpy(buf).cuda().T[:nrow]

    Ad = dev(A[np.ix_(rows, cols)])
    Vd = dev(V0[rows])
    V2 = dev(V0[rows])
    st = h.filter(Ad, Vd, degs, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))
    h.filter(Ad, V2, degs, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))     # repeat: same bits
    torch.cuda.synchronize()
    repeat_equal = bool(torch.equal(Vd, V2))
    rec, mv = h.record()
    Vf = Vd.T.cpu().numpy().T.copy()
    est = cb.chase_cond_est(lam, b.c, b.e, degs, 0)
    # Householder QR (Alg.4 l.9 fallback) of the filtered block over the column comm
    Vh = dev(Vf)
    h.hhqr(Vh)
    torch.cuda.synchronize()
    Hq = Vh.T.cpu().numpy().T.copy()
    qr = h.cholqr(Vd, est, raise_on_error=False)
    torch.cuda.synchronize()
    Q = Vd.T.cpu().numpy().T.copy()
    # residuals (Alg.2 l.23-28) of the orthonormal columns with Rayleigh-quotient values
    qs = [None] * world
    dist.all_gather_object(qs, (mycol, rows, Q))
    Qg = np.zeros((N, n), dtype=dt)
    for (j_, rr, qq) in qs:
        if j_ == 0:
            Qg[rr] = qq
    obj = [np.real(np.einsum("ij,ij->j", Qg.conj(), A @ Qg)) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ritz = obj[0]
    resid = h.residuals(Ad, Vd, ritz)
    # Rayleigh-Ritz (Alg.2 l.16-22) on the orthonormal Q
    theta, _ = h.rayleigh_ritz(Ad, Vd)
    torch.cuda.synchronize()
    Xr = Vd.T.cpu().numpy().T.copy()
    g = [None] * world
    dist.all_gather_object(g, (rank, myrow, mycol, rows, n_r, n_c, Vf, Q, rec, mv, qr, resid, ritz, repeat_equal,
                               theta, Xr, Hq))
    if rank == 0:
        Vfull = np.zeros((N, n), dtype=dt)
        Qfull = np.zeros((N, n), dtype=dt)
        Xfull = np.zeros((N, n), dtype=dt)
        Hfull = np.zeros((N, n), dtype=dt)
        replica = 0.0
        for x in g:
            if x[2] == 0:
                Vfull[x[3]] = x[6]
                Qfull[x[3]] = x[7]
                Xfull[x[3]] = x[15]
                Hfull[x[3]] = x[16]
        for x in g:
            replica = max(replica, float(np.max(np.abs(x[6] - Vfull[x[3]]))),
                          float(np.max(np.abs(x[7] - Qfull[x[3]]))),
                          float(np.max(np.abs(x[15] - Xfull[x[3]]))),
                          float(np.max(np.abs(x[16] - Hfull[x[3]]))))
        np.savez(out, V=Vfull, Q=Qfull, replica=replica, est=est,
                 variants=np.array([x[10]["variant"] for x in g]), passes=np.array([x[10]["passes"] for x in g]),
                 status=np.array([x[10]["status"] for x in g]), mv=np.array([x[9] for x in g]),
                 recs=np.array([str(x[8]) for x in g]), ranks=np.array([[x[1], x[2], x[4], x[5]] for x in g]),
                 resid=np.array([x[11] for x in g]), ritz=g[0][12],
                 repeat_equal=np.array([x[13] for x in g]), X=Xfull, H=Hfull,
                 theta=np.array([x[14] for x in g]))
    h.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
