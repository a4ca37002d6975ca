"""torchrun worker for tests/test_gpu_multi.py: one rank per GPU, p x q grid, NCCL.
Runs chase_filter and chase_cholqr through the C-ABI on a seeded problem and writes the
gathered result to <out>.npz on rank 0."""
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
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    assert world == p * q
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    myrow, mycol = cdist.grid_coords(rank, p, q)
    uid = cdist.share_unique_id(cb.chase_get_unique_id)
    degs = [2, 2, 4, 4, 4, 6, 8, 8, 10, 10, 12, 12, 12, 14, 16, 18, 20] * 3
    degs = sorted(degs)
    n = len(degs)
    lam = ci.uniform_spectrum(N)
    A = ci.dense_from_spectrum(lam, 77, complex_)
    V0 = ci.gaussian_block(N, n, 78, complex_)
    b = ci.bounds_from_spectrum(lam, n)
    h = cb.Chase(cb.CHASE_C128 if complex_ else cb.CHASE_R64, N, n, p, q, myrow, mycol, uid, local)
    n_r, n_c, r0, c0 = h.n_r, h.n_c, h.r0, h.c0
    dt = A.dtype
    if fused:
        cdist.enable_fused_comm(h)

    def dev(a):
        rows, cols = a.shape
        ld = rows + pad
        ld += (ld % 2 if not complex_ else 0)
        buf = np.zeros((cols, ld), dtype=dt)
        buf[:, :rows] = a.T
        return torch.from_numpy(buf).cuda().T[:rows]

    Ad = dev(A[r0:r0 + n_r, c0:c0 + n_c])
    Vd = dev(V0[r0:r0 + n_r])
    V2 = dev(V0[r0:r0 + n_r])
    st = h.filter(Ad, Vd, degs, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))
    h.filter(Ad, V2, degs, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))     # repeat: same bits
    torch.cuda.synchronize()
    repeat_equal = bool(torch.equal(Vd, V2))
    rec, mv = h.record()
    torch.cuda.synchronize()
    Vf = Vd.T.cpu().numpy().T.copy()
    est = cb.chase_cond_est(lam, b.c, b.e, degs, 0)
    qr = h.cholqr(Vd, est, raise_on_error=False)
    torch.cuda.synchronize()
    Q = Vd.T.cpu().numpy().T.copy()
    # residuals (Alg.2 l.23-28) of the orthonormal columns with Rayleigh-quotient values
    qs = [None] * world
    dist.all_gather_object(qs, (mycol, r0, n_r, Q))
    Qg = np.zeros((N, n), dtype=dt)
    for (j_, rr0, nr_, qq) in qs:
        if j_ == 0:
            Qg[rr0:rr0 + nr_] = qq
    obj = [np.real(np.einsum("ij,ij->j", Qg.conj(), A @ Qg)) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ritz = obj[0]
    resid = h.residuals(Ad, Vd, ritz)
    g = [None] * world
    dist.all_gather_object(g, (rank, myrow, mycol, r0, n_r, Vf, Q, rec, mv, qr, resid, ritz, repeat_equal))
    if rank == 0:
        Vfull = np.zeros((N, n), dtype=dt)
        Qfull = np.zeros((N, n), dtype=dt)
        replica = 0.0
        for (rk, i, j, rr0, nr, vf, qq, rc, m, qi, rs, rz, rq) in g:
            if j == 0:
                Vfull[rr0:rr0 + nr] = vf
                Qfull[rr0:rr0 + nr] = qq
        for (rk, i, j, rr0, nr, vf, qq, rc, m, qi, rs, rz, rq) in g:
            replica = max(replica, float(np.max(np.abs(vf - Vfull[rr0:rr0 + nr]))),
                          float(np.max(np.abs(qq - Qfull[rr0:rr0 + nr]))))
        np.savez(out, V=Vfull, Q=Qfull, replica=replica, est=est,
                 variants=np.array([x[9]["variant"] for x in g]), passes=np.array([x[9]["passes"] for x in g]),
                 status=np.array([x[9]["status"] for x in g]), mv=np.array([x[8] for x in g]),
                 recs=np.array([str(x[7]) for x in g]), ranks=np.array([[x[1], x[2], x[4]] for x in g]),
                 resid=np.array([x[10] for x in g]), ritz=g[0][11],
                 repeat_equal=np.array([x[12] for x in g]))
    h.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
