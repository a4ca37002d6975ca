"""torchrun worker: chase_solve (full Alg.2 loop) on a p x q grid; rank 0 writes eigenvalues,
residuals, stats and the gathered eigenvectors to <out>.npz.  argv: p q N nev nex out"""
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
    p, q, N, nev, nex, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), sys.argv[6]
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    myrow, mycol = cdist.grid_coords(rank, p, q)
    uid = cdist.share_unique_id(cb.chase_get_unique_id)
    lam = ci.uniform_spectrum(N)
    A = ci.dense_from_spectrum(lam, 21, True)
    h = cb.Chase(cb.CHASE_C128, N, nev + nex, p, q, myrow, mycol, uid, local)
    rows, cols = h.rows, h.cols
    Ad = torch.from_numpy(np.ascontiguousarray(A[np.ix_(rows, cols)].T)).cuda().T
    Vd = torch.zeros((nev + nex, len(rows)), dtype=torch.complex128, device="cuda").T
    res = h.solve(Ad, Vd, nev, nex, tol=1e-10, seed=7)
    torch.cuda.synchronize()
    g = [None] * world
    dist.all_gather_object(g, (mycol, rows, Vd.T.cpu().numpy().T.copy(), res))
    if rank == 0:
        X = np.zeros((N, nev + nex), dtype=np.complex128)
        for (j, rr, v, _) in g:
            if j == 0:
                X[rr] = v
        np.savez(out, X=X, lam=res["lambda"], resid=res["resid"], status=res["status"],
                 iters=res["stats"]["iterations"], matvecs=res["stats"]["matvecs"],
                 same=all(np.array_equal(x[3]["lambda"], res["lambda"]) for x in g))
    h.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
