"""torchrun worker for test_gpu_multi.test_spmd_check: with CHASE_SPMD_CHECK=1, a chase_filter
call whose degrees differ on one rank returns CHASE_EINVAL on every rank (no hang, V untouched);
identical arguments pass.  argv: out.json"""
import json
import os
import sys

os.environ["CHASE_SPMD_CHECK"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import torch.distributed as dist

import chase_inputs as ci
import paper_2309_15595_b200 as cb
from paper_2309_15595_b200 import dist as cdist


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    p, q = cdist.grid_shape(world)
    N, n = 256, 8
    uid = cdist.share_unique_id(cb.chase_get_unique_id)
    h = cb.Chase(cb.CHASE_C128, N, n, p, q, rank // q, rank % q, uid, local)
    lam = ci.uniform_spectrum(N)
    A = ci.dense_from_spectrum(lam, 3, True)
    b = ci.bounds_from_spectrum(lam, n)
    A_loc = torch.from_numpy(np.ascontiguousarray(A[h.r0:h.r0 + h.n_r, h.c0:h.c0 + h.n_c].T)).cuda().T
    V0 = ci.gaussian_block(N, n, 4, True)[h.r0:h.r0 + h.n_r]
    V = torch.from_numpy(np.ascontiguousarray(V0.T)).cuda().T
    res = {}
    degs = [4] * n if rank != 1 else [6] * n                     # rank 1 disagrees
    try:
        h.filter(A_loc, V, degs, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))
        res["mismatch_status"] = 0
    except cb.ChaseError as exc:
        res["mismatch_status"] = exc.status
    torch.cuda.synchronize()
    res["untouched"] = bool(np.array_equal(V.T.cpu().numpy().T, V0))
    h.filter(A_loc, V, [4] * n, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))   # agreeing call: fine
    res["agree_status"] = 0
    g = [None] * world
    dist.all_gather_object(g, res)
    if rank == 0:
        json.dump(g, open(sys.argv[1], "w"))
    h.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
