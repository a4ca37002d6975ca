"""Multi-process (world size 2, gloo, CPU) tests of the N > 1 host path: unique-id sharing,
per-rank geometry and the library's per-rank schedule (active widths, message sizes, the band
of -cI each rank owns and the rank that adds the beta term).  The schedule is then executed by
real processes with numpy HEMMs and gloo AllReduce (SUM) and compared with the global oracle:
this pins that the bands/beta roles chase_filter launches reproduce Eq.(1) on a 2D grid."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, grid, out_q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import chase_inputs as ci
    import oracle
    import paper_2309_15595_b200 as cb
    from paper_2309_15595_b200 import dist as cdist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, q = grid
        myrow, mycol = cdist.grid_coords(rank, p, q)
        uid = cdist.share_unique_id(cb.chase_get_unique_id)
        N = 61
        degs = [2, 2, 4, 4, 4, 6, 8, 8, 10, 10, 12, 12, 12, 14, 16, 18, 20]
        n = len(degs)
        n_r, n_c, r0, c0 = cb.chase_block_dims(N, p, q, myrow, mycol)
        rec, mv = cb.chase_filter_schedule(N, p, q, myrow, mycol, degs, full=True)

        # execute the schedule with numpy HEMMs + gloo AllReduce over row / column groups
        lam = ci.uniform_spectrum(N)
        A = ci.dense_from_spectrum(lam, 41, True)
        V0 = ci.gaussian_block(N, n, 42, True)
        b = ci.bounds_from_spectrum(lam, n)
        alpha, beta, _ = oracle.chebyshev_scalars(b.c, b.e, b.mu_1, max(degs))
        rows = [dist.new_group([i * q + j for j in range(q)]) for i in range(p)]   # rcomm
        cols = [dist.new_group([i * q + j for i in range(p)]) for j in range(q)]   # ccomm
        Aij = A[r0:r0 + n_r, c0:c0 + n_c]
        C = V0[r0:r0 + n_r].copy()
        B = np.full((n_c, n), np.nan, dtype=np.complex128)     # never read before written
        for s, (k, off, comm, elems, use_beta, blo, bhi) in enumerate(rec, start=1):
            if comm == "col":
                part = Aij.conj().T @ C[:, off:]
                part[blo:bhi] -= b.c * C[blo + c0 - r0:bhi + c0 - r0, off:]
                part = alpha[s - 1] * part
                if use_beta:
                    part = part + beta[s - 1] * B[:, off:]
                t = torch.from_numpy(np.ascontiguousarray(part))
                dist.all_reduce(t, group=cols[mycol])
                B[:, off:] = t.numpy()
                assert elems == n_c * k
            else:
                part = Aij @ B[:, off:]
                part[blo:bhi] -= b.c * B[blo + r0 - c0:bhi + r0 - c0, off:]
                part = alpha[s - 1] * part
                if use_beta:
                    part = part + beta[s - 1] * C[:, off:]
                t = torch.from_numpy(np.ascontiguousarray(part))
                dist.all_reduce(t, group=rows[myrow])
                C[:, off:] = t.numpy()
                assert elems == n_r * k
        gathered = [None] * world
        dist.all_gather_object(gathered, (rank, myrow, mycol, (n_r, n_c, r0, c0), rec, mv, uid, C))
        if rank == 0:
            out_q.put(gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("grid", [(2, 1), (1, 2)])
def test_two_process_grid(grid):
    import oracle
    import chase_inputs as ci

    world = 2
    ctx = mp.get_context("spawn")
    q_ = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, grid, q_)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = q_.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p, q = grid
    N, degs = 61, [2, 2, 4, 4, 4, 6, 8, 8, 10, 10, 12, 12, 12, 14, 16, 18, 20]
    # unique id identical on every rank
    assert len({r[6] for r in res}) == 1 and len(res[0][6]) == 128
    # blocks tile the matrix exactly
    cover = np.zeros((N, N), dtype=int)
    for (_, i, j, (n_r, n_c, r0, c0), *_r) in res:
        cover[r0:r0 + n_r, c0:c0 + n_c] += 1
    assert np.all(cover == 1)
    # per step: in every reducing communicator the bands cover the owned diagonal rows once
    # and exactly one rank adds beta (none at step 1)
    D = max(degs)
    for s in range(1, D + 1):
        if s % 2 == 1:
            groups = {}
            for (_, i, j, geo, rec, *_r) in res:
                groups.setdefault(j, []).append((geo, rec[s - 1]))
            for j, members in groups.items():
                n_c, c0 = members[0][0][1], members[0][0][3]
                hit = np.zeros(n_c, dtype=int)
                for (geo, r) in members:
                    hit[r[5]:r[6]] += 1
                assert np.all(hit == 1)
                assert sum(r[4] for (_, r) in members) == (0 if s == 1 else 1)
        else:
            groups = {}
            for (_, i, j, geo, rec, *_r) in res:
                groups.setdefault(i, []).append((geo, rec[s - 1]))
            for i, members in groups.items():
                n_r = members[0][0][0]
                hit = np.zeros(n_r, dtype=int)
                for (geo, r) in members:
                    hit[r[5]:r[6]] += 1
                assert np.all(hit == 1)
                assert sum(r[4] for (_, r) in members) == 1
    # the executed schedule reproduces the global oracle
    lam = ci.uniform_spectrum(N)
    A = ci.dense_from_spectrum(lam, 41, True)
    V0 = ci.gaussian_block(N, len(degs), 42, True)
    b = ci.bounds_from_spectrum(lam, len(degs))
    ref, _ = oracle.chebyshev_filter(A, V0, degs, b.c, b.e, b.mu_1)
    for (_, i, j, (n_r, n_c, r0, c0), rec, mv, uid, C) in res:
        assert mv == sum(degs)
        assert np.linalg.norm(C - ref[r0:r0 + n_r]) <= 1e-13 * np.linalg.norm(ref[r0:r0 + n_r])
