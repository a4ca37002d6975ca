"""Full-size (BASELINE.json configuration) parity run of the hot path on the launch
configuration bench.py uses, one rank per GPU (world 1 runs in-process; world > 1 under
torchrun).  Checks, on the same seeded inputs the bench uses:

* filter, all sampled columns: the FFT closed form p(A) V0 = Phi F g(mu) F^H Phi^H V0 of the
  DFT-phase / Hartley-sign matrices (a property at any size, pinned against the oracle at small N
  in tests/test_oracle_filter.py), relative error per column <= 1e-10;
* filter, columns 0 and n-1 against the oracle itself when the full A fits in host memory;
* CholeskyQR: orthogonality ||Q^H Q - I||_F <= 1e-12 of the distributed Q (Gram reduced over
  the column communicator) and the executed Alg.4 variant equal to the oracle's selection;
* bookkeeping: the per-rank record equals the oracle's record.

Usage (torchrun): python tests/full_worker.py CONFIG p q OUT.json [fused|nccl]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import chase_inputs as ci
import oracle
import paper_2309_15595_b200 as cb
from cheb_closed_form import dft_phase_closed_form, hartley_closed_form


def run_full(name, p, q, rank=0, local=0, dist=None, oracle_cols=True, mode="nccl"):
    cfg = ci.CONFIGS[name]
    N, n = cfg.N, cfg.n
    lam = cfg.spectrum_values()
    degrees = cfg.degrees()
    b = ci.bounds_from_spectrum(lam, n)
    myrow, mycol = rank // q, rank % q
    uid = None
    if dist is not None:
        from paper_2309_15595_b200 import dist as cdist
        uid = cdist.share_unique_id(cb.chase_get_unique_id)
    dev = torch.device("cuda", local)
    h = cb.Chase(cb.CHASE_C128 if cfg.complex_ else cb.CHASE_R64, N, n, p, q, myrow, mycol, uid, local)
    n_r, n_c, r0, c0 = h.n_r, h.n_c, h.r0, h.c0
    if mode == "fused" and dist is not None:
        from paper_2309_15595_b200 import dist as cdist
        cdist.enable_fused_comm(h)            # filter steps as fused HEMM + NVLink reduction
    gen = ci.dft_phase(lam, cfg.seed) if cfg.complex_ else ci.hartley_sign(lam, cfg.seed)
    A_t = gen.block(r0, n_r, c0, n_c, device=dev)
    V0 = ci.gaussian_block(N, n, cfg.seed + 1000, cfg.complex_)
    V_t = torch.from_numpy(np.ascontiguousarray(V0[r0:r0 + n_r].T)).to(dev)
    st = h.filter(A_t.T, V_t.T, degrees, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))
    rec, mv = h.record()
    torch.cuda.synchronize()
    Vf = V_t.cpu().numpy().T                                   # (n_r, n) of this rank
    res = {"config": name, "grid": f"{p}x{q}", "rank": rank, "mode": mode}

    # FFT closed form on a spread of columns
    cols = np.unique(np.linspace(0, n - 1, 48).astype(int))
    cf = dft_phase_closed_form if cfg.complex_ else hartley_closed_form
    ref = cf(gen, V0[:, cols], degrees[cols], b.c, b.e, b.mu_1)[r0:r0 + n_r]
    got = Vf[:, cols]
    res["closed_form_col_err"] = float(np.max(np.linalg.norm(got - ref, axis=0) / np.linalg.norm(ref, axis=0)))

    # oracle on two columns (full A on the host), single GPU only
    if oracle_cols and p * q == 1 and 16 * N * N < 100e9:
        torch.set_num_threads(len(os.sched_getaffinity(0)))
        A_host = A_t.cpu().numpy().T
        oc = [0, n - 1]
        o, _ = oracle.chebyshev_filter(A_host, np.asfortranarray(V0[:, oc]), [int(degrees[j]) for j in oc],
                                       b.c, b.e, b.mu_1)
        del A_host
        res["oracle_col_err"] = float(np.max(np.linalg.norm(Vf[:, oc] - o, axis=0) / np.linalg.norm(o, axis=0)))

    orec, omv = oracle.filter_record(list(degrees), n_r, n_c)
    res["record_equal"] = bool(rec == orec and mv == omv == st["matvecs"])

    # CholeskyQR on the filtered block
    est = cb.chase_cond_est(lam, b.c, b.e, degrees, 0)
    qr = h.cholqr(V_t.T, est)
    res["qr_variant"], res["qr_passes"] = qr["variant"], qr["passes"]
    res["oracle_variant"] = oracle.select_variant(oracle.cond_est(lam, b.c, b.e, degrees, 0))
    Q = V_t.T
    G = Q.conj().T @ Q                                          # test-side check (torch)
    if dist is not None and p > 1:
        groups = [dist.new_group([i * q + j for i in range(p)]) for j in range(q)]
        dist.all_reduce(G, group=groups[mycol])
    I = torch.eye(n, dtype=G.dtype, device=dev)
    res["orth"] = float(torch.linalg.norm(G - I).item())
    h.close()
    return res


def main():
    name, p, q, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    mode = sys.argv[5] if len(sys.argv) > 5 else "nccl"
    import torch.distributed as dist
    rank, local = int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    res = run_full(name, p, q, rank, local, dist, mode=mode)
    g = [None] * dist.get_world_size()
    dist.all_gather_object(g, res)
    if rank == 0:
        json.dump(g, open(out, "w"))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
