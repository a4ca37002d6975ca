"""Single-GPU coverage of the 2D-distributed filter and the fused compute+collective kernels
(P:146-149), so the driver's 1-GPU test box runs them:

* fused self mode (chase_set_fused_mode(h, 1)): a 1x1 grid whose every filter step runs
  zgemm_fused_kernel / dgemm_fused_kernel through the push/owner/broadcast protocol with m = 1;
* virtual grids (chase_create_virtual): all p*q ranks of a 2x1 / 1x2 / 2x2 / 1x4 / 2x4 grid
  (block and block-cyclic; 2x4 is BASELINE's 8-GPU grid) live in this process on one GPU, each on its own stream and host thread,
  with their fused regions peer-mapped to each other (same device), so the fused kernels run
  their multi-member protocol (m = 2 and 4) -- results equal to the global oracle, replicas
  bitwise identical;
* chase_filter_step: one rank's partial of one filter step (no reduction) with explicit bands
  (band_shift != 0 on off-diagonal ranks, empty bands) and use_beta = 0 / 1, against
  oracle.step_partial (readings #6, #7).
"""
import threading

import numpy as np
import pytest

import chase_inputs as ci
import oracle
import paper_2309_15595_b200 as cb
from gpu_util import colwise_rel, dev, host

pytestmark = pytest.mark.gpu
TOL = 1e-10
RAGGED = [2, 2, 4, 4, 4, 6, 8, 8, 10, 10, 12, 12, 12, 14, 16, 18, 20]


def problem(N, degs, complex_, seed):
    lam = ci.uniform_spectrum(N)
    A = ci.dense_from_spectrum(lam, seed, complex_)
    V0 = ci.gaussian_block(N, len(degs), seed + 1000, complex_)
    b = ci.bounds_from_spectrum(lam, len(degs))
    return A, V0, b


def num_sms():
    import torch
    return torch.cuda.get_device_properties(0).multi_processor_count


@pytest.mark.parametrize("complex_", [True, False])
@pytest.mark.parametrize("N,degs", [(300, sorted(RAGGED * 3)), (512, [20] * 60), (200, [2] * 5 + [36] * 9)])
def test_fused_self_mode_matches_oracle(complex_, N, degs):
    """1x1 grid, world = 1, peer_bases[0] = local, mode 1: every step is one fused kernel."""
    import torch
    A, V0, b = problem(N, degs, complex_, N + 7)
    ref, _ = oracle.chebyshev_filter(A, V0, degs, b.c, b.e, b.mu_1)
    h = cb.Chase(cb.CHASE_C128 if complex_ else cb.CHASE_R64, N, len(degs))
    region = torch.empty(cb.chase_fused_workspace_size(h.h), dtype=torch.uint8, device="cuda")
    cb.chase_set_fused_workspace(h.h, region.data_ptr(), [region.data_ptr()])
    cb.chase_set_fused_mode(h.h, 1)
    outs = []
    for _ in range(2):
        Vd = dev(V0)
        st = h.filter(dev(A), Vd, degs, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))
        torch.cuda.synchronize()
        outs.append(host(Vd))
    assert st["matvecs"] == sum(degs)
    assert colwise_rel(outs[0], ref) <= TOL
    assert np.array_equal(outs[0], outs[1])                    # deterministic repeat
    h.close()


def run_virtual(A, V0, degs, b, p, q, nb, complex_, budget=None):
    """All ranks of a p x q grid in this process; returns per-rank V outputs and handles' rows."""
    import torch
    N, n = V0.shape
    dt = cb.CHASE_C128 if complex_ else cb.CHASE_R64
    world = p * q
    budget = budget or num_sms() // world
    hs = []
    for r in range(world):
        i, j = divmod(r, q)
        hs.append(cb.Chase(dt, N, n, p, q, i, j, None, 0, torch.cuda.Stream(), nb=nb, virtual=True))
    size = cb.chase_fused_workspace_size(hs[0].h)
    assert all(cb.chase_fused_workspace_size(h.h) == size for h in hs)
    regions = [torch.empty(size, dtype=torch.uint8, device="cuda") for _ in hs]
    ptrs = [t.data_ptr() for t in regions]
    for h, t in zip(hs, regions):
        cb.chase_set_fused_workspace(h.h, t.data_ptr(), ptrs)
        cb.chase_set_fused_mode(h.h, 0, budget)
    A_loc = [dev(np.ascontiguousarray(A[np.ix_(h.rows, h.cols)])) for h in hs]
    torch.cuda.synchronize()
    outs, errs = [None] * world, [None] * world
    for rep in range(2):
        V_loc = [dev(np.ascontiguousarray(V0[h.rows])) for h in hs]
        torch.cuda.synchronize()

        def work(r):
            try:
                hs[r].filter(A_loc[r], V_loc[r], degs, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))
                hs[r].stream.synchronize()
            except Exception as exc:          # reported by the main thread
                errs[r] = exc

        th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join(120)
        assert not any(t.is_alive() for t in th), "virtual-grid filter hung"
        assert all(e is None for e in errs), errs
        res = [host(v) for v in V_loc]
        if rep == 0:
            outs = res
        else:
            assert all(np.array_equal(a, c) for a, c in zip(outs, res)), "not bitwise repeatable"
    recs = [h.record() for h in hs]
    rows = [h.rows for h in hs]
    for h in hs:
        h.close()
    return outs, rows, recs


@pytest.mark.parametrize("complex_", [True, False])
@pytest.mark.parametrize("grid,nb", [((2, 1), 0), ((1, 2), 0), ((2, 2), 0), ((1, 4), 0), ((2, 2), 16),
                                     ((2, 1), 7), ((2, 4), 0), ((2, 4), 9)])
def test_virtual_grid_fused_matches_oracle(complex_, grid, nb):
    """Fused multi-member kernels (m = p on odd steps, m = q on even steps) on one GPU."""
    p, q = grid
    N = 301
    degs = sorted(RAGGED * 3)
    A, V0, b = problem(N, degs, complex_, 77)
    ref, _ = oracle.chebyshev_filter(A, V0, degs, b.c, b.e, b.mu_1)
    outs, rows, recs = run_virtual(A, V0, degs, b, p, q, nb, complex_)
    for r, (V, ri) in enumerate(zip(outs, rows)):
        assert colwise_rel(V, ref[ri]) <= TOL, f"rank {r}"
    for i in range(p):                                            # row replicas: identical bits
        for j in range(1, q):
            assert np.array_equal(outs[i * q], outs[i * q + j])
    for r, (rec, mv) in enumerate(recs):
        i, j = divmod(r, q)
        n_r, n_c = len(rows[i * q]), len(oracle.grid._owned(N, q, j, nb))
        orec, omv = oracle.filter_record(degs, n_r, n_c)
        assert [x[:4] for x in rec] == orec and mv == omv


@pytest.mark.parametrize("complex_", [True, False])
@pytest.mark.parametrize("grid,nb,N,budget", [((2, 1), 0, 301, 2), ((2, 2), 0, 301, 2), ((1, 4), 0, 301, 2),
                                              ((2, 2), 16, 301, 2), ((2, 1), 0, 700, 4), ((2, 4), 9, 700, 2)])
def test_virtual_grid_fused_tail_matches_oracle(complex_, grid, nb, N, budget):
    """A small persistent grid (sm_budget CTAs) leaves a partial last round on most steps, so the
    fused step runs T_main tiles in the fused kernel and the rest as split-K copies reduced
    through the tail slots (fused_tail.cuh): result = oracle, replicas bitwise identical, bitwise
    repeatable (run_virtual runs twice)."""
    p, q = grid
    degs = sorted(RAGGED * 3)
    A, V0, b = problem(N, degs, complex_, 79)
    ref, _ = oracle.chebyshev_filter(A, V0, degs, b.c, b.e, b.mu_1)
    outs, rows, _ = run_virtual(A, V0, degs, b, p, q, nb, complex_, budget=budget)
    for r, (V, ri) in enumerate(zip(outs, rows)):
        assert colwise_rel(V, ref[ri]) <= TOL, f"rank {r}"
    for i in range(p):
        for j in range(1, q):
            assert np.array_equal(outs[i * q], outs[i * q + j])


@pytest.mark.parametrize("complex_", [True, False])
@pytest.mark.parametrize("grid,budget", [((2, 1), 5), ((2, 2), 3), ((1, 2), 5)])
def test_virtual_grid_fused_tail_wide_and_narrow(complex_, grid, budget):
    """Ragged width: one wide-tile and one narrow-tile launch per step (k = 84 complex: 64 + 20
    columns; k = 140 real: 128 + 12), each with a split-K tail on 16 m-tiles over a 3- or 5-CTA
    grid -- both launches' tails share the step's tail slot (wide and narrow tiles, one place
    each)."""
    p, q = grid
    N = 2000
    degs = [6] * (84 if complex_ else 140)
    A, V0, b = problem(N, degs, complex_, 83)
    ref, _ = oracle.chebyshev_filter(A, V0, degs, b.c, b.e, b.mu_1)
    outs, rows, _ = run_virtual(A, V0, degs, b, p, q, 0, complex_, budget=budget)
    for r, (V, ri) in enumerate(zip(outs, rows)):
        assert colwise_rel(V, ref[ri]) <= TOL, f"rank {r}"


@pytest.mark.parametrize("complex_", [True, False])
def test_fused_self_mode_tail_matches_oracle(complex_):
    """1x1 fused self mode with a 3-CTA persistent grid: the tail path with m = 1."""
    import torch
    N, degs = 520, sorted(RAGGED * 3)
    A, V0, b = problem(N, degs, complex_, 81)
    ref, _ = oracle.chebyshev_filter(A, V0, degs, b.c, b.e, b.mu_1)
    h = cb.Chase(cb.CHASE_C128 if complex_ else cb.CHASE_R64, N, len(degs))
    region = torch.empty(cb.chase_fused_workspace_size(h.h), dtype=torch.uint8, device="cuda")
    cb.chase_set_fused_workspace(h.h, region.data_ptr(), [region.data_ptr()])
    cb.chase_set_fused_mode(h.h, 1, 3)
    Vd = dev(V0)
    h.filter(dev(A), Vd, degs, b.c, b.e, (b.mu_1, b.mu_ne, b.b_sup))
    torch.cuda.synchronize()
    assert colwise_rel(host(Vd), ref) <= TOL
    h.close()


@pytest.mark.parametrize("complex_", [True, False])
@pytest.mark.parametrize("grid,nb", [((2, 2), 0), ((3, 2), 0), ((2, 3), 0), ((2, 2), 8), ((3, 2), 5)])
@pytest.mark.parametrize("odd", [True, False])
def test_filter_step_partials_match_oracle(complex_, grid, nb, odd):
    """Per-rank partial of one step, every rank of the grid, use_beta 0 and 1: the epilogue's
    band (including band_shift != 0 and empty bands on off-diagonal ranks) and beta term."""
    import torch
    p, q = grid
    N, k = 203, 70
    rng = np.random.default_rng(11)
    A = ci.dense_from_spectrum(ci.uniform_spectrum(N), 12, complex_)
    cplx = lambda *s: rng.standard_normal(s) + (1j * rng.standard_normal(s) if complex_ else 0)
    X, Y = cplx(N, k), cplx(N, k)
    alpha, beta, c = 1.3, -0.7, 0.45
    dt = cb.CHASE_C128 if complex_ else cb.CHASE_R64
    for r in range(p * q):
        i, j = divmod(r, q)
        h = cb.Chase(dt, N, k, p, q, i, j, None, 0, nb=nb, virtual=True)
        in_rows = h.rows if odd else h.cols
        out_rows = h.cols if odd else h.rows
        for use_beta in (False, True):
            Xd = dev(np.ascontiguousarray(X[in_rows]))
            Yd = dev(np.ascontiguousarray(Y[out_rows]), ld=len(out_rows) + 3)
            h.filter_step(dev(A[np.ix_(h.rows, h.cols)]), Xd, Yd, odd, alpha, beta, c, use_beta)
            torch.cuda.synchronize()
            ref = oracle.step_partial(A, X[in_rows], Y[out_rows], i, j, p, q, odd, alpha, beta, c,
                                      use_beta, nb)
            assert colwise_rel(host(Yd), ref) <= 1e-13, (r, use_beta)
        h.close()


def test_virtual_grid_refuses_nccl_calls():
    """A virtual 2x1 grid has no communicators: collective calls other than the fused filter
    return CHASE_ESTATE instead of touching NCCL."""
    N, n = 64, 4
    h = cb.Chase(cb.CHASE_C128, N, n, 2, 1, 0, 0, None, 0, virtual=True)
    V = dev(np.ones((h.n_r, n), dtype=np.complex128))
    A = dev(np.ones((h.n_r, h.n_c), dtype=np.complex128))
    with pytest.raises(cb.ChaseError) as ei:
        h.filter(A, V, [2] * n, 0.5, 0.5, (-1.0, 0.0, 1.0))      # no fused workspace
    assert ei.value.status == 8
    assert h.cholqr(V, 1e3, raise_on_error=False)["status"] == 8
    with pytest.raises(cb.ChaseError) as ei:
        h.residuals(A, V, [0.0] * n)
    assert ei.value.status == 8
    h.close()
