"""libchase.so loads on a CPU-only box and exports every entry point include/chase.h declares;
its pure host functions (schedule, block geometry, Alg.5, Alg.4 shift) agree bit-exactly with
the oracle / SPEC hand values.  No device work is issued here."""
import math
import os
import re

import numpy as np
import pytest

import chase_inputs as ci
import oracle
import paper_2309_15595_b200 as cb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "chase.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(chase_[a-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = cb.load()
    syms = header_symbols()
    assert len(syms) >= 15
    assert sorted(cb.EXPORTED) == syms
    for s in syms:
        assert hasattr(lib, s), s


def test_status_strings():
    assert cb.chase_status_string(0) == "CHASE_OK"
    assert cb.chase_status_string(2).startswith("CHASE_EDEGREE")


@pytest.mark.parametrize("N,p,q", [(10, 3, 4), (61, 2, 3), (512, 1, 1), (120000, 2, 4)])
def test_block_dims_match_generator(N, p, q):
    for i in range(p):
        for j in range(q):
            assert cb.chase_block_dims(N, p, q, i, j) == ci.block_dims(N, p, q, i, j)


def test_block_dims_errors():
    with pytest.raises(cb.ChaseError):
        cb.chase_block_dims(10, 2, 2, 2, 0)


@pytest.mark.parametrize("degrees", [
    [2, 2, 4, 4, 4, 6, 8, 8, 10, 10, 12, 12, 12, 14, 16, 18, 20],
    [20] * 60,
    list(ci.ramp_degrees(250)),
])
@pytest.mark.parametrize("grid", [(1, 1), (2, 1), (2, 4)])
def test_schedule_bit_exact_vs_oracle(degrees, grid):
    N = 1001
    p, q = grid
    for i in range(p):
        for j in range(q):
            n_r, n_c, _, _ = ci.block_dims(N, p, q, i, j)
            rec, mv = cb.chase_filter_schedule(N, p, q, i, j, degrees)
            orec, omv = oracle.filter_record(degrees, n_r, n_c)
            assert mv == omv == sum(int(d) for d in degrees)
            assert rec == orec


@pytest.mark.parametrize("bad", [[2, 3], [0, 2], [4, 2]])
def test_schedule_rejects_bad_degrees(bad):
    with pytest.raises(cb.ChaseError) as ei:
        cb.chase_filter_schedule(100, 1, 1, 0, 0, bad)
    assert ei.value.status == 2


def test_cond_est_golden(golden):
    g = golden["cond_est_t3"]
    est = cb.chase_cond_est([g["t"], g["t"]], 0.0, 1.0, [g["d"], g["d"]], 0)
    ref = g["cond_a"] + g["cond_b_sqrt2"] * math.sqrt(2.0)
    assert abs(est - ref) <= 4e-15 * ref
    g = golden["cond_est_inside"]
    assert cb.chase_cond_est([g["tp"], g["t"]], 0.0, 1.0, [2, g["d"]], 1) == g["cond"]
    assert math.isnan(cb.chase_cond_est([1.0], 0.0, -1.0, [2], 0))


@pytest.mark.parametrize("seed", range(5))
def test_cond_est_matches_oracle(seed):
    rng = np.random.default_rng(seed)
    ritz = np.sort(rng.uniform(-3, 1, 12))
    degs = np.sort(rng.integers(1, 19, 12) * 2)
    locked = int(rng.integers(0, 11))
    a = cb.chase_cond_est(ritz, 0.3, 0.6, degs, locked)
    b = oracle.cond_est(ritz, 0.3, 0.6, degs, locked)
    assert abs(a - b) <= 1e-13 * b


def test_shift_value_golden(golden):
    g = golden["shift"]
    assert cb.chase_shift_value(g["m"], g["n"], g["norm"]) == g["s_over_u"] * 2.0 ** -53


@pytest.mark.parametrize("N,P,nb", [(10, 2, 4), (61, 3, 1), (301, 4, 7), (1000, 2, 64)])
def test_cyclic_indices_partition(N, P, nb):
    """chase_cyclic_indices: grid rows partition 0..N-1, blocks of nb dealt round-robin."""
    seen = np.concatenate([cb.chase_cyclic_indices(N, P, k, nb) for k in range(P)])
    assert np.array_equal(np.sort(seen), np.arange(N))
    for k in range(P):
        idx = cb.chase_cyclic_indices(N, P, k, nb)
        assert np.all((idx // nb) % P == k) and np.all(np.diff(idx) > 0)
        assert np.array_equal(idx, ci.cyclic_indices(N, P, k, nb))
