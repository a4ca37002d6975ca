"""Full-size parity at the BASELINE configurations that fit one B200 (C2 = the bench workload,
C3 at 1x1), in the launch configuration bench.py times.  See tests/full_worker.py."""
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_full_size_single_gpu(name):
    import torch
    from full_worker import run_full
    free, total = torch.cuda.mem_get_info()
    need = {"C2": 25e9, "C3": 75e9}[name]
    if free < need:
        pytest.skip(f"needs {need / 1e9:.0f} GB free")
    r = run_full(name, 1, 1)
    print(r)
    assert r["closed_form_col_err"] <= 1e-10, r
    assert r.get("oracle_col_err", 0.0) <= 1e-10, r
    assert r["record_equal"], r
    assert r["qr_variant"] == r["oracle_variant"], r
    assert r["orth"] <= 1e-12, r
