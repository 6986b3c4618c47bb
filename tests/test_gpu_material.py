"""K1 parity: the sm_100a batched material point vs the CPU oracle on
identical seeded inputs (BASELINE config 1 distribution and edge cases).

Tolerances (BASELINE.json north_star): stresses and history 1e-10 relative
per point (Frobenius, absolute floor 1e-14 * scale); tangents 1e-9 per point
normwise (componentwise 1e-9 is below the FD roundoff floor, SURVEY §0
fact 5).  Status codes must match exactly.
"""
import numpy as np
import pytest

from paper_2307_16894_b200 import synth

pytestmark = pytest.mark.gpu

TOL_P = 1e-10
TOL_A = 1e-9


def _run_gpu(F, st, mats, region=None):
    import torch
    from paper_2307_16894_b200 import api
    dev = torch.device("cuda:0")
    Ft = torch.from_numpy(F).to(dev)
    St = torch.from_numpy(st).to(dev)
    Rt = None if region is None else torch.from_numpy(region.astype(np.int32)).to(dev)
    r = api.material_batch(Ft, St, mats, region=Rt)
    torch.cuda.synchronize()
    return {k: (v.cpu().numpy() if v is not None else None) for k, v in r.items()}


def _rel(a, b, floor):
    num = np.sqrt(((a - b) ** 2).sum(0))
    den = np.maximum(np.sqrt((b ** 2).sum(0)), floor)
    return num / den


def _compare(g, o, ok):
    rp = _rel(g["P"][:, ok], o["P"][:, ok], 1e-14)
    ra = _rel(g["A"][:, ok], o["A"][:, ok], 1e-14)
    rs = _rel(g["st"][:, ok], o["st"][:, ok], 1e-14)
    return rp, ra, rs


def test_config1_distribution_parity(orc):
    from paper_2307_16894_b200.api import matrix_params
    F, st = synth.config1_points(1 << 16, 2027)
    mats = [matrix_params()]
    g = _run_gpu(F, st, mats)
    o = orc.material_batch(F, st, mats)
    assert np.array_equal(g["status"], o["status"])
    ok = o["status"] == 0
    rp, ra, rs = _compare(g, o, ok)
    print(f"P max rel {rp.max():.3e}  A max rel {ra.max():.3e} (p99.99 {np.quantile(ra, 0.9999):.3e})"
          f"  state {rs.max():.3e}  P bitwise {np.mean(rp == 0):.4f}  A bitwise {np.mean(ra == 0):.4f}")
    assert rp.max() <= TOL_P
    assert rs.max() <= TOL_P
    assert ra.max() <= TOL_A


def test_edge_cases_parity(orc):
    from paper_2307_16894_b200.api import inclusion_params, matrix_params
    cols = [
        [1, 0, 0, 1],            # identity: repeated root, elastic
        [1.05, 0, 0, 1.05],      # equal biaxial: repeated root
        [1.0, 0.0, 0.0, -0.5],   # det F < 0 -> SolveError
        [0, 0, 0, 0],            # singular
        [1.2, 0.1, -0.05, 0.9],  # plastic
        [1.0 + 1e-9, 0, 0, 1.0], # near-repeated
    ]
    F = np.array(cols, dtype=np.float64).T.copy()
    n = F.shape[1]
    st = np.zeros((6, n))
    st[0] = st[3] = st[4] = 1.0
    mats = [matrix_params(), inclusion_params()]
    for region in (np.zeros(n, np.int32), np.ones(n, np.int32)):
        g = _run_gpu(F, st, mats, region)
        o = orc.material_batch(F, st, mats, region=region)
        assert np.array_equal(g["status"], o["status"]), (g["status"], o["status"])
        ok = o["status"] == 0
        rp, ra, rs = _compare(g, o, ok)
        assert rp.max() <= TOL_P and rs.max() <= TOL_P and ra.max() <= TOL_A


def test_mixed_regions_history_parity(orc):
    from paper_2307_16894_b200.api import inclusion_params, matrix_params
    rng = np.random.default_rng(7)
    n = 1 << 14
    F = np.array([1.0, 0, 0, 1.0])[:, None] + rng.uniform(-0.2, 0.2, (4, n))
    F = F[:, (F[0] * F[3] - F[1] * F[2]) > 0.3].copy()
    n = F.shape[1]
    st = synth.plastic_history(rng, n, 0.05)
    region = rng.integers(0, 2, n).astype(np.int32)
    mats = [matrix_params(), inclusion_params()]
    g = _run_gpu(F, st, mats, region)
    o = orc.material_batch(F, st, mats, region=region)
    assert np.array_equal(g["status"], o["status"])
    ok = o["status"] == 0
    rp, ra, rs = _compare(g, o, ok)
    assert rp.max() <= TOL_P and rs.max() <= TOL_P and ra.max() <= TOL_A


def test_empty_batch():
    import torch
    from paper_2307_16894_b200 import api
    F = torch.empty((4, 0), dtype=torch.float64, device="cuda")
    st = torch.empty((6, 0), dtype=torch.float64, device="cuda")
    r = api.material_batch(F, st, [api.matrix_params()])
    assert r["P"].shape == (4, 0)


def test_failure_is_reported_like_solveerror():
    import torch
    from paper_2307_16894_b200 import api
    F = torch.tensor([[1.0], [0.0], [0.0], [-0.5]], dtype=torch.float64, device="cuda")
    st = torch.tensor([[1.0], [0.0], [0.0], [1.0], [1.0], [0.0]], dtype=torch.float64, device="cuda")
    ctx = api.Context.default()
    api.material_batch(F, st, [api.matrix_params()], ctx=ctx)
    with pytest.raises(api.SolveError):
        ctx.check()
    ctx.check()  # flag cleared
