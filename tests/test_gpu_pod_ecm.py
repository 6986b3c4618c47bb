"""K4 parity: offline POD (DMMA Gram + syevd + MGS) and the greedy ECM on the
factored integrand, vs the CPU oracle (podkit.cpp / ecm.cpp restated with
LAPACK), on a reduced config-4 analogue (32x32 mesh, 200 snapshots, 12 modes,
60 points).  ECM ids must be bit-exact; POD eigenvalues 1e-10 relative;
modes compared up to sign.
"""
import numpy as np
import pytest

from paper_2307_16894_b200 import synth

pytestmark = pytest.mark.gpu


def _mats():
    from paper_2307_16894_b200.api import inclusion_params, matrix_params
    return [matrix_params(), inclusion_params()]


@pytest.fixture(scope="module")
def case(orc):
    from oracle import pod_ecm
    from paper_2307_16894_b200 import api
    g = api.Rve(32, _mats())
    o = orc.Rve(32, _mats())
    t = o.export()
    U = synth.c4_snapshots(t, L=200, n_terms=6, kmax=4, seed=5)
    modes, lam = pod_ecm.pod_diag(U, None, 12)
    W, nf = o.stress_snapshots(U)
    assert nf == 0
    H = pod_ecm.mode_grads(t, modes)
    return g, o, t, U, modes, lam, W, H


def _sign_fix(M):  # columns: largest-|.| entry positive
    idx = np.abs(M).argmax(0)
    return M * np.sign(M[idx, np.arange(M.shape[1])])


def test_pod_gram_and_modes(case):
    import torch
    from paper_2307_16894_b200 import api
    g, o, t, U, modes, lam, W, H = case
    Ut = torch.from_numpy(np.ascontiguousarray(U.T)).cuda()
    mt, ev = api.pod(Ut, 12)
    torch.cuda.synchronize()
    ev = ev.cpu().numpy()
    assert mt.shape[0] == 12
    rel = np.abs(ev[:12] - lam[:12]) / lam[:12]
    print(f"eigenvalue max rel {rel.max():.2e}")
    assert rel.max() <= 1e-10
    gm = _sign_fix(mt.cpu().numpy().T)
    om = _sign_fix(modes)
    err = np.abs(gm - om).max() / np.abs(om).max()
    print(f"modes max rel (up to sign) {err:.2e}")
    assert err <= 1e-8
    # orthonormality after the MGS pass (test_podkit.cpp:94-99)
    assert np.abs(gm.T @ gm - np.eye(12)).max() <= 1e-12


def test_stress_snapshots_and_mode_grads(case):
    import torch
    from paper_2307_16894_b200 import api
    g, o, t, U, modes, lam, W, H = case
    Wg, st = api.ecm_stress_snapshots(g, torch.from_numpy(np.ascontiguousarray(U.T)).cuda())
    Hg = api.ecm_mode_grads(g, torch.from_numpy(np.ascontiguousarray(modes.T)).cuda())
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    Wg = Wg.cpu().numpy()
    d = np.sqrt(((Wg - W) ** 2).sum(-1)) / np.maximum(np.sqrt((W ** 2).sum(-1)), 1e-14)
    print(f"W max rel {d.max():.2e}, bitwise {np.mean(Wg == W):.4f}")
    assert d.max() <= 1e-10
    assert np.array_equal(Hg.cpu().numpy(), H)


def test_ecm_ids_bit_exact(case):
    import torch
    from oracle import pod_ecm
    from paper_2307_16894_b200 import api
    g, o, t, U, modes, lam, W, H = case
    ids_o, w_o, rel_o, it_o = pod_ecm.ecm_select(H, W, t["w"], 1e-8, max_points=60, stop_at_count=True)
    ids_g, w_g, rel_g, it_g = api.ecm_select(g, torch.from_numpy(H).cuda(), torch.from_numpy(W).cuda(),
                                             api.EcmOpts(eps=1e-8, max_points=60, stop_at_count=True))
    print(f"ids equal {np.array_equal(ids_g, ids_o)}; resid {rel_g:.6e} vs {rel_o:.6e}; iters {it_g} vs {it_o}")
    assert np.array_equal(ids_g, ids_o)
    assert it_g == it_o
    assert np.abs(w_g - w_o).max() <= 1e-8 * np.abs(w_o).max()
    assert abs(rel_g - rel_o) <= 1e-8 * max(rel_o, 1e-30) + 1e-14


def test_ecm_residual_contract(case):
    """test_ecm.cpp:164-185: converged rule meets eps in RMS and per row,
    positive weights, ascending ids; volume row integrates |cell|."""
    import torch
    from paper_2307_16894_b200 import api
    g, o, t, U, modes, lam, W, H = case
    eps = 0.05
    ids, w, rel, it = api.ecm_select(g, torch.from_numpy(H).cuda(), torch.from_numpy(W).cuda(),
                                     api.EcmOpts(eps=eps))
    assert rel <= eps
    assert np.all(w > 0) and np.all(np.diff(ids) > 0)
    assert abs(w.sum() - t["w"].sum()) <= 0.05 * t["w"].sum()  # test_ecm.cpp:195-202


def test_ecm_budget_exhaustion_raises(case):
    """ecm.cpp:159-162: without stop_at_count, hitting max_points throws."""
    import torch
    from paper_2307_16894_b200 import api
    g, o, t, U, modes, lam, W, H = case
    with pytest.raises(api.SolveError):
        api.ecm_select(g, torch.from_numpy(H).cuda(), torch.from_numpy(W).cuda(),
                       api.EcmOpts(eps=1e-12, max_points=5))


def test_ecm_wide_basis_ids_bit_exact(case):
    """N = 80 displacement modes (> 56 rows of the DMMA scoring tile): the
    first J^T rhs pass runs in row blocks, later iterations use the Gram
    update; ids still bit-exact vs the oracle."""
    import torch
    from oracle import pod_ecm
    from paper_2307_16894_b200 import api
    g, o, t, U, modes, lam, W, H = case
    modes80, _ = pod_ecm.pod_diag(U, None, 80)
    H80 = pod_ecm.mode_grads(t, modes80)
    Ws = np.ascontiguousarray(W[:40])
    ids_o, w_o, rel_o, it_o = pod_ecm.ecm_select(H80, Ws, t["w"], 1e-8, max_points=40, stop_at_count=True)
    ids_g, w_g, rel_g, it_g = api.ecm_select(g, torch.from_numpy(H80).cuda(), torch.from_numpy(Ws).cuda(),
                                             api.EcmOpts(eps=1e-8, max_points=40, stop_at_count=True))
    print(f"N=80: ids equal {np.array_equal(ids_g, ids_o)}; resid {rel_g:.6e} vs {rel_o:.6e}")
    assert np.array_equal(ids_g, ids_o) and it_g == it_o
    assert np.abs(w_g - w_o).max() <= 1e-8 * np.abs(w_o).max()


@pytest.mark.parametrize("spec", [0, 1, 3])
def test_ecm_speculative_gram_columns_change_nothing(case, monkeypatch, spec):
    """The Gram-column cache (k_ecm.cu: each pass over W also computes the
    columns of the scoring pass's runner-up candidates, on the DMMA path) only
    changes how often W is streamed: ids, weights, residual and iteration
    count are bit-identical to the uncached greedy, which computes one column
    per pass."""
    import torch
    from paper_2307_16894_b200 import api
    g, o, t, U, modes, lam, W, H = case
    Hd, Wd = torch.from_numpy(H).cuda(), torch.from_numpy(W).cuda()
    opts = api.EcmOpts(eps=1e-8, max_points=60, stop_at_count=True)
    monkeypatch.setenv("PODECM_ECM_SPEC", "0")
    ref = api.ecm_select(g, Hd, Wd, opts)
    monkeypatch.setenv("PODECM_ECM_SPEC", str(spec))
    got = api.ecm_select(g, Hd, Wd, opts)
    assert np.array_equal(got[0], ref[0])
    assert np.array_equal(np.asarray(got[1]).view(np.int64), np.asarray(ref[1]).view(np.int64))
    assert got[2] == ref[2] and got[3] == ref[3]
