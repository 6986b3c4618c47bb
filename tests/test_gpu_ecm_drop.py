"""restore_feasible's weight-drop branch (ecm.cpp:56-90) on the device:
synthetic nonnegative integrands (8x8 cell, N = 3 modes, L = 4 snapshots,
volume row; seeds found by a search with the oracle) whose greedy refits
produce a non-positive least-squares weight, so the device path steps
alpha = min x/(x - z), drops the zero weight, compacts the selected columns
(J_sel, and the Gram columns in the default scoring mode) and rebuilds the QR
(k_ecm.cu).  ids, weights, residual and iteration count must match the
oracle (ecm.cpp restated) in both scoring modes."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEEDS = [(0, 0), (8, 0), (47, 3), (48, 0)]  # (seed, power): H, W ~ U[0,1]^(1+power)


def _case(seed, power, nq):
    rng = np.random.default_rng(seed)
    H = rng.uniform(0, 1, size=(nq, 3, 4)) ** (1 + power)
    W = rng.uniform(0, 1, size=(4, nq, 4)) ** (1 + power)
    return np.ascontiguousarray(H), np.ascontiguousarray(W)


@pytest.mark.parametrize("mode", ["gram", "direct"])
@pytest.mark.parametrize("seed,power", SEEDS)
def test_ecm_weight_drop_matches_oracle(orc, monkeypatch, mode, seed, power):
    import torch
    from oracle import pod_ecm
    from paper_2307_16894_b200 import api
    if mode == "direct":
        monkeypatch.setenv("PODECM_ECM_SCORE", "direct")
    else:
        monkeypatch.delenv("PODECM_ECM_SCORE", raising=False)
    mats = [api.matrix_params(), api.inclusion_params()]
    g = api.Rve(8, mats)
    t = orc.Rve(8, mats).export()
    H, W = _case(seed, power, g.n_qp)
    st = {}
    ids_o, w_o, rel_o, it_o = pod_ecm.ecm_select(H, W, t["w"], 1e-6, max_points=60, stop_at_count=True, stats=st)
    assert st.get("drops", 0) >= 1, "case does not exercise the drop branch"
    ids_g, w_g, rel_g, it_g = api.ecm_select(g, torch.from_numpy(H).cuda(), torch.from_numpy(W).cuda(),
                                             api.EcmOpts(eps=1e-6, max_points=60, stop_at_count=True))
    print(f"seed {seed} {mode}: drops {st['drops']} at iters {st['drop_iters']}; ids equal "
          f"{np.array_equal(ids_g, ids_o)}; iters {it_g} vs {it_o}; resid {rel_g:.3e} vs {rel_o:.3e}")
    assert np.array_equal(ids_g, ids_o)
    assert it_g == it_o
    assert np.abs(w_g - w_o).max() <= 1e-10 * np.abs(w_o).max()
    assert rel_g <= 1e-6 and rel_o <= 1e-6
