"""Oracle restatement of POD / ECM pinned by the reference's property tests
(test_podkit.cpp:94-143, test_ecm.cpp:164-212) on a reduced config-4
analogue."""
import numpy as np
import pytest

from paper_2307_16894_b200 import synth
from paper_2307_16894_b200.api import inclusion_params, matrix_params


@pytest.fixture(scope="module")
def c4(orc):
    from oracle import pod_ecm
    r = orc.Rve(16, [matrix_params(), inclusion_params()])
    t = r.export()
    U = synth.c4_snapshots(t, L=80, n_terms=5, kmax=3, seed=9)
    W, nf = r.stress_snapshots(U)
    assert nf == 0
    return pod_ecm, r, t, U, W


def test_pod_orthonormal_sorted_nested(c4):
    pod_ecm, r, t, U, W = c4
    modes, lam = pod_ecm.pod_diag(U, None, 10)
    assert modes.shape[1] == 10
    assert np.abs(modes.T @ modes - np.eye(10)).max() <= 1e-10      # :94-99
    assert np.all(np.diff(lam) <= 0)                                   # :101-107
    m6, _ = pod_ecm.pod_diag(U, None, 6)
    assert np.array_equal(m6, modes[:, :6])                            # :116-122 bitwise
    # dropped energy == projection error (:124-136)
    P = modes @ (modes.T @ U)
    err = np.linalg.norm(U - P) ** 2
    assert abs(err - lam[10:].sum()) <= 1e-8 * lam.sum()


def test_pod_rank_drop(c4):
    """test_podkit.cpp:138-143: a dependent column is dropped (tol 1e-6)."""
    pod_ecm, r, t, U, W = c4
    S = U[:, :8].copy()
    S[:, 7] = 2.0 * S[:, 3] - S[:, 4]
    modes, lam = pod_ecm.pod_diag(S, None, 8, 1e-6)
    assert modes.shape[1] == 7


def test_ecm_contract_and_determinism(c4):
    pod_ecm, r, t, U, W = c4
    modes, _ = pod_ecm.pod_diag(U, None, 6)
    H = pod_ecm.mode_grads(t, modes)
    eps = 0.02
    ids, w, rel, it = pod_ecm.ecm_select(H, W, t["w"], eps)
    assert rel <= eps and np.all(w > 0) and np.all(np.diff(ids) > 0)
    # per-row contract via the explicit integrand on the selected set
    J = pod_ecm._J_cols(H, W, np.arange(r.n_qp), 1)
    rhs = J @ t["w"]
    res = rhs - J[:, ids] @ w
    assert np.abs(res).max() <= eps * np.linalg.norm(rhs) / np.sqrt(len(rhs)) * (1 + 1e-12)
    assert abs(w.sum() - 1.0) <= 0.05  # volume row (:195-202)
    ids2, w2, _, _ = pod_ecm.ecm_select(H, W, t["w"], eps)
    assert np.array_equal(ids, ids2) and np.array_equal(w, w2)        # :204-212


def test_ecm_budget_failure(c4):
    pod_ecm, r, t, U, W = c4
    modes, _ = pod_ecm.pod_diag(U, None, 6)
    H = pod_ecm.mode_grads(t, modes)
    with pytest.raises(RuntimeError):
        pod_ecm.ecm_select(H, W, t["w"], 1e-12, max_points=3)
