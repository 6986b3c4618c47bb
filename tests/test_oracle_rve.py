"""Oracle restatement of the Q4 RVE path pinned by the reference's property
tests: periodic pairing counts (test_mesh.cpp:181-208), quadrature /
partition of unity (test_mesh.cpp:30-108), homogeneous cell == point driver
(test_microfem.cpp:44-65), consistent tangent vs FD of the residual
(test_microfem.cpp:111-142) and the ROM exact limit (test_rom.cpp:44-125)."""
import numpy as np
import pytest
import scipy.sparse as sp

from paper_2307_16894_b200 import synth
from paper_2307_16894_b200.api import PlasticityParams, inclusion_params, matrix_params


def mats():
    return [matrix_params(), inclusion_params()]


@pytest.mark.parametrize("n,n_red,nnz", [(64, 8190, 147388), (16, 510, 8764)])
def test_periodic_pattern_sizes(orc, n, n_red, nnz):
    r = orc.Rve(n, mats())
    assert r.n_red == n_red
    if n == 64:
        assert r.nnz == nnz
    t = r.export()
    nd = t["node_dof"]
    assert nd[r.anchor] == -1
    # slaves alias masters: every master dof appears for exactly 1, 2 (edge) nodes
    vals, counts = np.unique(nd[nd >= 0], return_counts=True)
    assert set(counts) <= {1, 2} and len(vals) * 2 == r.n_red
    # CSR rows sorted, structurally symmetric
    rp, ci = t["row_ptr"], t["col_idx"]
    for row in range(0, r.n_red, max(1, r.n_red // 50)):
        assert np.all(np.diff(ci[rp[row]:rp[row + 1]]) > 0)
    A = sp.csr_matrix((np.ones(len(ci)), ci, rp), shape=(r.n_red, r.n_red))
    assert (A != A.T).nnz == 0


def test_quadrature_and_partition_of_unity(orc):
    t = orc.Rve(8, mats()).export()
    assert abs(t["w"].sum() - 1.0) <= 1e-14
    assert np.abs(t["grad"].sum(axis=1)).max() <= 1e-12


def _assemble_one(r, fbar, w, st0, geom=(0.25, 0.25), tangent=True):
    return r.assemble(np.array([geom]), np.array([fbar]), np.array([w]), st0[None], tangent=tangent,
                      store_stress=True)


def test_homogeneous_cell_matches_point_driver(orc):
    m = matrix_params()
    r = orc.Rve(8, [m, m])
    t = r.export()
    nq = r.n_qp
    st = np.tile(np.array([1.0, 0, 0, 1, 1, 0])[:, None], (1, nq))
    point = np.array([1.0, 0, 0, 1, 1, 0])[:, None]
    for fbar in ([1.06, 0.0, 0.04, 0.95], [1.02, 0.01, -0.03, 1.01]):
        fbar = np.array(fbar)
        res = _assemble_one(r, fbar, np.zeros(r.n_red), st)
        assert np.linalg.norm(res["f"][0]) <= 1e-12
        pbar = (res["p_field"][0] * t["w"][None, :]).sum(1)  # det = 1 (identity morph)
        pt = orc.material_batch(fbar[:, None], point, [m])
        assert np.linalg.norm(pbar - pt["P"][:, 0]) <= 1e-10
        st = res["st1"][0]
        point = pt["st"]


def test_tangent_matches_fd_of_residual(orc):
    r = orc.Rve(6, mats())
    t = r.export()
    rng = np.random.default_rng(3)
    _, fbar, w, st = synth.rve_instances(1, r.n_red, np.repeat(t["regions"], 4), 4, 0.05)
    geom = (0.3, 0.2)
    base = _assemble_one(r, fbar[0], w[0], st[0], geom)
    K = sp.csr_matrix((base["K"][0], t["col_idx"], t["row_ptr"]), shape=(r.n_red, r.n_red))
    for _ in range(10):
        d = rng.standard_normal(r.n_red)
        d /= np.linalg.norm(d)
        h = 1e-6
        fp = _assemble_one(r, fbar[0], w[0] + h * d, st[0], geom, tangent=False)["f"][0]
        fm = _assemble_one(r, fbar[0], w[0] - h * d, st[0], geom, tangent=False)["f"][0]
        fd = (fp - fm) / (2 * h)
        assert np.linalg.norm(K @ d - fd) <= 1e-5 * np.linalg.norm(fd) + 1e-10


from oracle.fe import exact_limit_model, fe_newton_pbar  # noqa: E402


def test_rom_exact_limit_equals_full_order(orc):
    """test_rom.cpp:44-125: full basis + full quadrature => ROM == FE."""
    r = orc.Rve(4, mats())
    t = r.export()
    ids, wts, mg = exact_limit_model(r, t)
    geom = (0.3, 0.2)
    H = np.array([0.06, 0.02, -0.03, -0.04])
    sched = np.array([[1, 0, 0, 1] + (k / 6) * H for k in range(1, 7)])
    fe = fe_newton_pbar(r, t, geom, sched)
    ro = r.rom_solve(ids, wts, mg, np.array([geom]), sched[None], eps_rel=1e-10)
    assert ro["status"][0] == 0
    err = np.abs(ro["pbar"][0] - fe).max() / np.abs(fe).max()
    assert err <= 1e-8, err
