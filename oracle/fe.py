"""ORACLE — TEST INFRASTRUCTURE ONLY.

Full-order Newton (solve_rve / solve_step, microfem.cpp:142-238) around the
oracle assembly with a dense solve (tiny meshes only), and the exact-limit
reduced model of test_rom.cpp:44-103 (full periodic basis + full
quadrature), used to pin the ROM against the full-order model.
"""
import numpy as np
import scipy.sparse as sp

from paper_2307_16894_b200 import synth


def _assemble_one(r, fbar, w, st0, geom=(0.25, 0.25), tangent=True):
    return r.assemble(np.array([geom]), np.array([fbar]), np.array([w]), st0[None], tangent=tangent,
                      store_stress=True)


def fe_newton_pbar(r, t, geom, sched, tol=1e-10):
    """Full-order solve_rve restated with a dense solve (tiny meshes): the
    reference's Newton (microfem.cpp:142-188) around the oracle assembly."""
    nq = r.n_qp
    st = np.tile(np.array([1.0, 0, 0, 1, 1, 0])[:, None], (1, nq))
    w = np.zeros(r.n_red)
    fmi, det, _ = r.morph(*geom)
    out = []
    for fbar in sched:
        r0 = None
        for it in range(26):
            res = _assemble_one(r, fbar, w, st, geom)
            rn = np.linalg.norm(res["f"][0])
            if r0 is None:
                r0 = rn
                tl = max(tol * r0, 1e-12)
            if rn <= tl:
                break
            K = sp.csr_matrix((res["K"][0], t["col_idx"], t["row_ptr"]), shape=(r.n_red, r.n_red)).toarray()
            w = w + np.linalg.solve(K, -res["f"][0])
        pbar = (res["p_field"][0] * (t["w"] * det)[None, :]).sum(1)
        out.append(pbar)
        st = res["st1"][0]
    return np.array(out)


def exact_limit_model(r, t):
    """Full periodic basis (injection of every reduced dof) + full quadrature."""
    N = r.n_red
    modes = synth.expand(t["node_dof"], np.eye(N)).T  # [2 n_nodes, N]
    nq = r.n_qp
    ids = np.arange(nq, dtype=np.int32)
    mg = np.zeros((nq, N, 4))
    for q in range(nq):
        e = q // 4
        h = np.zeros((N, 2, 2))
        for a in range(4):
            node = t["elems"][e, a]
            h[:, 0, :] = h[:, 0, :] + modes[2 * node, :, None] * t["grad"][q, a][None, :]
            h[:, 1, :] = h[:, 1, :] + modes[2 * node + 1, :, None] * t["grad"][q, a][None, :]
        mg[q] = np.stack([h[:, 0, 0], h[:, 1, 0], h[:, 0, 1], h[:, 1, 1]], -1)
    return ids, t["w"].copy(), mg


