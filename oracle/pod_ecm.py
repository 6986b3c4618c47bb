"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the offline reduction of the reference
(/root/reference/proj/src/podkit.cpp:43-127 and ecm.cpp:20-204) in numpy /
scipy.  The reference delegates this dense linear algebra to Eigen
(SelfAdjointEigenSolver, ColPivHouseholderQR); here LAPACK does the same
jobs: ``numpy.linalg.eigh`` (dsyevd) for the snapshot eigenproblem and
``scipy.linalg.lstsq(..., lapack_driver="gelsy")`` (column-pivoted QR, the
algorithm of Eigen's colPivHouseholderQr) for every refit, recomputed from
scratch each iteration as the reference does.  The integrand is used in
factored form J[(i L + s), q] = H_q[i] . W_s(q).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


def pod_diag(S, gram_diag, max_modes, tol_rel=1e-10):
    """pod_diag (podkit.cpp:117-127) -> (modes [n_dof, keep], eigenvalues desc)."""
    g = np.ones(S.shape[0]) if gram_diag is None else gram_diag
    corr = S.T @ (g[:, None] * S)
    corr = 0.5 * (corr + corr.T)
    lam, V = np.linalg.eigh(corr)
    lam = lam[::-1].copy()
    V = V[:, ::-1]
    lead = max(lam[0], 0.0)
    cut = tol_rel * tol_rel * lead
    keep = 0
    while keep < len(lam) and keep < max_modes and lam[keep] > cut and lam[keep] > 0.0:
        keep += 1
    modes = np.empty((S.shape[0], keep))
    for i in range(keep):
        modes[:, i] = (S @ V[:, i]) / np.sqrt(lam[i])
    gm = g[:, None] * modes
    for i in range(keep):  # mgs_pass (podkit.cpp:75-86)
        for j in range(i):
            c = gm[:, j] @ modes[:, i]
            modes[:, i] -= c * modes[:, j]
            gm[:, i] -= c * gm[:, j]
        nrm = np.sqrt(gm[:, i] @ modes[:, i])
        modes[:, i] /= nrm
        gm[:, i] /= nrm
    return modes, lam


def mode_grads(tables, modes):
    """H[q][i][c]: parent gradient of each mode at every qp, flatten order
    (build_rom's per-point formula, rom.cpp:91-104)."""
    grad, elems = tables["grad"], tables["elems"]
    nq = grad.shape[0]
    e = np.arange(nq) // 4
    N = modes.shape[1]
    h = np.zeros((nq, N, 2, 2))
    for a in range(4):
        node = elems[e, a]
        ux = modes[2 * node, :]
        uy = modes[2 * node + 1, :]
        h[:, :, 0, :] = h[:, :, 0, :] + ux[:, :, None] * grad[:, None, a, :]
        h[:, :, 1, :] = h[:, :, 1, :] + uy[:, :, None] * grad[:, None, a, :]
    H = np.empty((nq, N, 4))
    H[:, :, 0] = h[:, :, 0, 0]
    H[:, :, 1] = h[:, :, 1, 0]
    H[:, :, 2] = h[:, :, 0, 1]
    H[:, :, 3] = h[:, :, 1, 1]
    return H


def _J_cols(H, W, q, vol):
    """Columns q of the factored integrand: (N L + vol) x len(q)."""
    blk = np.einsum("qic,sqc->isq", H[q], W[:, q])  # N, L, nq
    J = blk.reshape(-1, len(q))
    if vol:
        J = np.vstack([J, np.ones((1, len(q)))])
    return J


def ecm_select(H, W, wq, eps, volume_row=True, max_points=0, stop_at_count=False, trace=None, stats=None):
    """ecm_select (ecm.cpp:132-204) with restore_feasible (:56-90).
    Returns (ids ascending, weights, residual_rel, iterations).  ``stats``
    (a dict) receives the number of restore_feasible weight drops."""
    nq, N, _ = H.shape
    L = W.shape[0]
    vol = 1 if volume_row else 0
    m = N * L + vol
    rhs = np.einsum("qic,sqc->is", H * wq[:, None, None], W).reshape(-1)
    if vol:
        rhs = np.concatenate([rhs, [wq.sum()]])
    rhs_norm = np.linalg.norm(rhs)
    row_tol = eps * rhs_norm / np.sqrt(float(m))
    cap = max_points if max_points > 0 else nq
    col_norm = np.empty(nq)
    bs = max(1, int(2e7 // max(m, 1)))
    for q0 in range(0, nq, bs):
        q = np.arange(q0, min(nq, q0 + bs))
        col_norm[q] = np.sqrt((_J_cols(H, W, q, vol) ** 2).sum(0))
    selected = []
    unavailable = np.zeros(nq, bool)
    x = np.zeros(0)
    resid = rhs.copy()
    iters = 0
    Wf = W.reshape(L, nq * 4)

    def converged(r):
        if rhs_norm == 0.0:
            return True
        return np.linalg.norm(r) <= eps * rhs_norm and np.abs(r).max() <= row_tol

    while not converged(resid):
        if len(selected) >= cap:
            if stop_at_count:
                break
            raise RuntimeError("cubature did not reach the requested accuracy within the point budget")
        T = resid[: N * L].reshape(N, L) @ Wf  # N x (nq*4)
        corr = np.einsum("iqc,qic->q", T.reshape(N, nq, 4), H)
        if vol:
            corr = corr + resid[-1]
        ok = (~unavailable) & (col_norm != 0.0)
        v = np.where(ok, corr / np.where(col_norm != 0.0, col_norm, 1.0), -np.inf)
        best = int(np.argmax(v))  # first maximum (strict '>' scan)
        if not (v[best] > 0.0):
            raise RuntimeError("cubature stalled: no remaining point improves the residual")
        if trace is not None:
            top2 = np.partition(v[np.isfinite(v)], -2)[-2:] if np.isfinite(v).sum() > 1 else [v[best], 0]
            trace.append((best, float(v[best]), float((max(top2) - min(top2)) / abs(max(top2)))))
        selected.append(best)
        unavailable[best] = True
        x = np.concatenate([x, [0.0]])
        # restore_feasible
        while selected:
            A = _J_cols(H, W, np.array(selected), vol)
            z = sla.lstsq(A, rhs, lapack_driver="gelsy")[0]
            if z.min() > 0.0:
                x = z
                break
            alpha = 1.0
            for k in range(len(z)):
                if z[k] <= 0.0:
                    alpha = min(alpha, x[k] / (x[k] - z[k]))
            x = x + alpha * (z - x)
            zero_tol = 1e-12 * max(np.abs(x).max(), 1e-30)
            keep = x > zero_tol
            if stats is not None:
                stats["drops"] = stats.get("drops", 0) + int((~keep).sum())
                stats["drop_iters"] = stats.get("drop_iters", []) + [iters]
            selected = [s for s, kp in zip(selected, keep) if kp]
            x = x[keep]
        iters += 1
        resid = rhs.copy()
        if selected:
            A = _J_cols(H, W, np.array(selected), vol)
            for k in range(len(selected)):
                resid -= x[k] * A[:, k]
    order = np.argsort(np.array(selected, dtype=np.int64), kind="stable")
    ids = np.array(selected, dtype=np.int64)[order]
    weights = x[order]
    rel = 0.0 if rhs_norm == 0.0 else np.linalg.norm(resid) / rhs_norm
    return ids, weights, rel, iters


def ecm_select_sharded(H_loc, W_loc, wq, q0, eps, volume_row=True, max_points=0, stop_at_count=False):
    """The candidate-sharded greedy of the device path (
    podecm_ecm_select_sharded) restated for the host: this rank holds
    candidates [q0, q0 + nq_local) (H_loc [nq_local, N, 4], W_loc
    [L, nq_local, 4]; wq = all quadrature weights).  rhs = J w summed over the
    shards, each iteration's local best (score, global index) reduced with
    the strict-'>' first-index rule (ecm.cpp:164-173), the selected column
    broadcast from its owner, refit / residual replicated.  Uses the
    torch.distributed helpers of paper_2307_16894_b200.shard (gloo in the
    CPU tests); with one rank it is ecm_select."""
    from paper_2307_16894_b200 import shard
    nql, N, _ = H_loc.shape
    nq = wq.shape[0]
    L = W_loc.shape[0]
    vol = 1 if volume_row else 0
    m = N * L + vol
    part = np.ascontiguousarray(np.einsum("qic,sqc->is", H_loc * wq[q0:q0 + nql, None, None], W_loc).reshape(-1))
    shard.allreduce_host(part)
    rhs = np.concatenate([part, [wq.sum()]]) if vol else part
    rhs_norm = np.linalg.norm(rhs)
    row_tol = eps * rhs_norm / np.sqrt(float(m))
    cap = max_points if max_points > 0 else nq
    col_norm = np.sqrt((_J_cols(H_loc, W_loc, np.arange(nql), vol) ** 2).sum(0)) if nql else np.zeros(0)
    selected, cols = [], []
    unavailable = np.zeros(nql, bool)
    x = np.zeros(0)
    resid = rhs.copy()
    iters = 0
    Wf = W_loc.reshape(L, nql * 4)

    def converged(r):
        if rhs_norm == 0.0:
            return True
        return np.linalg.norm(r) <= eps * rhs_norm and np.abs(r).max() <= row_tol

    while not converged(resid):
        if len(selected) >= cap:
            if stop_at_count:
                break
            raise RuntimeError("cubature did not reach the requested accuracy within the point budget")
        loc_s, loc_i = 0.0, -1
        if nql:
            T = resid[: N * L].reshape(N, L) @ Wf
            corr = np.einsum("iqc,qic->q", T.reshape(N, nql, 4), H_loc)
            if vol:
                corr = corr + resid[-1]
            ok = (~unavailable) & (col_norm != 0.0)
            v = np.where(ok, corr / np.where(col_norm != 0.0, col_norm, 1.0), -np.inf)
            k = int(np.argmax(v))
            if v[k] > 0.0:
                loc_s, loc_i = float(v[k]), q0 + k
        s, best, owner = shard.argmax_owner(loc_s, loc_i)
        if best < 0:
            raise RuntimeError("cubature stalled: no remaining point improves the residual")
        col = np.zeros(m)
        if q0 <= best < q0 + nql:
            unavailable[best - q0] = True
            col[:] = _J_cols(H_loc, W_loc, np.array([best - q0]), vol)[:, 0]
        shard.bcast_host(col, owner)
        selected.append(best)
        cols.append(col)
        x = np.concatenate([x, [0.0]])
        while selected:  # restore_feasible (ecm.cpp:56-90), replicated
            A = np.stack(cols, 1)
            z = sla.lstsq(A, rhs, lapack_driver="gelsy")[0]
            if z.min() > 0.0:
                x = z
                break
            alpha = 1.0
            for kk in range(len(z)):
                if z[kk] <= 0.0:
                    alpha = min(alpha, x[kk] / (x[kk] - z[kk]))
            x = x + alpha * (z - x)
            zero_tol = 1e-12 * max(np.abs(x).max(), 1e-30)
            keep = x > zero_tol
            selected = [s_ for s_, kp in zip(selected, keep) if kp]
            cols = [c_ for c_, kp in zip(cols, keep) if kp]
            x = x[keep]
        iters += 1
        resid = rhs.copy()
        for kk in range(len(selected)):
            resid -= x[kk] * cols[kk]
    order = np.argsort(np.array(selected, dtype=np.int64), kind="stable")
    ids = np.array(selected, dtype=np.int64)[order]
    rel = 0.0 if rhs_norm == 0.0 else np.linalg.norm(resid) / rhs_norm
    return ids, x[order], rel, iters
