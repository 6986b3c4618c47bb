"""Seeded synthetic inputs for BASELINE.json configs 0-3 (numpy, host).

The reference measures on no public suite; these generators realise the
configs' stated shapes and distributions.  Every array is
produced once on the host and the identical bytes feed both the CUDA path and
the CPU oracle.  Seeds: ``2026 + config index`` unless overridden.

History convention (reference terms, material.hpp:55-59): a plastic history
with equivalent plastic strain eps_p is Fp = exp(sqrt(3/2) eps_p n) on the
in-plane block and Fp_zz = exp(sqrt(3/2) eps_p n_zz), n a random unit
deviatoric plane-strain direction (so det Fp * Fp_zz = 1), xi = eps_p.
"""
from __future__ import annotations

import numpy as np

IDENT = np.array([1.0, 0.0, 0.0, 1.0])


def expm_sym2(a, b, c):
    """exp of the symmetric 2x2 [[a, c], [c, b]] (vectorised closed form).
    Returns flatten order (00, 10, 01, 11)."""
    m = 0.5 * (a + b)
    h = 0.5 * (a - b)
    d = np.sqrt(h * h + c * c)
    em = np.exp(m)
    ch = np.cosh(d)
    sh = np.where(d > 1e-300, np.sinh(d) / np.where(d > 1e-300, d, 1.0), 1.0)
    e00 = em * (ch + sh * h)
    e11 = em * (ch - sh * h)
    e01 = em * sh * c
    return np.stack([e00, e01, e01, e11])


def plastic_history(rng, n, eps_max):
    """[6, n] states: Fp = exp(sqrt(3/2) eps_p n_dev), xi = eps_p ~ U[0, eps_max]."""
    g = rng.standard_normal((4, n))
    tr = (g[0] + g[1] + g[2]) / 3.0
    g[0] -= tr
    g[1] -= tr
    g[2] -= tr
    nrm = np.sqrt(g[0] ** 2 + g[1] ** 2 + g[2] ** 2 + 2.0 * g[3] ** 2)
    g /= nrm
    ep = rng.uniform(0.0, eps_max, n)
    s = np.sqrt(1.5) * ep
    fp = expm_sym2(s * g[0], s * g[1], s * g[3])
    st = np.empty((6, n))
    st[:4] = fp
    st[4] = np.exp(s * g[2])
    st[5] = ep
    return st


def config1_points(n: int = 1 << 22, seed: int = 2027):
    """Config 1: F = I + N(0, 0.08^2) resampled until det F > 0.5; history
    Fp = exp(-L/2) with L symmetric N(0, 0.02^2) (xx, yy, zz, xy),
    xi ~ U[0, 0.1].  Returns F [4, n], st [6, n]."""
    rng = np.random.default_rng(seed)
    F = IDENT[:, None] + rng.normal(0.0, 0.08, (4, n))
    bad = (F[0] * F[3] - F[1] * F[2]) <= 0.5
    while bad.any():
        k = int(bad.sum())
        F[:, bad] = IDENT[:, None] + rng.normal(0.0, 0.08, (4, k))
        bad = (F[0] * F[3] - F[1] * F[2]) <= 0.5
    L = rng.normal(0.0, 0.02, (4, n))
    st = np.empty((6, n))
    st[:4] = expm_sym2(-0.5 * L[0], -0.5 * L[1], -0.5 * L[3])
    st[4] = np.exp(-0.5 * L[2])
    st[5] = rng.uniform(0.0, 0.1, n)
    return np.ascontiguousarray(F), np.ascontiguousarray(st)


def rve_instances(n_inst: int, n_red: int, regions_qp: np.ndarray, seed: int,
                  hm: float, geom_range=None, geom_fixed=(0.3, 0.2), w_sigma: float = 1e-3,
                  eps_max: float = 0.05):
    """Configs 0/2: per instance geometry (a, b), Fbar = I + H_M
    (H_M ~ U[-hm, hm]^4), w_red ~ N(0, w_sigma^2), plastic history of the
    matrix phase (virgin Fp = I in the elastic inclusion)."""
    rng = np.random.default_rng(seed)
    nq = regions_qp.shape[0]
    if geom_range is None:
        geom = np.tile(np.asarray(geom_fixed, dtype=np.float64), (n_inst, 1))
    else:
        geom = rng.uniform(geom_range[0], geom_range[1], (n_inst, 2))
    fbar = IDENT[None, :] + rng.uniform(-hm, hm, (n_inst, 4))
    w_red = rng.normal(0.0, w_sigma, (n_inst, n_red))
    st = np.empty((n_inst, 6, nq))
    incl = regions_qp != 0
    for s in range(n_inst):
        h = plastic_history(rng, nq, eps_max)
        h[:, incl] = np.array([1.0, 0.0, 0.0, 1.0, 1.0, 0.0])[:, None]
        st[s] = h
    return (np.ascontiguousarray(geom), np.ascontiguousarray(fbar), np.ascontiguousarray(w_red),
            st)


def expand(node_dof: np.ndarray, v_red: np.ndarray) -> np.ndarray:
    """DofMap::expand (mesh.cpp:390-400) of [..., n_red] -> [..., 2 n_nodes]."""
    n_nodes = node_dof.shape[0]
    out = np.zeros(v_red.shape[:-1] + (2 * n_nodes,))
    ok = node_dof >= 0
    idx = np.nonzero(ok)[0]
    out[..., 2 * idx] = v_red[..., node_dof[idx]]
    out[..., 2 * idx + 1] = v_red[..., node_dof[idx] + 1]
    return out


def rom_model(tables: dict, n_red: int, N: int = 50, Q: int = 400, seed: int = 2029):
    """Config 3 model: N modes = QR of a seeded Gaussian in the reduced
    periodic space (n_red x N), expanded to full nodal dofs (periodicity kept);
    Q ECM ids drawn without replacement (ascending); weights U[0.5,1.5]/Q
    (|cell| = 1).  mode_grads per build_rom (rom.cpp:80-109)."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n_red, N))
    qm, _ = np.linalg.qr(g)
    modes = expand(tables["node_dof"], qm.T).T  # [2 n_nodes, N]
    nq = tables["w"].shape[0]
    ids = np.sort(rng.choice(nq, size=Q, replace=False)).astype(np.int32)
    weights = rng.uniform(0.5, 1.5, Q) / Q
    grad = tables["grad"]  # [nq, 4, 2]
    elems = tables["elems"]
    mg = np.zeros((Q, N, 4))
    for p, qp in enumerate(ids):
        e = qp // 4
        h = np.zeros((N, 2, 2))
        for a in range(4):  # h.row(0) += modes(2 node, i) g.row(a), rom.cpp:96-100
            node = elems[e, a]
            h[:, 0, :] = h[:, 0, :] + modes[2 * node, :, None] * grad[qp, a][None, :]
            h[:, 1, :] = h[:, 1, :] + modes[2 * node + 1, :, None] * grad[qp, a][None, :]
        mg[p, :, 0] = h[:, 0, 0]
        mg[p, :, 1] = h[:, 1, 0]
        mg[p, :, 2] = h[:, 0, 1]
        mg[p, :, 3] = h[:, 1, 1]
    return {"modes": modes, "ids": ids, "weights": weights, "mode_grads": mg}


def rom_instances(n_inst: int, K: int = 20, seed: int = 2030, hm: float = 0.2):
    """Config 3 loading: (a, b) ~ U[0.15, 0.35]^2, proportional schedule
    Fbar_k = I + (k/K) H_M, H_M ~ U[-hm, hm]^4.  Returns geom [n,2],
    sched [n,K,4]."""
    rng = np.random.default_rng(seed)
    geom = rng.uniform(0.15, 0.35, (n_inst, 2))
    H = rng.uniform(-hm, hm, (n_inst, 4))
    k = (np.arange(1, K + 1) / K)[None, :, None]
    sched = IDENT[None, None, :] + k * H[:, None, :]
    return np.ascontiguousarray(geom), np.ascontiguousarray(sched)


def c4_snapshots(tables: dict, L: int = 4000, n_terms: int = 20, kmax: int = 8, seed: int = 2030,
                 target_rms: float = 0.05, xp=np, device=None):
    """Config 4 snapshots: L periodic displacement fields at the mesh nodes,
    u_comp(X) = sum_m A_m cos(2 pi k_m . X + phi_m) per component, integer
    wave vectors with 1 <= |k|_inf <= kmax, A ~ N(0, 1/|k|_2^2).  The literal
    amplitudes give RMS |grad u| = 2 pi sqrt(n_terms) (~28 for 20 terms,
    SURVEY §8d), so one global scale pins RMS |grad u| = target_rms.  The
    anchor node's value is subtracted (fluctuation convention: anchor dof
    pinned, mesh.cpp:370).  Returns U column-major [2 n_nodes, L] (numpy or,
    with xp=torch, a device tensor of shape [L, 2 n_nodes] whose transpose is
    the column-major matrix)."""
    rng = np.random.default_rng(seed)
    X = tables["nodes"]
    n_nodes = X.shape[0]
    anchor = int(np.nonzero((np.abs(X[:, 0]) < 1e-12) & (np.abs(X[:, 1]) < 1e-12))[0][0])
    k = rng.integers(-kmax, kmax + 1, size=(L, 2, n_terms, 2))
    zero = (k[..., 0] == 0) & (k[..., 1] == 0)
    while zero.any():
        k[zero] = rng.integers(-kmax, kmax + 1, size=(int(zero.sum()), 2))
        zero = (k[..., 0] == 0) & (k[..., 1] == 0)
    kn = np.sqrt((k.astype(np.float64) ** 2).sum(-1))
    amp = rng.standard_normal((L, 2, n_terms)) / kn
    phi = rng.uniform(0.0, 2 * np.pi, (L, 2, n_terms))
    scale = target_rms / (2 * np.pi * np.sqrt(n_terms))
    if xp is np:
        U = np.zeros((L, n_nodes, 2))
        for m in range(n_terms):
            arg = 2 * np.pi * (k[:, :, m, 0, None] * X[None, None, :, 0] +
                               k[:, :, m, 1, None] * X[None, None, :, 1]) + phi[:, :, m, None]
            U += np.transpose(amp[:, :, m, None] * np.cos(arg), (0, 2, 1))
        U -= U[:, anchor:anchor + 1, :]
        U *= scale
        return np.asfortranarray(U.reshape(L, 2 * n_nodes).T)
    torch = xp
    Xt = torch.from_numpy(X).to(device)
    kt = torch.from_numpy(k.astype(np.float64)).to(device)
    at = torch.from_numpy(amp).to(device)
    pt = torch.from_numpy(phi).to(device)
    U = torch.zeros((L, n_nodes, 2), dtype=torch.float64, device=device)
    for m in range(n_terms):
        arg = 2 * np.pi * (kt[:, :, m, 0, None] * Xt[None, None, :, 0] +
                           kt[:, :, m, 1, None] * Xt[None, None, :, 1]) + pt[:, :, m, None]
        U += (at[:, :, m, None] * torch.cos(arg)).permute(0, 2, 1)
    U -= U[:, anchor:anchor + 1, :].clone()
    U *= scale
    return U.reshape(L, 2 * n_nodes).contiguous()
