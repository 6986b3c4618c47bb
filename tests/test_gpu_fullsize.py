"""Configs 2, 3 and 4 at BASELINE.json's full sizes, checked through
size-independent properties plus oracle parity on a spread sample:

  * C2 (1024 x 128^2 assembly): no failed instance; bitwise run-to-run
    determinism; batch invariance (a sub-batch assembled alone is bitwise the
    same as inside the full batch, although the chunking and grid differ);
    oracle parity of 32 spread instances (f 1e-10, K 1e-9 relative).
  * C3 (65,536 ROM instances, N = 50, Q = 400, 20 increments): no failed
    instance; batch invariance of a spread sub-batch (pbar bitwise, Newton
    iteration counts equal); oracle parity of 256 spread instances (pbar
    1e-8, iteration counts equal).
  * C4 (POD of 33,282 x 4,000 snapshots, ECM over 65,536 candidates to 400
    points): the 400 ids bit-exact against the CPU oracle's full-size
    selection (tests/golden/c4_ecm_golden.npz), orthonormal modes and eigenvalues against an independent fp64
    torch Gram + eigvalsh (1e-10); ECM ids unique and ascending with positive
    weights; the reported residual equals ||J_sel w - J w_full|| / ||J w_full||
    recomputed from the factored integrand (ecm.cpp:20-48, 132-204), and the
    weights are the unconstrained least-squares fit on the selected set
    whenever that fit is positive (restore_feasible leaves it unchanged).

The torch / numpy arithmetic here is the checker, not the product path.
"""
import numpy as np
import pytest

from paper_2307_16894_b200 import synth

pytestmark = pytest.mark.gpu


def _mats():
    from paper_2307_16894_b200.api import inclusion_params, matrix_params
    return [matrix_params(), inclusion_params()]


def test_config2_full_size(orc):
    import torch

    import bench
    from paper_2307_16894_b200 import api
    dev = torch.device("cuda:0")
    rve = api.Rve(128, _mats())
    n = 1024
    geom, fbar, w_red, st0 = bench.rve_inputs_gpu(torch, rve, n, 2028, 0.2, (0.15, 0.35), dev)
    a = rve.assemble(fbar, w_red, st0, geom=geom)
    b = rve.assemble(fbar, w_red, st0, geom=geom)
    torch.cuda.synchronize()
    assert int((a["status"] != 0).sum()) == 0
    for k in ("f", "K", "st1"):
        assert torch.equal(a[k], b[k]), k
    sub = torch.tensor([0, 1, 377, 511, 512, 800, 1022, 1023], device=dev)
    c = rve.assemble(fbar[sub].contiguous(), w_red[sub].contiguous(), st0[sub].contiguous(),
                     geom=geom[sub].contiguous())
    torch.cuda.synchronize()
    for k in ("f", "K", "st1"):
        assert torch.equal(c[k], a[k][sub]), k
    o = orc.Rve(128, _mats())
    pick = list(np.unique(np.linspace(0, n - 1, 32).astype(np.int64)))  # 32 spread instances
    h = lambda t: t[pick].cpu().numpy().copy()
    ro = o.assemble(h(geom), h(fbar), h(w_red), h(st0), nthreads=orc.max_threads())
    for j, s in enumerate(pick):
        ef = np.linalg.norm(a["f"][s].cpu().numpy() - ro["f"][j]) / np.linalg.norm(ro["f"][j])
        eK = np.linalg.norm(a["K"][s].cpu().numpy() - ro["K"][j]) / np.linalg.norm(ro["K"][j])
        print(f"instance {s}: f {ef:.2e}  K {eK:.2e}")
        assert ef <= 1e-10 and eK <= 1e-9


def test_config3_full_size(orc):
    import torch

    from paper_2307_16894_b200 import api
    dev = torch.device("cuda:0")
    rve = api.Rve(128, _mats())
    model = synth.rom_model(rve.export(), rve.n_red, N=50, Q=400, seed=2029)
    rom = api.Rom(rve, model["ids"], model["weights"], model["mode_grads"])
    n, K = 65536, 20
    geom_np, sched_np = synth.rom_instances(n, K, 2030, 0.2)
    geom, sched = torch.from_numpy(geom_np).to(dev), torch.from_numpy(sched_np).to(dev)
    opts = api.NewtonOpts(eps_rel=1e-10, eps_abs=1e-12, max_iter=25, max_bisect=5)
    full = rom.solve(geom, sched, opts)
    torch.cuda.synchronize()
    assert int((full["status"] != 0).sum()) == 0
    sub = np.unique(np.linspace(0, n - 1, 97).astype(np.int64))
    ts = torch.from_numpy(sub).to(dev)
    part = rom.solve(geom[ts].contiguous(), sched[ts].contiguous(), opts)
    torch.cuda.synchronize()
    assert torch.equal(part["pbar"], full["pbar"][ts])
    assert torch.equal(part["iters"], full["iters"][ts])
    pick = np.unique(np.linspace(0, n - 1, 256).astype(np.int64))  # 256 spread instances
    o = orc.Rve(128, _mats())
    ro = o.rom_solve(model["ids"], model["weights"], model["mode_grads"], geom_np[pick], sched_np[pick],
                     eps_rel=1e-10, eps_abs=1e-12, max_iter=25, max_bisect=5, nthreads=orc.max_threads())
    tp = torch.from_numpy(pick).to(dev)
    pg = full["pbar"][tp].cpu().numpy()
    rel = np.linalg.norm(pg - ro["pbar"], axis=-1) / np.maximum(np.linalg.norm(ro["pbar"], axis=-1), 1e-14)
    it = full["iters"][tp].cpu().numpy()
    rg = full["resid"][tp].cpu().numpy()
    # Newton counts per increment equal, except where the stop is decided at
    # the round-off floor of the increment's own tolerance
    # tol = max(eps_rel r0, eps_abs) (r0: its initial residual, rom.cpp:128-131;
    # ~1e-12 here): the side that stopped FIRST did so with its converged
    # residual in the band [1e-2, 1] x tol, where the order of the reduced sums
    # decides whether ||f|| <= tol one iteration earlier or later (the
    # reference's own Eigen order is a third one); the side that went on ends
    # at or below tol.  P-bar is unaffected (<= 1e-8).
    mism = np.argwhere(it != ro["iters"])
    tol = np.maximum(1e-10 * ro["init_resid"], 1e-12)
    assert tol.max() <= 1e-11
    first = [(rg[s, k] if it[s, k] < ro["iters"][s, k] else ro["resid"][s, k]) for s, k in mism]
    later = [(ro["resid"][s, k] if it[s, k] < ro["iters"][s, k] else rg[s, k]) for s, k in mism]
    floor = [bool(1e-2 * tol[s, k] <= a <= tol[s, k] * (1 + 1e-9) and b <= tol[s, k] * (1 + 1e-9))
             for (s, k), a, b in zip(mism, first, later)]
    print(f"sampled instances {len(pick)}: pbar max rel {rel.max():.2e}; iteration-count mismatches "
          f"{len(mism)} of {it.size} increments, all at the round-off floor: {all(floor)} "
          f"({[(int(pick[s]), int(k), int(it[s, k]), int(ro['iters'][s, k]), float(rg[s, k]), float(ro['resid'][s, k])) for s, k in mism]})")
    assert len(pick) >= 256
    assert rel.max() <= 1e-8
    assert all(floor) and len(mism) <= 1e-3 * it.size


def test_config4_full_size():
    import torch

    from paper_2307_16894_b200 import api
    dev = torch.device("cuda:0")
    rve = api.Rve(128, _mats())
    L, N, Q = 4000, 50, 400
    U = synth.c4_snapshots(rve.export(), L=L, n_terms=20, kmax=8, seed=2030, xp=torch, device=dev)
    modes, ev = api.pod(U, N)
    torch.cuda.synchronize()
    # POD: orthonormal modes; eigenvalues against an independent Gram + eigvalsh
    eye = modes @ modes.T
    assert float((eye - torch.eye(N, dtype=eye.dtype, device=dev)).abs().max()) <= 1e-10
    lam = torch.linalg.eigvalsh(U @ U.T).flip(0)[:N]
    assert torch.all(ev[:N][:-1] >= ev[:N][1:])
    assert float(((ev[:N] - lam).abs() / lam[0]).max()) <= 1e-10
    # ECM on the factored integrand
    W, _ = api.ecm_stress_snapshots(rve, U)
    H = api.ecm_mode_grads(rve, modes)
    opts = api.EcmOpts(eps=1e-6, volume_row=True, max_points=Q, stop_at_count=True)
    ids, w, rel, _ = api.ecm_select(rve, H, W, opts)
    ids_np = np.asarray(ids)
    w_t = torch.as_tensor(np.asarray(w), dtype=torch.float64, device=dev)
    assert len(ids_np) == Q
    assert np.all(np.diff(ids_np) > 0) and ids_np[0] >= 0 and ids_np[-1] < rve.n_qp
    assert bool(torch.all(w_t > 0))
    # J[(i, l), q] = H_q[i] . W_l(q) (+ a row of ones); rhs = J w_full
    wq = torch.as_tensor(rve.export()["w"], dtype=torch.float64, device=dev)
    Hq = H.reshape(rve.n_qp, N, 4)
    Wq = W.reshape(L, rve.n_qp, 4)
    rhs = torch.einsum("qic,lqc->il", Hq * wq[:, None, None], Wq).reshape(-1)
    rhs = torch.cat([rhs, wq.sum().reshape(1)])
    sel = torch.from_numpy(ids_np).to(dev)
    Jsel = torch.einsum("sic,lsc->ils", Hq[sel], Wq[:, sel]).reshape(N * L, Q)
    Jsel = torch.cat([Jsel, torch.ones((1, Q), dtype=torch.float64, device=dev)])
    r = Jsel @ w_t - rhs
    rel_t = float(r.norm() / rhs.norm())
    print(f"ECM residual: reported {rel:.6e}, recomputed {rel_t:.6e}")
    assert abs(rel_t - rel) <= 1e-8 * max(rel, 1e-30) + 1e-14
    ls = torch.linalg.lstsq(Jsel, rhs.unsqueeze(1), driver="gels").solution.squeeze(1)
    positive = bool(torch.all(ls > 0))
    d = float(((ls - w_t).abs() / w_t.abs().max()).max())
    print(f"ECM weights vs unconstrained LS on the selected set: positive {positive}, max rel diff {d:.2e}")
    if positive:
        assert d <= 1e-8
    # the CPU oracle's own full-size selection (tests/golden/make_c4_golden.py:
    # numpy snapshots, numpy POD, oracle stress snapshots, direct-scoring
    # greedy with from-scratch QR refits): ids bit-exact
    from pathlib import Path
    gp = Path(__file__).resolve().parent / "golden" / "c4_ecm_golden.npz"
    if gp.exists():
        gold = np.load(gp)
        print(f"vs golden: ids equal {np.array_equal(ids_np, gold['ids'])}, resid {rel:.9e} vs "
              f"{float(gold['resid_rel']):.9e}, min top-2 gap {gold['top2_gap'].min():.2e}")
        assert np.array_equal(ids_np, gold["ids"])
        assert float(np.abs(np.asarray(w) - gold["weights"]).max() / np.abs(gold["weights"]).max()) <= 1e-8
        assert abs(rel - float(gold["resid_rel"])) <= 1e-8 * float(gold["resid_rel"])
