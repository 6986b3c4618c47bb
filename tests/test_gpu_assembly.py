"""K2 parity: batched Q4 assembly (configs 0 and 2) vs the CPU oracle.

Bit-exact: mesh tables, quadrature cache, periodic dof map, CSR pattern
(row_ptr / col_idx) and the morph (no transcendental on that path).
Tolerances: residual 1e-10 (vector 2-norm relative), K 1e-9
(||dK||_F / ||K||_F per instance), history 1e-10 per point.
"""
import numpy as np
import pytest

from paper_2307_16894_b200 import synth

pytestmark = pytest.mark.gpu


def _mats():
    from paper_2307_16894_b200.api import inclusion_params, matrix_params
    return [matrix_params(), inclusion_params()]


@pytest.fixture(scope="module")
def pair64(orc):
    from paper_2307_16894_b200 import api
    return api.Rve(64, _mats()), orc.Rve(64, _mats())


@pytest.fixture(scope="module")
def pair128(orc):
    from paper_2307_16894_b200 import api
    return api.Rve(128, _mats()), orc.Rve(128, _mats())


def test_tables_bit_exact(pair64):
    g, o = pair64
    tg, to = g.export(), o.export()
    assert (g.n_red, g.nnz) == (8190, 147388)
    for k in ("nodes", "elems", "regions", "grad", "w", "node_dof", "row_ptr", "col_idx"):
        assert np.array_equal(tg[k], to[k]), k


def test_tables_bit_exact_128(pair128):
    g, o = pair128
    assert (g.n_red, g.nnz) == (32766, 589756)
    tg, to = g.export(), o.export()
    for k in ("row_ptr", "col_idx", "node_dof", "grad", "w"):
        assert np.array_equal(tg[k], to[k]), k


def test_morph_bit_exact(pair64):
    import torch
    g, o = pair64
    geom = torch.tensor([[0.3, 0.2], [0.15, 0.35]], dtype=torch.float64, device="cuda")
    fmi, det, st = g.morph(geom)
    for s, (a, b) in enumerate(((0.3, 0.2), (0.15, 0.35))):
        ofmi, odet, rc = o.morph(a, b)
        assert rc == 0 and int(st[s]) == 0
        assert np.array_equal(fmi[s].cpu().numpy(), ofmi)
        assert np.array_equal(det[s].cpu().numpy(), odet)


def _assemble_both(g, o, n_inst, seed, hm, geom_range=None):
    import torch
    tg = g.export()
    regions_qp = np.repeat(tg["regions"], 4)
    geom, fbar, w_red, st0 = synth.rve_instances(n_inst, g.n_red, regions_qp, seed, hm,
                                                 geom_range=geom_range)
    dev = torch.device("cuda:0")
    T = lambda a: torch.from_numpy(a).to(dev)
    rg = g.assemble(T(fbar), T(w_red), T(st0), geom=T(geom), store_stress=True)
    torch.cuda.synchronize()
    rg = {k: v.cpu().numpy() for k, v in rg.items() if v is not None}
    ro = o.assemble(geom, fbar, w_red, st0, store_stress=True)
    return rg, ro


def _check(rg, ro, n_inst):
    assert np.array_equal(rg["status"], ro["status"])
    for s in range(n_inst):
        ef = np.linalg.norm(rg["f"][s] - ro["f"][s]) / np.linalg.norm(ro["f"][s])
        eK = np.linalg.norm(rg["K"][s] - ro["K"][s]) / np.linalg.norm(ro["K"][s])
        dP = rg["p_field"][s] - ro["p_field"][s]
        eP = (np.sqrt((dP ** 2).sum(0)) / np.maximum(np.sqrt((ro["p_field"][s] ** 2).sum(0)), 1e-14)).max()
        dS = rg["st1"][s] - ro["st1"][s]
        eS = (np.sqrt((dS ** 2).sum(0)) / np.maximum(np.sqrt((ro["st1"][s] ** 2).sum(0)), 1e-14)).max()
        print(f"inst {s}: f {ef:.2e} K {eK:.2e} P {eP:.2e} st {eS:.2e} "
              f"K bitwise {np.mean(rg['K'][s] == ro['K'][s]):.4f}")
        assert ef <= 1e-10 and eP <= 1e-10 and eS <= 1e-10 and eK <= 1e-9


def test_config0_single_rve(pair64):
    g, o = pair64
    rg, ro = _assemble_both(g, o, 1, 2026, 0.1)
    _check(rg, ro, 1)


def test_config2_instances(pair128):
    g, o = pair128
    rg, ro = _assemble_both(g, o, 3, 2028, 0.2, geom_range=(0.15, 0.35))
    _check(rg, ro, 3)


def test_residual_only_matches_full(pair64):
    """AssemblyOpts.tangent = false gives the same residual and history."""
    import torch
    g, _ = pair64
    tg = g.export()
    geom, fbar, w_red, st0 = synth.rve_instances(2, g.n_red, np.repeat(tg["regions"], 4), 5, 0.1)
    T = lambda a: torch.from_numpy(a).cuda()
    a = g.assemble(T(fbar), T(w_red), T(st0), geom=T(geom))
    b = g.assemble(T(fbar), T(w_red), T(st0), geom=T(geom), tangent=False)
    assert torch.equal(a["f"], b["f"]) and torch.equal(a["st1"], b["st1"])


def test_morph_field_input_equals_geom(pair64):
    """Passing the MorphField (fmu_inv, det) instead of (a, b) is identical."""
    import torch
    g, _ = pair64
    tg = g.export()
    geom, fbar, w_red, st0 = synth.rve_instances(2, g.n_red, np.repeat(tg["regions"], 4), 6, 0.1,
                                                 geom_range=(0.15, 0.35))
    T = lambda a: torch.from_numpy(a).cuda()
    fmi, det, _ = g.morph(T(geom))
    morph = torch.cat([fmi, det[:, None, :]], 1).contiguous()
    a = g.assemble(T(fbar), T(w_red), T(st0), geom=T(geom))
    b = g.assemble(T(fbar), T(w_red), T(st0), morph=morph)
    assert torch.equal(a["f"], b["f"]) and torch.equal(a["K"], b["K"])


def test_deterministic(pair64):
    import torch
    g, _ = pair64
    tg = g.export()
    geom, fbar, w_red, st0 = synth.rve_instances(1, g.n_red, np.repeat(tg["regions"], 4), 9, 0.1)
    T = lambda a: torch.from_numpy(a).cuda()
    a = g.assemble(T(fbar), T(w_red), T(st0), geom=T(geom))
    b = g.assemble(T(fbar), T(w_red), T(st0), geom=T(geom))
    assert torch.equal(a["K"], b["K"]) and torch.equal(a["f"], b["f"])


def test_empty_batch(pair64):
    import torch
    g, _ = pair64
    z = lambda *s: torch.zeros(*s, dtype=torch.float64, device="cuda")
    r = g.assemble(z(0, 4), z(0, g.n_red), z(0, 6, g.n_qp), geom=z(0, 2))
    assert r["f"].shape == (0, g.n_red) and r["status"].numel() == 0


def test_failed_instance_is_isolated(pair64):
    """A singular macro gradient fails its instance only (SolveError status,
    microfem.cpp:76 via material.cpp:128-130); the neighbours are unaffected
    and still match the oracle."""
    import torch
    g, o = pair64
    tg = g.export()
    geom, fbar, w_red, st0 = synth.rve_instances(3, g.n_red, np.repeat(tg["regions"], 4), 11, 0.1)
    fbar[1] = 0.0
    w_red[1] = 0.0
    T = lambda a: torch.from_numpy(a).cuda()
    rg = g.assemble(T(fbar), T(w_red), T(st0), geom=T(geom), store_stress=True)
    st = rg["status"].cpu().numpy()
    ro = o.assemble(geom, fbar, w_red, st0, store_stress=True)
    print("status gpu", st, "oracle", ro["status"])
    assert st[1] != 0 and st[0] == 0 and st[2] == 0
    assert np.array_equal(st, ro["status"])
    with pytest.raises(Exception):
        g.ctx.check()
    rg = {k: v.cpu().numpy() for k, v in rg.items() if v is not None}
    for s in (0, 2):
        assert np.linalg.norm(rg["f"][s] - ro["f"][s]) <= 1e-10 * np.linalg.norm(ro["f"][s])
        assert np.linalg.norm(rg["K"][s] - ro["K"][s]) <= 1e-9 * np.linalg.norm(ro["K"][s])


@pytest.mark.parametrize("n_inst", [1, 3])
def test_exact_order_mode_bitwise(pair64, monkeypatch, n_inst):
    """PODECM_ASM_EXACT=1: every qp's 64 K-terms and 8 f-terms in the
    reference's expression order, each CSR slot and residual row summed in
    setFromTriplets' order (microfem.cpp:76-128) — with the bitwise material
    (glibc exp/log on the device) the whole assembly equals the oracle BIT FOR
    BIT: f, K values, stresses and history (config 0)."""
    g, o = pair64
    monkeypatch.setenv("PODECM_ASM_EXACT", "1")
    rg, ro = _assemble_both(g, o, n_inst, 2026 + n_inst, 0.1, geom_range=(0.15, 0.35) if n_inst > 1 else None)
    assert np.array_equal(rg["status"], ro["status"])
    for k, ko in (("f", "f"), ("K", "K"), ("p_field", "p_field"), ("st1", "st1")):
        ndiff = int((rg[k].view(np.int64) != ro[ko].view(np.int64)).sum())
        print(f"exact mode, {k}: {ndiff} of {rg[k].size} values differ")
        assert ndiff == 0, k


@pytest.mark.parametrize("n_cells,n_inst", [(64, 3), (16, 5)])
def test_tiled_assembly_bitwise_equals_gathered(monkeypatch, n_cells, n_inst):
    """The tiled default (8 x 4 element tiles: items whose element sums all
    come from one tile are summed in shared memory, the rest through the halo
    gather) adds every CSR slot and residual row in the same group order as
    the all-gather path (PODECM_ASM_TILED=0): K, f and the history are
    bit-identical, with and without the tangent."""
    import torch
    from paper_2307_16894_b200 import api
    g = api.Rve(n_cells, _mats())
    tg = g.export()
    geom, fbar, w_red, st0 = synth.rve_instances(n_inst, g.n_red, np.repeat(tg["regions"], 4), 90 + n_cells, 0.15,
                                                 geom_range=(0.15, 0.35))
    T = lambda a: torch.from_numpy(a).cuda()
    res = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("PODECM_ASM_TILED", mode)
        a = g.assemble(T(fbar), T(w_red), T(st0), geom=T(geom))
        b = g.assemble(T(fbar), T(w_red), T(st0), geom=T(geom), tangent=False)
        torch.cuda.synchronize()
        res[mode] = (a, b)
    for k in ("f", "K", "st1"):
        assert torch.equal(res["1"][0][k], res["0"][0][k]), k
    assert torch.equal(res["1"][1]["f"], res["0"][1]["f"])
    assert torch.equal(res["1"][0]["f"], res["1"][1]["f"])
