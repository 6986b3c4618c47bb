"""GPU path vs the committed golden fixtures (no oracle at test time):
BASELINE parity tolerances, bit-exact patterns and ECM ids."""
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


def _mats():
    from paper_2307_16894_b200.api import inclusion_params, matrix_params
    return [matrix_params(), inclusion_params()]


def T(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_material_vs_golden():
    from paper_2307_16894_b200 import api
    d = np.load(G / "material_c1_256.npz")
    r = api.material_batch(T(d["F"]), T(d["st"]), _mats()[:1])
    st = r["status"].cpu().numpy()
    assert np.array_equal(st, d["status"])
    ok = st == 0
    P, A = r["P"].cpu().numpy()[:, ok], r["A"].cpu().numpy()[:, ok]
    rp = np.linalg.norm(P - d["P"][:, ok], axis=0) / np.maximum(np.linalg.norm(d["P"][:, ok], axis=0), 1e-14)
    ra = np.linalg.norm(A - d["A"][:, ok], axis=0) / np.maximum(np.linalg.norm(d["A"][:, ok], axis=0), 1e-14)
    assert rp.max() <= 1e-10 and ra.max() <= 1e-9


def test_assemble_vs_golden():
    from paper_2307_16894_b200 import api
    d = np.load(G / "assemble_8x8.npz")
    g = api.Rve(8, _mats())
    t = g.export()
    assert np.array_equal(t["row_ptr"], d["row_ptr"]) and np.array_equal(t["col_idx"], d["col_idx"])
    a = g.assemble(T(d["fbar"]), T(d["w_red"]), T(d["st0"]), geom=T(d["geom"]))
    for s in range(2):
        f, K = a["f"][s].cpu().numpy(), a["K"][s].cpu().numpy()
        assert np.linalg.norm(f - d["f"][s]) <= 1e-10 * np.linalg.norm(d["f"][s])
        assert np.linalg.norm(K - d["K"][s]) <= 1e-9 * np.linalg.norm(d["K"][s])


def test_rom_vs_golden():
    from paper_2307_16894_b200 import api
    d = np.load(G / "rom_16x16_N10_Q40.npz")
    g = api.Rve(16, _mats())
    rom = api.Rom(g, d["ids"], d["weights"], d["mode_grads"])
    r = rom.solve(T(d["geom"]), T(d["sched"]), api.NewtonOpts(eps_rel=1e-10))
    assert np.array_equal(r["status"].cpu().numpy(), d["status"])
    assert np.array_equal(r["iters"].cpu().numpy(), d["iters"])
    pb = r["pbar"].cpu().numpy()
    assert np.abs(pb - d["pbar"]).max() <= 1e-8 * np.abs(d["pbar"]).max()


def test_pod_ecm_vs_golden():
    from paper_2307_16894_b200 import api
    d = np.load(G / "pod_ecm_12x12.npz")
    g = api.Rve(12, _mats())
    mt, ev = api.pod(T(d["U"].T), 5)
    ev = ev.cpu().numpy()
    assert np.abs(ev[:5] - d["evals"][:5]).max() <= 1e-10 * d["evals"][0]
    W, st = api.ecm_stress_snapshots(g, T(d["U"].T))
    H = api.ecm_mode_grads(g, T(d["modes"].T))
    ids, w, rel, it = api.ecm_select(g, H, W, api.EcmOpts(eps=1e-10, max_points=20, stop_at_count=True))
    assert np.array_equal(ids, d["ids"])
    assert np.abs(w - d["weights"]).max() <= 1e-8 * np.abs(d["weights"]).max()
