"""The reference-signature drop-in (paper_2307_16894_b200/dropin/
podecm_dropin.cpp), compiled against the reference's own headers, against the
reference's own sources (oracle/_ref: material.cpp, microfem.cpp, rom.cpp
compiled unchanged): the functions a reference caller links —
large_strain_update / large_strain_tangent (material.hpp:69-75), assemble
(microfem.hpp:74-77), rom_solve (rom.hpp:86-88) — and their batch forms.

  * material: P, the FD tangent, the history and dgamma / f_trial / q_trial /
    mises BIT FOR BIT, and the same SolveError points, per call and batched;
  * assemble: the exact-order device mode bit for bit (f, K(r, c) on the
    pattern, stresses, history); the default mode within the BASELINE
    tolerances (1e-10 residual, 1e-9 tangent);
  * rom_solve: P-bar histories within 1e-12 and Newton counts equal per
    increment, RomSolution::steps[k].a within 1e-9, bisection exercised.

Both libraries are built in the build container (the reference sources are
not on the GPU box) and travel with the repository snapshot."""
import numpy as np
import pytest

from paper_2307_16894_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref(orc):
    if not (orc.ref_available() and orc.dropin_available()):
        pytest.skip("oracle/_ref or the drop-in test library was not built")
    return orc


def _mats():
    from paper_2307_16894_b200.api import inclusion_params, matrix_params
    return [matrix_params(), inclusion_params()]


def _same(a, b):
    return np.array_equal(a.view(np.int64), b.view(np.int64))


@pytest.mark.parametrize("per_call", [1, 0])
def test_dropin_material_bitwise(ref, per_call):
    from paper_2307_16894_b200.api import matrix_params
    n = 512 if per_call else 1 << 16
    F, st = synth.config1_points(n, 61)
    F[:, :8] = 0.0  # singular: SolveError on both sides
    r = ref.ref_material_batch(F, st, matrix_params())
    d = ref.dropin_material(F, st, matrix_params(), per_call)
    assert np.array_equal(r["status"], d["status"]) and (r["status"] != 0).sum() == 8
    ok = r["status"] == 0
    for k in ("P", "A", "st", "extra"):
        assert _same(r[k][:, ok], d[k][:, ok]), k


@pytest.mark.parametrize("exact", [True, False])
def test_dropin_assemble(ref, monkeypatch, exact):
    if exact:
        monkeypatch.setenv("PODECM_ASM_EXACT", "1")
    else:
        monkeypatch.delenv("PODECM_ASM_EXACT", raising=False)
    n_cells = 16
    o = ref.Rve(n_cells, _mats())
    t = o.export()
    geom, fbar, w_red, st0 = synth.rve_instances(1, o.n_red, np.repeat(t["regions"], 4), 71, 0.1,
                                                 geom_range=(0.15, 0.35))
    fmi, det, rc = o.morph(*geom[0])
    rc_r, r = ref.ref_assemble(n_cells, t, _mats(), fmi, det, st0[0], fbar[0], w_red[0])
    rc_d, d = ref.dropin_assemble(n_cells, t, _mats(), fmi, det, st0[0], fbar[0], w_red[0])
    assert rc_r == 0 and rc_d == 0
    if exact:
        for k in ("f", "K", "p_field", "st1"):
            assert _same(r[k], d[k]), k
    else:
        ef = np.linalg.norm(d["f"] - r["f"]) / np.linalg.norm(r["f"])
        eK = np.linalg.norm(d["K"] - r["K"]) / np.linalg.norm(r["K"])
        print(f"default mode vs reference source: f {ef:.2e} K {eK:.2e}")
        assert ef <= 1e-10 and eK <= 1e-9
        assert _same(r["p_field"], d["p_field"]) and _same(r["st1"], d["st1"])


def test_dropin_assemble_rejects_foreign_mesh(ref):
    """A mesh outside the device path raises ConfigError (rc 2), never a
    silent host fallback: here a quadrature cache that differs from the Q4
    cell's."""
    n_cells = 8
    o = ref.Rve(n_cells, _mats())
    t = dict(o.export())
    t["w"] = t["w"] * 1.5
    nq = t["w"].shape[0]
    fmi = np.tile(np.array([1.0, 0.0, 0.0, 1.0])[:, None], (1, nq))
    st0 = np.tile(np.array([1.0, 0.0, 0.0, 1.0, 1.0, 0.0])[:, None], (1, nq))
    rc, _ = ref.dropin_assemble(n_cells, t, _mats(), fmi, np.ones(nq), st0, np.array([1.0, 0, 0, 1.0]),
                                np.zeros(o.n_red))
    assert rc == 2


@pytest.mark.parametrize("per_call,max_iter", [(1, 25), (0, 3)])
def test_dropin_rom_solve(ref, per_call, max_iter):
    n_cells, N, Q, n, K = 16, 10, 40, 8, 6
    o = ref.Rve(n_cells, _mats())
    t = o.export()
    model = synth.rom_model(t, o.n_red, N=N, Q=Q, seed=5)
    geom, sched = synth.rom_instances(n, K, 6, 0.2)
    fmi_q, det_q = np.empty((n, Q, 4)), np.empty((n, Q))
    for s in range(n):
        fmi, det, rc = o.morph(*geom[s])
        fmi_q[s] = fmi[:, model["ids"]].T
        det_q[s] = det[model["ids"]]
    kw = dict(eps_rel=1e-10, eps_abs=1e-12, max_iter=max_iter)
    r = ref.ref_rom_solve(n_cells, t["regions"], _mats(), model["ids"], model["weights"], model["mode_grads"],
                          fmi_q, det_q, sched, **kw)
    d = ref.dropin_rom_solve(n_cells, t, _mats(), model["ids"], model["weights"], model["mode_grads"], fmi_q, det_q,
                             sched, per_call=bool(per_call), **kw)
    assert np.array_equal(r["status"], d["status"])
    ok = r["status"] == 0
    assert np.array_equal(r["iters"][ok], d["iters"][ok])
    dp = np.abs(r["pbar"][ok] - d["pbar"][ok]).max() / np.abs(r["pbar"][ok]).max()
    da = np.abs(r["a_final"][ok] - d["a_hist"][ok][:, -1]).max() / np.abs(r["a_final"][ok]).max()
    print(f"rom_solve drop-in (per_call {per_call}, max_iter {max_iter}): pbar {dp:.2e}, a {da:.2e}, "
          f"iters {r['iters'][ok].sum()}")
    assert dp <= 1e-12 and da <= 1e-9
    if max_iter == 3:
        assert (r["iters"][ok] > 3).any()
