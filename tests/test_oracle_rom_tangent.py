"""Oracle pin for rom_effective_stiffness / rom_sensitivity (rom.cpp:202-263):
the restated Abar is the derivative of the final homogenised stress with
respect to the last macro gradient (the property behind the reference's
ExactLimit.EffectiveStiffnessMatches, test_rom.cpp:127-156), and the
sensitivity equals its own definition from two rom_solve runs."""
import numpy as np
import pytest

from paper_2307_16894_b200 import synth


@pytest.fixture(scope="module")
def small(orc):
    from paper_2307_16894_b200.api import inclusion_params, matrix_params
    o = orc.Rve(16, [matrix_params(), inclusion_params()])
    m = synth.rom_model(o.export(), o.n_red, N=10, Q=60, seed=1)
    return o, m


def test_abar_is_stress_derivative(small):
    o, m = small
    geom, sched = synth.rom_instances(3, 4, 5, 0.15)
    kw = dict(eps_rel=1e-12, eps_abs=1e-14)
    r = o.rom_solve(m["ids"], m["weights"], m["mode_grads"], geom, sched, abar=True, **kw)
    assert np.all(r["status"] == 0)
    h = 1e-5
    fd = np.zeros((3, 16))
    for c in range(4):
        sp, sm = sched.copy(), sched.copy()
        sp[:, -1, c] += h
        sm[:, -1, c] -= h
        pp = o.rom_solve(m["ids"], m["weights"], m["mode_grads"], geom, sp, **kw)["pbar"][:, -1]
        pm = o.rom_solve(m["ids"], m["weights"], m["mode_grads"], geom, sm, **kw)["pbar"][:, -1]
        fd[:, 4 * c:4 * c + 4] = (pp - pm) / (2 * h)
    rel = np.linalg.norm(r["abar"] - fd, axis=-1) / np.linalg.norm(fd, axis=-1)
    assert rel.max() < 1e-6, rel


def test_standalone_equals_run_online_request(small):
    """rom_effective_stiffness called with the last increment's start
    history (virgin for K = 1), fbar and final a equals the solve's abar."""
    o, m = small
    geom, sched = synth.rom_instances(2, 1, 6, 0.15)
    r = o.rom_solve(m["ids"], m["weights"], m["mode_grads"], geom, sched, abar=True)
    Q = m["ids"].shape[0]
    st0 = np.zeros((2, 6, Q))
    st0[:, 0] = st0[:, 3] = st0[:, 4] = 1.0
    ab, st = o.rom_effective_stiffness(m["ids"], m["weights"], m["mode_grads"], geom, st0,
                                       sched[:, -1], r["a_final"])
    assert np.all(st == 0)
    assert np.array_equal(ab, r["abar"])


def test_sensitivity_definition(small):
    o, m = small
    geom, sched = synth.rom_instances(2, 3, 7, 0.15)
    h = 1e-4
    g, st = o.rom_sensitivity(m["ids"], m["weights"], m["mode_grads"], geom, sched, h)
    assert np.all(st == 0)
    k = 1
    step = h * np.maximum(1.0, np.abs(geom[:, k]))
    lo, hi = geom.copy(), geom.copy()
    lo[:, k] -= step
    hi[:, k] += step
    pl = o.rom_solve(m["ids"], m["weights"], m["mode_grads"], lo, sched)["pbar"][:, -1]
    ph = o.rom_solve(m["ids"], m["weights"], m["mode_grads"], hi, sched)["pbar"][:, -1]
    assert np.array_equal(g[:, k], (ph - pl) / (2.0 * step)[:, None])


def test_engine_first_response_equals_rom_solve(small):
    """RomMicroEngine::respond from the virgin state is rom_solve_step_adaptive
    from (I, a = 0): the first response equals a one-increment rom_solve, and
    responding twice without commit gives the same answer (twoscale.cpp:65-89)."""
    import oracle
    o, m = small
    geom, sched = synth.rom_instances(3, 1, 8, 0.15)
    e = oracle.RomEngines(o, m["ids"], m["weights"], m["mode_grads"], geom)
    r1 = e.respond(sched[:, 0], abar=True)
    r2 = e.respond(sched[:, 0], abar=True)
    rs = o.rom_solve(m["ids"], m["weights"], m["mode_grads"], geom, sched, abar=True)
    assert np.array_equal(r1["pbar"], rs["pbar"][:, 0]) and np.array_equal(r1["abar"], rs["abar"])
    assert np.array_equal(r1["iters"], rs["iters"][:, 0])
    assert np.array_equal(r1["pbar"], r2["pbar"])


def test_oracle_full_order_newton_matches_dense_python(orc):
    """oracle fe_solve (C++, microfem.cpp:142-238 with bisection) agrees with
    the independent Python Newton of oracle/fe.py on a case without bisection."""
    from oracle.fe import fe_newton_pbar
    from paper_2307_16894_b200.api import inclusion_params, matrix_params
    o = orc.Rve(8, [matrix_params(), inclusion_params()])
    t = o.export()
    geom, sched = synth.rom_instances(2, 3, 5, 0.15)
    r = o.fe_solve(geom, sched, eps_rel=1e-10)
    assert np.all(r["status"] == 0)
    for s in range(2):
        ref = fe_newton_pbar(o, t, tuple(geom[s]), sched[s])
        assert np.abs(r["pbar"][s] - ref).max() <= 1e-12 * np.abs(ref).max()


def test_oracle_twoscale_linear_engine_is_single_scale(orc):
    """test_twoscale.cpp:93-134: with the linear engine the FE2 driver is the
    single-scale linear problem, so compliance = factor^2 x const and the
    unloaded plate returns to u = 0."""
    r, st = orc.run_twoscale(nx=2, ny=1, steps=10, peak=0.02, E=1.0, nu=0.3)
    assert st == 0
    lf = r["load_factor"]
    ratio = r["compliance"][lf > 0] / lf[lf > 0] ** 2
    assert np.abs(ratio / ratio[0] - 1.0).max() <= 1e-10
    assert r["residual_norm"] <= 1e-12
    assert np.all(r["iters"] == 1)
