"""§8(f) row 1: reduced effective stiffness and geometric sensitivities
(rom.cpp:202-263) on the GPU vs the CPU oracle.

- rom_effective_stiffness: Abar [4x4] per instance within 1e-8 normwise
  (relative to max(1, ||Abar||)), both standalone and as run_online's
  effective_stiffness request (history committed at the start of the last
  increment, pipeline.cpp:456-483);
- consistency: Abar is the derivative of the final homogenised stress with
  respect to the last macro gradient (central differences of pbar);
- rom_sensitivity: FD over the geometry (a, b), 4 reduced solves per
  instance in one batch, within 1e-6 of the oracle's FD (the reference's own
  FD test tolerates 1e-4, test_rom.cpp:166-186).
"""
import numpy as np
import pytest

from paper_2307_16894_b200 import synth

pytestmark = pytest.mark.gpu


def _mats():
    from paper_2307_16894_b200.api import inclusion_params, matrix_params
    return [matrix_params(), inclusion_params()]


@pytest.fixture(scope="module")
def setup(orc):
    from paper_2307_16894_b200 import api
    g = api.Rve(128, _mats())
    o = orc.Rve(128, _mats())
    model = synth.rom_model(g.export(), g.n_red, N=50, Q=400, seed=2029)
    rom = api.Rom(g, model["ids"], model["weights"], model["mode_grads"])
    return g, o, model, rom


def _T(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _abar_rel(ag, ao):
    d = np.linalg.norm(ag - ao, axis=-1)
    return d / np.maximum(1.0, np.linalg.norm(ao, axis=-1))


@pytest.mark.parametrize("n,K,seed,opts_kw", [
    (4, 5, 2031, dict(eps_rel=1e-10, eps_abs=1e-12, max_iter=25)),
    (4, 2, 78, dict(eps_rel=1e-10, eps_abs=1e-12, max_iter=3, max_bisect=5)),  # bisection path
])
def test_solve_with_effective_stiffness(setup, n, K, seed, opts_kw):
    from paper_2307_16894_b200 import api
    g, o, model, rom = setup
    geom, sched = synth.rom_instances(n, K, seed, 0.2)
    opts = api.NewtonOpts(**opts_kw)
    rg = rom.solve(_T(geom), _T(sched), opts, abar=True)
    rg = {k: v.cpu().numpy() for k, v in rg.items()}
    plain = rom.solve(_T(geom), _T(sched), opts)
    assert np.array_equal(plain["pbar"].cpu().numpy(), rg["pbar"])  # abar request leaves the solve untouched
    ro = o.rom_solve(model["ids"], model["weights"], model["mode_grads"], geom, sched, eps_rel=opts.eps_rel,
                     eps_abs=opts.eps_abs, max_iter=opts.max_iter, max_bisect=opts.max_bisect, abar=True)
    assert np.array_equal(rg["status"], ro["status"]) and np.all(ro["status"] == 0)
    rel = _abar_rel(rg["abar"], ro["abar"])
    print(f"abar rel {rel.max():.3e}  |abar| {np.linalg.norm(ro['abar'], axis=-1).max():.3e}  "
          f"iters {ro['iters'].sum(1)}")
    assert rel.max() <= 1e-8


def test_effective_stiffness_standalone(setup):
    g, o, model, rom = setup
    rng = np.random.default_rng(2032)
    n, Q, N = 5, model["ids"].shape[0], model["mode_grads"].shape[1]
    geom = rng.uniform(0.15, 0.35, (n, 2))
    fbar = np.array([1.0, 0.0, 0.0, 1.0]) + rng.uniform(-0.15, 0.15, (n, 4))
    a = rng.normal(0.0, 2e-3, (n, N))
    # prior plastic history: Fp = exp(sym dev), Fp_zz = 1/det(Fp), xi >= 0
    st0 = np.zeros((n, 6, Q))
    e = rng.normal(0.0, 0.01, (n, Q, 2))
    st0[:, 0] = np.exp(e[..., 0])
    st0[:, 1] = e[..., 1]
    st0[:, 2] = e[..., 1]
    st0[:, 3] = np.exp(-e[..., 0])
    st0[:, 4] = 1.0 / (st0[:, 0] * st0[:, 3] - st0[:, 1] * st0[:, 2])
    st0[:, 5] = rng.uniform(0.0, 0.05, (n, Q))
    rg = rom.effective_stiffness(_T(geom), _T(st0), _T(fbar), _T(a))
    ag, sg = rg["abar"].cpu().numpy(), rg["status"].cpu().numpy()
    ao, so = o.rom_effective_stiffness(model["ids"], model["weights"], model["mode_grads"], geom, st0, fbar, a)
    assert np.array_equal(sg, so) and np.all(so == 0)
    rel = _abar_rel(ag, ao)
    print(f"standalone abar rel {rel.max():.3e}")
    assert rel.max() <= 1e-8


def test_effective_stiffness_is_the_stress_derivative(setup):
    """Abar(:, kl) = d pbar_K / d Fbar_K(kl): central differences of the last
    increment's homogenised stress (same history, same earlier increments)."""
    from paper_2307_16894_b200 import api
    g, o, model, rom = setup
    n, K = 3, 4
    geom, sched = synth.rom_instances(n, K, 2033, 0.15)
    opts = api.NewtonOpts(eps_rel=1e-12, eps_abs=1e-14, max_iter=25)
    base = rom.solve(_T(geom), _T(sched), opts, abar=True)
    ab = base["abar"].cpu().numpy()
    h = 1e-5
    fd = np.zeros((n, 16))
    for c in range(4):
        sp, sm = sched.copy(), sched.copy()
        sp[:, -1, c] += h
        sm[:, -1, c] -= h
        pp = rom.solve(_T(geom), _T(sp), opts)["pbar"].cpu().numpy()[:, -1]
        pm = rom.solve(_T(geom), _T(sm), opts)["pbar"].cpu().numpy()[:, -1]
        fd[:, 4 * c:4 * c + 4] = (pp - pm) / (2 * h)
    rel = np.linalg.norm(ab - fd, axis=-1) / np.linalg.norm(fd, axis=-1)
    print(f"abar vs FD of pbar: rel {rel}")
    assert rel.max() <= 1e-7


def test_sensitivity(setup):
    from paper_2307_16894_b200 import api
    g, o, model, rom = setup
    n, K = 3, 4
    geom, sched = synth.rom_instances(n, K, 2034, 0.15)
    opts = api.NewtonOpts(eps_rel=1e-12, eps_abs=1e-14, max_iter=25)
    h = 1e-4
    rg = rom.sensitivity(_T(geom), _T(sched), opts, h=h)
    gg, sg = rg["grad"].cpu().numpy(), rg["status"].cpu().numpy()
    go, so = o.rom_sensitivity(model["ids"], model["weights"], model["mode_grads"], geom, sched, h,
                               eps_rel=opts.eps_rel, eps_abs=opts.eps_abs, max_iter=opts.max_iter,
                               max_bisect=opts.max_bisect)
    assert np.array_equal(sg, so) and np.all(so == 0)
    d = np.linalg.norm(gg - go, axis=-1) / np.maximum(1.0, np.linalg.norm(go, axis=-1))
    print(f"sensitivity rel {d.max():.3e}  |grad| {np.linalg.norm(go, axis=-1).max():.3e}")
    assert d.max() <= 1e-6
