"""§8(f) row 2: batched RomMicroEngine (twoscale.cpp:53-96) on the GPU vs the
oracle's restatement.  A macro-Newton-like sequence: per load step several
trial macro gradients are answered from the committed history, then the
step is committed.  pbar within 1e-8 and Newton iteration counts and
out-of-range counters equal vs the glibc oracle.

Abar has a conditioning floor here that the converged-step test does not:
after a plastic commit the history sits on the yield surface, so for the
next trial gradients many ECM points have f_trial ~ 0 and the yield kink
falls inside the reference's FD interval [F - h, F + h] (h = 1e-7 |F|).
The FD column then moves by (slope jump) * dF / h for a shift dF of F, so
ulp differences in F become ~1e-7 in Abar.  The device material is bitwise
the glibc oracle's (tests/test_gpu_material_fullscale.py), so the remaining
ulp differences in F are summation order: F = Fbar + R(Fmu^-1)^T (G_p^T a)
and the reduced coordinates a come out of a DMMA contraction and a warp LU,
neither in Eigen's (nor the oracle's) order — the reference's own Eigen
GEMV/GEMM order is not reproducible by any other implementation.  The size
of that floor is measured in the same run by two CPU oracles that differ
only at the ulp level (glibc vs the portable exp/log): the criterion is
normwise Abar difference (relative to max(1, ||Abar||)) vs either oracle
<= max(1e-8, 10 x the oracle-vs-oracle difference) and <= 1e-6.  P-bar
(no FD) stays within 1e-8 and the Newton counts are equal."""
import numpy as np
import pytest

from paper_2307_16894_b200 import synth

pytestmark = pytest.mark.gpu


def _mats():
    from paper_2307_16894_b200.api import inclusion_params, matrix_params
    return [matrix_params(), inclusion_params()]


def _T(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("max_iter", [25, 3])  # 3: trials that need bisection
def test_engines_macro_sequence(orc, max_iter):
    import oracle
    from paper_2307_16894_b200 import api
    g = api.Rve(64, _mats())
    o = orc.Rve(64, _mats())
    model = synth.rom_model(g.export(), g.n_red, N=24, Q=120, seed=2035)
    rom = api.Rom(g, model["ids"], model["weights"], model["mode_grads"])
    n = 8
    rng = np.random.default_rng(2036)
    geom = rng.uniform(0.15, 0.35, (n, 2))
    H = rng.uniform(-0.15, 0.15, (n, 4))
    bounds = [(0.95, 1.08), (0.95, 1.08), (-0.06, 0.06)]
    opts = api.NewtonOpts(eps_rel=1e-10, eps_abs=1e-12, max_iter=max_iter, max_bisect=5)
    eg = api.RomEngines(rom, _T(geom), stretch_bounds=bounds)
    eo = oracle.RomEngines(o, model["ids"], model["weights"], model["mode_grads"], geom, bounds=bounds,
                           eps_rel=opts.eps_rel, eps_abs=opts.eps_abs, max_iter=max_iter, max_bisect=5)
    op = orc.Rve(64, _mats(), libm="pdm")
    ep = oracle.RomEngines(op, model["ids"], model["weights"], model["mode_grads"], geom, bounds=bounds,
                           eps_rel=opts.eps_rel, eps_abs=opts.eps_abs, max_iter=max_iter, max_bisect=5)
    worst_p = worst_a = worst_same = worst_oo = 0.0
    for k in range(1, 5):
        for j in range(3):  # macro Newton iterates around the step's target
            fb = np.array([1.0, 0.0, 0.0, 1.0]) + (k / 4) * H + (0.01 / (j + 1)) * rng.normal(size=(n, 4)) * (j < 2)
            rg = eg.respond(_T(fb), opts, abar=True)
            rg = {kk: v.cpu().numpy() for kk, v in rg.items()}
            ro = eo.respond(fb, abar=True)
            rp = ep.respond(fb, abar=True)
            assert np.array_equal(rg["status"], ro["status"]), (rg["status"], ro["status"])
            ok = ro["status"] == 0
            assert np.array_equal(rg["iters"][ok], ro["iters"][ok]), (k, j, rg["iters"], ro["iters"])
            dp = np.linalg.norm(rg["pbar"][ok] - ro["pbar"][ok], axis=-1) / np.maximum(
                1.0, np.linalg.norm(ro["pbar"][ok], axis=-1))
            da = np.linalg.norm(rg["abar"][ok] - ro["abar"][ok], axis=-1) / np.maximum(
                1.0, np.linalg.norm(ro["abar"][ok], axis=-1))
            worst_p = max(worst_p, dp.max(initial=0.0))
            worst_a = max(worst_a, da.max(initial=0.0))
            okp = (rp["status"] == 0) & ok
            ds = np.linalg.norm(rg["abar"][okp] - rp["abar"][okp], axis=-1) / np.maximum(
                1.0, np.linalg.norm(rp["abar"][okp], axis=-1))
            worst_same = max(worst_same, ds.max(initial=0.0))
            do = np.linalg.norm(ro["abar"][okp] - rp["abar"][okp], axis=-1) / np.maximum(
                1.0, np.linalg.norm(ro["abar"][okp], axis=-1))
            worst_oo = max(worst_oo, do.max(initial=0.0))
        eg.commit()
        eo.commit()
        ep.commit()
    print(f"engines: pbar rel {worst_p:.3e}  abar rel vs same-libm oracle {worst_same:.3e}, "
          f"vs glibc oracle {worst_a:.3e}, oracle vs oracle {worst_oo:.3e}  out_of_range {eo.out_of_range()}")
    floor = max(1e-8, 10.0 * worst_oo)
    assert worst_p <= 1e-8
    assert worst_same <= min(floor, 1e-6) and worst_a <= min(floor, 1e-6)
    assert np.array_equal(eg.out_of_range().cpu().numpy(), eo.out_of_range())
