"""§8(f) item 2: the FE2 macro driver (run_twoscale, twoscale.cpp:131-242)
around the batched micro engines, vs the oracle's restatement.  Linear
engine: the single-scale plate (compliance to 1e-12).  ROM engines: a small
hyper-reduced RVE at every macro Gauss point, elasto-plastic loading and
unloading; compliance history and final displacement within 1e-8 and equal
macro Newton iteration counts."""
import numpy as np
import pytest

from paper_2307_16894_b200 import synth

pytestmark = pytest.mark.gpu


def _mats():
    from paper_2307_16894_b200.api import inclusion_params, matrix_params
    return [matrix_params(), inclusion_params()]


def test_linear_engine_matches_oracle(orc):
    from paper_2307_16894_b200 import api
    cfg = api.MacroConfig(nx=5, ny=3, steps=6, peak_traction=0.02)
    rg = api.run_twoscale(cfg, None, E=1.0, nu=0.3)
    ro, st = orc.run_twoscale(nx=5, ny=3, steps=6, peak=0.02, E=1.0, nu=0.3)
    assert st == 0
    rel = np.abs(rg["compliance"] - ro["compliance"]).max() / np.abs(ro["compliance"]).max()
    print(f"linear FE2: compliance rel {rel:.2e}")
    assert rel <= 1e-12 and np.array_equal(rg["iters"], ro["iters"])
    assert rg["micro_evals"] == 6 * 2 * cfg.info()["n_qp"]


def test_rom_engines_match_oracle(orc):
    import oracle
    import torch
    from paper_2307_16894_b200 import api
    g = api.Rve(8, _mats())
    o = orc.Rve(8, _mats())
    model = synth.rom_model(g.export(), g.n_red, N=8, Q=30, seed=2050)
    rom = api.Rom(g, model["ids"], model["weights"], model["mode_grads"])
    cfg = api.MacroConfig(nx=2, ny=1, steps=6, peak_traction=0.02,
                          newton=api.NewtonOpts(eps_rel=1e-9, eps_abs=1e-12, max_iter=25))
    x = cfg.qp_positions()
    geom = np.stack([0.2 + 0.1 * x[:, 0] / 2.0, 0.3 - 0.1 * x[:, 1]], 1)  # graded (a, b) field over the plate
    micro = api.NewtonOpts(eps_rel=1e-10, eps_abs=1e-12, max_iter=25)
    eng = api.RomEngines(rom, torch.from_numpy(geom).cuda())
    rg = api.run_twoscale(cfg, eng, micro)
    eo = oracle.RomEngines(o, model["ids"], model["weights"], model["mode_grads"], geom, eps_rel=1e-10,
                           eps_abs=1e-12, max_iter=25)
    ro, st = orc.run_twoscale(nx=2, ny=1, steps=6, peak=0.02, eps_rel=1e-9, eps_abs=1e-12, engines=eo)
    assert st == 0
    rel = np.abs(rg["compliance"] - ro["compliance"]).max() / np.abs(ro["compliance"]).max()
    # u_final is the small residual displacement after unloading: measure its
    # error against the displacement scale of the loaded plate (compliance
    # = f . u at the peak)
    u_scale = np.sqrt(np.abs(ro["compliance"]).max())
    du = np.linalg.norm(rg["u_final"] - ro["u_final"]) / u_scale
    print(f"ROM FE2: compliance rel {rel:.2e}, u_final rel {du:.2e}, iters {rg['iters']} vs {ro['iters']}, "
          f"residual displacement {ro['residual_norm']:.3e} (scale {u_scale:.3e})")
    assert rel <= 1e-8 and du <= 1e-8
    assert np.array_equal(rg["iters"], ro["iters"])
