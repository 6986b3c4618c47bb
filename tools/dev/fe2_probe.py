import time, numpy as np, torch
from paper_2307_16894_b200 import api, synth
mats = [api.matrix_params(), api.inclusion_params()]
g = api.Rve(128, mats)
t = g.export()
model = synth.rom_model(t, g.n_red, N=50, Q=595, seed=2060)
rom = api.Rom(g, model["ids"], model["weights"], model["mode_grads"])
for peak, steps in ((0.05, 50), (0.07, 50), (0.1, 50)):
    cfg = api.MacroConfig(nx=20, ny=10, steps=steps, peak_traction=peak, newton=api.NewtonOpts(eps_rel=1e-8, eps_abs=1e-12, max_iter=25))
    x = cfg.qp_positions()
    geom = np.stack([0.2 + 0.1 * (1 - x[:, 0] / 2.0) ** 2, 0.2 + 0.1 * (1 - x[:, 1])], 1)
    eng = api.RomEngines(rom, torch.from_numpy(geom).cuda())
    t0 = time.perf_counter()
    try:
        r = api.run_twoscale(cfg, eng, api.NewtonOpts(eps_rel=1e-10, eps_abs=1e-12, max_iter=25))
        dt = time.perf_counter() - t0
        print(peak, steps, f"{dt:.2f}s", r["iters"], r["residual_norm"], r["micro_evals"], flush=True)
    except Exception as ex:
        print(peak, "failed", ex, flush=True)
