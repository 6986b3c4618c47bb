"""FE2 Example-2 sizes: run_twoscale with the current macro solver; prints
wall, iterations and the compliance history head (A/B of the macro LU)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2307_16894_b200 import api, synth
ctx = api.Context()
mats = [api.matrix_params(), api.inclusion_params()]
rve = api.Rve(128, mats, ctx=ctx)
model = synth.rom_model(rve.export(), rve.n_red, N=50, Q=595, seed=2060)
rom = api.Rom(rve, model["ids"], model["weights"], model["mode_grads"])
macro_newton = api.NewtonOpts(eps_rel=1e-8, eps_abs=1e-12, max_iter=25)
micro = api.NewtonOpts(eps_rel=1e-10, eps_abs=1e-12, max_iter=25)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
peak = float(sys.argv[2]) if len(sys.argv) > 2 else 0.07
cfg = api.MacroConfig(nx=20, ny=10, steps=steps, peak_traction=peak, newton=macro_newton)
x = cfg.qp_positions()
geom = np.stack([0.2 + 0.1 * (1 - x[:, 0] / cfg.width) ** 2, 0.2 + 0.1 * (1 - x[:, 1] / cfg.height)], 1)
eng = api.RomEngines(rom, torch.from_numpy(geom).cuda())
t0 = time.perf_counter()
try:
    r = api.run_twoscale(cfg, eng, micro)
    print("wall", round(time.perf_counter() - t0, 3), "iters", r["iters"].tolist(), "comp", r["compliance"][:6].tolist(),
          "resid", r["residual_norm"])
except Exception as e:
    print("failed after", round(time.perf_counter() - t0, 3), e)
