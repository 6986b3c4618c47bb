"""FE2 wall time vs load steps (timing off): fixed set-up cost vs per-step cost."""
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
def run(steps, timing=False):
    cfg = api.MacroConfig(nx=20, ny=10, steps=steps, peak_traction=0.07, newton=macro_newton)
    x = cfg.qp_positions()
    geom = np.stack([0.2 + 0.1 * (1 - x[:, 0] / cfg.width) ** 2, 0.2 + 0.1 * (1 - x[:, 1] / cfg.height)], 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng = api.RomEngines(rom, torch.from_numpy(geom).cuda())
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ctx.set_timing(timing)
    r = api.run_twoscale(cfg, eng, micro)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    ctx.set_timing(False)
    ctx.timings()
    return t1 - t0, t2 - t1, int(r["iters"].sum())
run(2)
for st in (2, 10, 50):
    print(st, [round(v, 4) for v in run(st)])
print("timing on", [round(v, 4) for v in run(50, True)])
