"""Dev probe: ROM solve status / pbar over a few sizes (A/B kernel variants via env)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2307_16894_b200 import api, synth

dev = torch.device("cuda:0")
T = lambda a: torch.from_numpy(a).to(dev)
mats = [api.matrix_params(), api.inclusion_params()]
for cells, N, Q, n in [(16, 8, 24, 2), (32, 20, 100, 64), (128, 50, 400, 256), (128, 50, 400, 4096)]:
    rve = api.Rve(cells, mats)
    t = rve.export()
    model = synth.rom_model(t, rve.n_red, N=N, Q=Q, seed=5)
    rom = api.Rom(rve, model["ids"], model["weights"], model["mode_grads"])
    geom, sched = synth.rom_instances(n, 4, 7, 0.2)
    for abar in (False, True):
        try:
            r = rom.solve(T(geom), T(sched), api.NewtonOpts(eps_rel=1e-10), abar=abar)
            torch.cuda.synchronize()
            st = r["status"].cpu().numpy()
            extra = float(r["abar"].double().abs().sum()) if abar else 0.0
            print(cells, N, Q, n, "abar", abar, "fail", int((st != 0).sum()), "pbar sum",
                  float(r["pbar"].double().sum()), extra, flush=True)
        except Exception as e:
            print(cells, N, Q, n, "abar", abar, "EXC", str(e)[:200], flush=True)
