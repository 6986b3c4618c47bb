"""Dev probe: repeat the exact-limit FE / ROM solves and report run-to-run deviations."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
from oracle.fe import exact_limit_model
from paper_2307_16894_b200 import api

mats = [api.matrix_params(), api.inclusion_params()]
o = oracle.Rve(4, mats)
t = o.export()
ids, wts, mg = exact_limit_model(o, t)
g = api.Rve(4, mats)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
geom = np.array([[0.3, 0.2], [0.22, 0.31]])
H = np.array([0.06, 0.02, -0.03, -0.04])
sched = np.array([[[1, 0, 0, 1] + (k / 6) * H for k in range(1, 7)]] * 2)
opts = api.NewtonOpts(eps_rel=1e-12, eps_abs=1e-14)
ref_fe = ref_rom = ref_it = None
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 40):
    fe = api.FullOrder(g).solve(T(geom), T(sched), opts)
    rom = api.Rom(g, ids, wts, mg).solve(T(geom), T(sched), opts)
    torch.cuda.synchronize()
    if ref_fe is None:
        ref_fe, ref_rom = fe["pbar"].clone(), rom["pbar"].clone()
        ref_it = fe["iters"].clone()
        print("first fe iters", ref_it.tolist(), "resid", fe["resid"].tolist())
    dfe = ((fe["pbar"] - ref_fe).norm(dim=-1) / ref_fe.norm(dim=-1)).max().item()
    drom = ((rom["pbar"] - ref_rom).norm(dim=-1) / ref_rom.norm(dim=-1)).max().item()
    x = ((fe["pbar"] - rom["pbar"]).norm(dim=-1) / fe["pbar"].norm(dim=-1)).max().item()
    if dfe > 1e-10 or drom > 1e-10 or x > 1e-8 or it % 10 == 0:
        print(it, f"fe-vs-first {dfe:.2e} rom-vs-first {drom:.2e} fe-vs-rom {x:.2e}",
              "fe status", fe["status"].tolist(), "rom status", rom["status"].tolist(), flush=True)
        if dfe > 1e-10:
            print("   fe iters", fe["iters"].tolist(), "resid", fe["resid"].tolist(), flush=True)
