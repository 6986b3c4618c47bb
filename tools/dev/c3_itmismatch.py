"""Which of the 256 spread C3 instances differ in Newton iteration count from
the oracle, and how close their residuals sit to the convergence tolerance."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import oracle
from paper_2307_16894_b200 import api, synth
mats = [api.matrix_params(), api.inclusion_params()]
rve = api.Rve(128, mats)
model = synth.rom_model(rve.export(), rve.n_red, N=50, Q=400, seed=2029)
rom = api.Rom(rve, model["ids"], model["weights"], model["mode_grads"])
n, K = 65536, 20
geom_np, sched_np = synth.rom_instances(n, K, 2030, 0.2)
pick = np.unique(np.linspace(0, n - 1, 256).astype(np.int64))
opts = api.NewtonOpts(eps_rel=1e-10, eps_abs=1e-12, max_iter=25, max_bisect=5)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
g = rom.solve(T(geom_np[pick]), T(sched_np[pick]), opts)
o = oracle.Rve(128, mats)
ro = o.rom_solve(model["ids"], model["weights"], model["mode_grads"], geom_np[pick], sched_np[pick],
                 eps_rel=1e-10, eps_abs=1e-12, max_iter=25, max_bisect=5, nthreads=oracle.max_threads())
gi, gr = g["iters"].cpu().numpy(), g["resid"].cpu().numpy()
bad = np.argwhere(gi != ro["iters"])
print("mismatches", len(bad))
for s, k in bad[:20]:
    print(f"inst {pick[s]} incr {k}: gpu iters {gi[s, k]} resid {gr[s, k]:.6e} | oracle iters {ro['iters'][s, k]} "
          f"resid {ro['resid'][s, k]:.6e}; rows {gi[s].tolist()} vs {ro['iters'][s].tolist()}")
