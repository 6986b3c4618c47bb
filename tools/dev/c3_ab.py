"""A/B helper: one C3 solve (N=50, Q=400) at n instances; saves pbar / iters /
status to an npz so two builds or env settings can be compared bit for bit,
and prints the per-kernel times of a second (timed) solve."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2307_16894_b200 import api, synth  # noqa: E402

n = int(sys.argv[1])
outp = sys.argv[2]
dev = torch.device("cuda:0")
ctx = api.Context()
mats = [api.matrix_params(), api.inclusion_params()]
rve = api.Rve(128, mats, ctx=ctx)
t = rve.export()
model = synth.rom_model(t, rve.n_red, N=50, Q=400, seed=2029)
rom = api.Rom(rve, model["ids"], model["weights"], model["mode_grads"])
geom_np, sched_np = synth.rom_instances(n, 20, 2030, 0.2)
geom = torch.from_numpy(geom_np).to(dev)
sched = torch.from_numpy(sched_np).to(dev)
opts = api.NewtonOpts(eps_rel=1e-10, eps_abs=1e-12, max_iter=25, max_bisect=5)
r = rom.solve(geom, sched, opts)
torch.cuda.synchronize()
ctx.check()
ctx.timings()
ctx.set_timing(True)
t0 = time.perf_counter()
r = rom.solve(geom, sched, opts, out=r)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
tk = ctx.timings()
np.savez(outp, pbar=r["pbar"].cpu().numpy(), iters=r["iters"].cpu().numpy(), status=r["status"].cpu().numpy())
print(json.dumps({"n": n, "wall_s": round(wall, 4), "kernels_ms": {k: round(v[0], 3) for k, v in tk.items()}}))
