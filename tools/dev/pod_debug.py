import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch
from paper_2307_16894_b200 import api, synth
mats = [api.matrix_params(), api.inclusion_params()]
rve = api.Rve(128, mats)
U = synth.c4_snapshots(rve.export(), L=4000, n_terms=20, kmax=8, seed=2030, xp=torch, device=torch.device("cuda:0"))
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    modes, ev = api.pod(U, 50)
    torch.cuda.synchronize(); print("pod wall", time.perf_counter() - t0, flush=True)
lam = torch.linalg.eigvalsh(U @ U.T).flip(0)[:50]
print("eig rel err", float(((ev[:50] - lam).abs() / lam[0]).max()))
ctx = api.Context.default()
ctx.timings(); ctx.set_timing(True)
api.pod(U, 50)
ctx.set_timing(False)
for k, v in ctx.timings().items(): print(k, round(v[0], 3), v[1])
