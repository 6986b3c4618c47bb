"""End to end on the device: the offline stage of the paper (run_offline,
pipeline.cpp:157-253) — full-order training solves -> displacement and stress
snapshots -> POD of both -> ECM on the factored integrand -> build_rom — and
then the online ROM reproduces a training trajectory of the full-order model.
Every step runs through this repository's kernels; the tolerance is a model
error (reduced basis + cubature), not a parity bound."""
import numpy as np
import pytest

from paper_2307_16894_b200 import synth

pytestmark = pytest.mark.gpu


def test_offline_online_pipeline():
    import torch
    from paper_2307_16894_b200 import api
    mats = [api.matrix_params(), api.inclusion_params()]
    g = api.Rve(16, mats)
    geom_np, sched_np = synth.rom_instances(6, 4, 31, 0.1)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    geom, sched = T(geom_np), T(sched_np)
    opts = api.NewtonOpts(eps_rel=1e-10, eps_abs=1e-12)
    fe = api.FullOrder(g)
    snap = fe.collect_snapshots(geom, sched, opts)               # collect_snapshots
    disp_t = snap["disp"].T.contiguous()                         # [S K, 2 n_nodes]
    stress_t = snap["stress"].T.contiguous()                     # [S K, 4 n_qp]
    modes_t, ev = api.pod(disp_t, 20)                            # displacement POD (unit metric)
    w_q = torch.as_tensor(g.export()["w"], device="cuda").repeat_interleave(4).contiguous()
    smodes_t, sev = api.pod(stress_t, 20, gram_diag=w_q)         # stress POD (quadrature metric)
    H = api.ecm_mode_grads(g, modes_t.contiguous())              # [n_qp][N][4]
    W = smodes_t.reshape(smodes_t.shape[0], g.n_qp, 4).contiguous()
    ids, wts, rel, it = api.ecm_select(g, H, W, api.EcmOpts(eps=1e-6, max_points=200, stop_at_count=True))
    assert np.all(np.diff(ids) > 0) and np.all(wts > 0)
    mg = H[torch.as_tensor(ids, device="cuda", dtype=torch.int64)].cpu().numpy()  # build_rom (rom.cpp:80-109)
    rom = api.Rom(g, ids, wts, mg)
    r_rom = rom.solve(geom, sched, opts)
    r_fe = fe.solve(geom, sched, opts)
    err = (torch.linalg.norm(r_rom["pbar"] - r_fe["pbar"], dim=-1) /
           torch.linalg.norm(r_fe["pbar"], dim=-1)).max().item()
    print(f"pipeline: N={modes_t.shape[0]} stress modes={smodes_t.shape[0]} ECM points={len(ids)} "
          f"(resid {rel:.2e}); ROM vs FE on the training set: max rel {err:.2e}")
    assert int(r_rom["status"].abs().sum()) == 0
    assert err <= 2e-2
