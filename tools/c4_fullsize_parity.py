#!/usr/bin/env python
"""Config 4 at its full BASELINE size: GPU ECM selection vs the CPU oracle.

POD of the 33,282 x 4,000 seeded snapshot matrix (N = 50 modes) and the
stress snapshots / mode gradients run on the GPU.  Both selectors then get
the SAME factored integrand (H, W), so the check isolates ecm_select +
restore_feasible (ecm.cpp:132-204, 56-90): the GPU's Gram-updated scoring and
incremental CGS2 refit against the oracle's direct J^T r scores and
from-scratch column-pivoted QR (oracle/pod_ecm.py, LAPACK gelsy), 400 points
over 65,536 candidates.  The oracle is the checker; it runs on the host cores
of the GPU box (several minutes).

usage: python tools/c4_fullsize_parity.py [out.json]
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import oracle  # noqa: F401  (checker)
    from oracle import pod_ecm
    from paper_2307_16894_b200 import api, synth
    dev = torch.device("cuda:0")
    mats = [api.matrix_params(), api.inclusion_params()]
    rve = api.Rve(128, mats)
    t = rve.export()
    L, N, Q = 4000, 50, 400
    U = synth.c4_snapshots(t, L=L, n_terms=20, kmax=8, seed=2030, xp=torch, device=dev)
    modes, ev = api.pod(U, N)
    W, _ = api.ecm_stress_snapshots(rve, U)
    H = api.ecm_mode_grads(rve, modes)
    opts = api.EcmOpts(eps=1e-6, volume_row=True, max_points=Q, stop_at_count=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ids_g, w_g, rel_g, it_g = api.ecm_select(rve, H, W, opts)
    t_gpu = time.perf_counter() - t0
    Hn, Wn = H.cpu().numpy(), W.cpu().numpy()
    del W, U
    torch.cuda.empty_cache()
    trace = []
    t0 = time.perf_counter()
    ids_o, w_o, rel_o, it_o = pod_ecm.ecm_select(Hn, Wn, t["w"], 1e-6, volume_row=True, max_points=Q,
                                                  stop_at_count=True, trace=trace)
    t_cpu = time.perf_counter() - t0
    same = bool(np.array_equal(ids_g, ids_o))
    mism = int(np.sum(ids_g != ids_o)) if len(ids_g) == len(ids_o) else None
    gaps = np.array([g for _, _, g in trace])
    out = {
        "config": "C4 full size: 33,282 dofs x 4,000 snapshots, N = 50, 65,536 candidates, 400 points",
        "ids_bit_exact": same, "id_mismatches": mism,
        "iterations": {"gpu": it_g, "oracle": it_o},
        "weights_max_rel_diff": float(np.abs(w_g - w_o).max() / np.abs(w_o).max()) if same else None,
        "residual_rel": {"gpu": rel_g, "oracle": rel_o},
        "smallest_top2_score_gap_rel": float(gaps.min()) if gaps.size else None,
        "seconds": {"gpu_select": round(t_gpu, 3), "oracle_select": round(t_cpu, 1)},
        "oracle_threads": os.cpu_count(),
    }
    print(json.dumps(out, indent=1))
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
