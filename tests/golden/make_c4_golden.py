#!/usr/bin/env python
"""Config 4 golden ECM selection at its full BASELINE size, CPU only.

Everything here is the oracle: the seeded numpy snapshots (synth.c4_snapshots:
33,282 dofs x 4,000 fields), the POD of oracle/pod_ecm.py (numpy Gram +
dsyevd, podkit.cpp:43-127), the weighted stress snapshots of the CPU oracle
(glibc libm, material.cpp / ecm.cpp:10-18), the mode gradients and the greedy
ecm_select + restore_feasible (ecm.cpp:132-204, 56-90; direct J^T r scores,
from-scratch column-pivoted QR refits).  400 points over 65,536 candidates,
eps 1e-6 with the count stop.  The selection (ids, weights, residual,
iteration count, smallest relative top-2 score gap) is committed as
tests/golden/c4_ecm_golden.npz; tests/test_gpu_fullsize.py compares the GPU
pipeline (device snapshots, POD, stress snapshots and selection) against it.
Takes about an hour on 8 host cores.

  python tests/golden/make_c4_golden.py
"""
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

import oracle  # noqa: E402
from oracle import pod_ecm  # noqa: E402
from paper_2307_16894_b200 import synth  # noqa: E402
from paper_2307_16894_b200.api import inclusion_params, matrix_params  # noqa: E402


def main():
    t0 = time.time()
    oracle.build()
    mats = [matrix_params(), inclusion_params()]
    o = oracle.Rve(128, mats)
    t = o.export()
    L, N, Q = 4000, 50, 400
    U = synth.c4_snapshots(t, L=L, n_terms=20, kmax=8, seed=2030)
    print(f"snapshots {time.time() - t0:.0f} s", flush=True)
    modes, lam = pod_ecm.pod_diag(U, None, N)
    print(f"pod {time.time() - t0:.0f} s", flush=True)
    W, nf = o.stress_snapshots(U)
    assert nf == 0
    del U
    H = pod_ecm.mode_grads(t, modes)
    print(f"stress snapshots {time.time() - t0:.0f} s", flush=True)
    trace = []
    ids, w, rel, it = pod_ecm.ecm_select(H, W, t["w"], 1e-6, volume_row=True, max_points=Q, stop_at_count=True,
                                         trace=trace)
    gaps = np.array([g for _, _, g in trace])
    print(f"ecm {time.time() - t0:.0f} s: {len(ids)} ids, iters {it}, resid {rel:.6e}, min gap {gaps.min():.3e}")
    np.savez_compressed(HERE / "c4_ecm_golden.npz", ids=ids.astype(np.int32), weights=w, resid_rel=rel,
                        iterations=it, top2_gap=gaps, eigenvalues=lam[:N])


if __name__ == "__main__":
    main()
