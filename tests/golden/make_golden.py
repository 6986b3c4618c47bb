#!/usr/bin/env python
"""Regenerate the committed golden fixtures from the CPU oracle.

The reference ships no golden vectors and cannot be built here,
so these fixtures pin the oracle restatement (itself validated against the
reference's closed-form / property tests in tests/test_oracle_*.py) and let
the GPU tests check parity without running the oracle.

  python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

import oracle  # noqa: E402
from oracle import pod_ecm  # noqa: E402
from paper_2307_16894_b200 import synth  # noqa: E402
from paper_2307_16894_b200.api import inclusion_params, matrix_params  # noqa: E402


def main():
    mats = [matrix_params(), inclusion_params()]
    # K1: 256 config-1 points + edge cases
    F, st = synth.config1_points(256, 101)
    F[:, 0] = [1, 0, 0, 1]
    F[:, 1] = [1.05, 0, 0, 1.05]
    F[:, 2] = [1.0, 0, 0, 0.0]  # singular -> SolveError
    r = oracle.material_batch(F, st, mats[:1], nthreads=1)
    np.savez_compressed(HERE / "material_c1_256.npz", F=F, st=st, P=r["P"], A=r["A"], st_out=r["st"],
                        status=r["status"], dgamma=r["dgamma"])
    # K2: 8x8 cell, 2 instances
    o = oracle.Rve(8, mats)
    t = o.export()
    geom, fbar, w, st0 = synth.rve_instances(2, o.n_red, np.repeat(t["regions"], 4), 102, 0.1,
                                             geom_range=(0.15, 0.35))
    a = o.assemble(geom, fbar, w, st0, store_stress=True, nthreads=1)
    np.savez_compressed(HERE / "assemble_8x8.npz", geom=geom, fbar=fbar, w_red=w, st0=st0, f=a["f"], K=a["K"],
                        st1=a["st1"], p_field=a["p_field"], row_ptr=t["row_ptr"], col_idx=t["col_idx"],
                        node_dof=t["node_dof"])
    # K3: 16x16 cell, N=10, Q=40, 3 instances x 5 increments
    o16 = oracle.Rve(16, mats)
    t16 = o16.export()
    model = synth.rom_model(t16, o16.n_red, N=10, Q=40, seed=103)
    g3, s3 = synth.rom_instances(3, 5, 104, 0.2)
    ro = o16.rom_solve(model["ids"], model["weights"], model["mode_grads"], g3, s3, eps_rel=1e-10, nthreads=1)
    np.savez_compressed(HERE / "rom_16x16_N10_Q40.npz", ids=model["ids"], weights=model["weights"],
                        mode_grads=model["mode_grads"], geom=g3, sched=s3, pbar=ro["pbar"], iters=ro["iters"],
                        status=ro["status"])
    # K4: 12x12 cell, 40 snapshots, 5 modes, 20 points
    o12 = oracle.Rve(12, mats)
    t12 = o12.export()
    U = synth.c4_snapshots(t12, L=40, n_terms=5, kmax=3, seed=105)
    modes, lam = pod_ecm.pod_diag(U, None, 5)
    W, _ = o12.stress_snapshots(U, nthreads=1)
    H = pod_ecm.mode_grads(t12, modes)
    ids, wts, rel, it = pod_ecm.ecm_select(H, W, t12["w"], 1e-10, max_points=20, stop_at_count=True)
    np.savez_compressed(HERE / "pod_ecm_12x12.npz", U=U, modes=modes, evals=lam, H=H, W=W, ids=ids,
                        weights=wts, resid_rel=rel, iterations=it)
    for p in sorted(HERE.glob("*.npz")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
