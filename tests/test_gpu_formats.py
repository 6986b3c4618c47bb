"""Interchange formats on a real model (test_rom.cpp:188-216 analogue): a
reduced model written to PODECM1 and read back replays a batched solve
bit-identically; the content tag is the cell's fingerprint, recomputed here
independently from the exported mesh tables and by the reference's own
Mesh::fingerprint (mesh.cpp:158-180, compiled into oracle/_ref)."""
import struct

import numpy as np
import pytest

from paper_2307_16894_b200 import synth

pytestmark = pytest.mark.gpu


def _py_fingerprint(t) -> int:
    h = 14695981039346656037

    def fnv(b):
        nonlocal h
        for c in b:
            h ^= c
            h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF

    fnv(bytes([1]))  # mesh.cpp:160: every non-Tri6 kind hashes as 1
    fnv(struct.pack("<qqq", t["nodes"].shape[0], t["elems"].shape[0], 0))
    fnv(np.asfortranarray(t["nodes"]).tobytes(order="F"))
    fnv(t["elems"].astype(np.int64).tobytes())
    fnv(t["regions"].astype(np.int64).tobytes())
    return h


def test_model_round_trips_through_disk(tmp_path):
    import torch
    from paper_2307_16894_b200 import api
    mats = [api.matrix_params(), api.inclusion_params()]
    g = api.Rve(16, mats)
    t = g.export()
    assert g.fingerprint() == _py_fingerprint(t)
    import oracle
    if oracle.ref_available():  # the reference's own Mesh::fingerprint (oracle/_ref)
        assert g.fingerprint() == oracle.ref_fingerprint(16, t["regions"])
    m = synth.rom_model(t, g.n_red, N=10, Q=60, seed=3)
    n_dof = 2 * g.n_nodes
    modes = np.random.default_rng(4).normal(size=(n_dof, 10))
    f = tmp_path / "model.bin"
    api.rom_model_save(f, {"modes": modes, "ids": m["ids"], "weights": m["weights"], "mode_grads": m["mode_grads"],
                           "mesh_tag": g.fingerprint(), "kind": 0, "n_stress_modes": 0, "ecm_eps": 1e-6})
    r = api.rom_model_load(f)
    assert r["mesh_tag"] == g.fingerprint()
    geom, sched = synth.rom_instances(4, 3, 5, 0.15)
    T = lambda a: torch.from_numpy(a).cuda()
    a = api.Rom(g, m["ids"], m["weights"], m["mode_grads"]).solve(T(geom), T(sched))
    b = api.Rom(g, r["ids"], r["weights"], r["mode_grads"]).solve(T(geom), T(sched))
    assert torch.equal(a["pbar"], b["pbar"]) and torch.equal(a["a_final"], b["a_final"])
