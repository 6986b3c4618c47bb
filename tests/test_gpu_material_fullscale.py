"""K1 parity over the full config-1 population (2^22 points, the bench's own
inputs), against the faithful oracle (oracle/material.cpp: material.cpp
restated, glibc exp/log like the reference) and — when it was built here
from the reference's own source — oracle/_ref (reference material.cpp
compiled unchanged): the CUDA kernel must reproduce P, the FD tangent A,
the updated history and the status BIT FOR BIT.

Every device operation is correctly rounded and in the reference's order
(--fmad=false; sqrt and '/' are IEEE), and exp/log are csrc/gmath.h, the
device restatement of the host glibc functions (tests/test_gmath.py,
tests/test_gpu_gmath.py), so bitwise equality is the criterion: it implies
the BASELINE tolerances (1e-10 stresses / history, 1e-9 tangents) with no
libm floor left."""
import numpy as np
import pytest

from paper_2307_16894_b200 import synth

pytestmark = pytest.mark.gpu


def test_config1_full_population(orc):
    import torch
    from paper_2307_16894_b200 import api
    F, st = synth.config1_points(1 << 22, 2027)
    mats = [api.matrix_params()]
    g = api.material_batch(torch.from_numpy(F).cuda(), torch.from_numpy(st).cuda(), mats)
    G = {k: g[k].cpu().numpy() for k in ("P", "A", "st", "status")}
    del g
    o = orc.material_batch(F, st, mats)
    assert np.array_equal(G["status"], o["status"])
    for k in ("P", "A", "st"):
        ndiff = int((G[k].view(np.int64) != o[k].view(np.int64)).any(0).sum())
        print(f"{k}: {ndiff} of {F.shape[1]} points differ from the glibc oracle")
        assert ndiff == 0, k
    if orc.ref_available():
        r = orc.ref_material_batch(F, st, mats[0])
        for k in ("P", "A", "st"):
            assert np.array_equal(G[k].view(np.int64), r[k].view(np.int64)), ("oracle/_ref", k)
