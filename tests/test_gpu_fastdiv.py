"""The material kernels replace IEEE divisions by a shared correctly rounded
reciprocal plus one Markstein correction (csrc/material.cuh div_rcp) and
1.0/d by __drcp_rn.  Both must be bit-identical to '/' over the value ranges
the material sees (and far beyond): checked here on the device."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _probe(which, a, b):
    import ctypes as C
    import torch
    from paper_2307_16894_b200 import api
    ctx = api.Context.default()
    ta = torch.from_numpy(a).cuda()
    tb = torch.from_numpy(b).cuda()
    out = torch.empty_like(ta)
    rc = ctx.lib.podecm_probe_math(ctx.h, ctx.stream(), which, a.size, C.c_void_p(ta.data_ptr()),
                                   C.c_void_p(tb.data_ptr()), C.c_void_p(out.data_ptr()))
    assert rc == 0
    return out.cpu().numpy()


def _random(n, lo, hi, seed):
    rng = np.random.default_rng(seed)
    m = rng.uniform(1.0, 2.0, n) * rng.choice([-1.0, 1.0], n)
    e = rng.integers(lo, hi, n)
    return np.ldexp(m, e)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_div_rcp_bit_identical(seed):
    n = 1 << 24
    a = _random(n, -200, 200, seed)
    b = _random(n, -200, 200, seed + 10)
    # adversarial mantissas: all-ones / near-power-of-two divisors and constants
    b[: n // 8] = np.ldexp(1.0 - np.ldexp(1.0, -np.random.default_rng(seed).integers(1, 53, n // 8)), 1)
    b[n // 8: n // 4] = 3.0
    q_ieee = _probe(0, a, b)
    q_rcp = _probe(1, a, b)
    assert np.array_equal(q_ieee.view(np.int64), q_rcp.view(np.int64))


def test_drcp_equals_one_over():
    n = 1 << 22
    b = _random(n, -300, 300, 7)
    assert np.array_equal(_probe(2, b, b).view(np.int64), _probe(3, b, b).view(np.int64))
