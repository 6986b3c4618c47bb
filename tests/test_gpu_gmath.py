"""The device build of csrc/gmath.h (the material's exp/log) equals the host
glibc exp/log bit for bit: scalar forms and the pair forms the material
kernels call (both arguments of a pair drawn from the same population, so
pairs mix the near-1 / table log paths and the tiny / main exp paths), over
the material's ranges, the rare paths and raw bit patterns."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _probe(which, a, b):
    import ctypes as C
    import torch
    from paper_2307_16894_b200 import api
    ctx = api.Context.default()
    ta = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    tb = torch.from_numpy(np.ascontiguousarray(b)).cuda()
    out = torch.empty_like(ta)
    rc = ctx.lib.podecm_probe_math(ctx.h, ctx.stream(), which, a.size, C.c_void_p(ta.data_ptr()),
                                   C.c_void_p(tb.data_ptr()), C.c_void_p(out.data_ptr()))
    assert rc == 0
    return out.cpu().numpy()


def _same(g, d):
    return np.array_equal(np.isnan(g), np.isnan(d)) and np.array_equal(
        g[~np.isnan(g)].view(np.int64), d[~np.isnan(d)].view(np.int64))


def _args(which, n, seed):
    rng = np.random.default_rng(seed)
    k = n // 8
    raw = rng.integers(0, 2 ** 63, k, dtype=np.int64).view(np.float64) * rng.choice([-1.0, 1.0], k)
    if which == "exp":
        parts = [rng.uniform(-2, 2, 3 * k), rng.uniform(-0.02, 0.02, k), rng.uniform(-745.2, 709.9, k),
                 np.exp(rng.uniform(-690, -11, k)) * rng.choice([-1.0, 1.0], k), raw,
                 np.zeros(16), np.full(16, 512.0), np.array([np.inf, -np.inf, np.nan, 1e-300])]
    else:
        parts = [rng.uniform(0.5, 2.0, 3 * k), rng.uniform(0.9375, 1.0648, 2 * k),
                 np.exp(rng.uniform(-690, 690, k)), raw, np.array([0.0, -1.0, np.inf, np.nan, 5e-324, 1.0])]
    x = np.concatenate(parts)
    return x[rng.permutation(x.size)]


@pytest.mark.parametrize("which", ["exp", "log"])
def test_gm_device_equals_glibc(orc, which):
    n = 1 << 25
    x = _args(which, n, 31 if which == "exp" else 37)
    y = np.roll(x, 1)
    g = orc.libm(which, x)
    base = 6 if which == "exp" else 7
    pair = 8 if which == "exp" else 10
    assert _same(g, _probe(base, x, y)), "scalar"
    assert _same(g, _probe(pair, x, y)), "pair, first"
    assert _same(g, _probe(pair + 1, x, y)), "pair, second"
    # the round-1 portable variant is NOT glibc (documents why it was replaced)
    p = _probe(12 if which == "exp" else 13, x, y)
    fin = np.isfinite(g)
    print(f"{which}: pdm differs from glibc in {np.mean(p[fin] != g[fin]):.5f} of finite results")
