"""The portable exp/log used by the material kernels (csrc/pdmath.h), built
for the host: accuracy against an extended-precision reference (x87 long
double) over the material's ranges and beyond, and agreement with glibc."""
import numpy as np
import pytest


def _ulp_err(v, ref):
    ulp = np.spacing(np.abs(ref.astype(np.float64)))
    return np.abs((v.astype(np.longdouble) - ref) / ulp.astype(np.longdouble)).astype(np.float64)


@pytest.mark.parametrize("name", ["exp", "log"])
def test_pdm_accuracy(orc, name):
    rng = np.random.default_rng(11)
    if name == "log":
        xs = np.concatenate([rng.uniform(0.3, 3.0, 300000), 1 + rng.uniform(-1e-2, 1e-2, 100000),
                             1 + rng.uniform(-1e-9, 1e-9, 20000), np.exp(rng.uniform(-700, 700, 50000))])
        ref = np.log(xs.astype(np.longdouble))
    else:
        xs = np.concatenate([rng.uniform(-1, 1, 300000), rng.uniform(-1e-7, 1e-7, 20000),
                             rng.uniform(-690, 690, 50000)])
        ref = np.exp(xs.astype(np.longdouble))
    p = orc.libm("pdm_" + name, xs)
    g = orc.libm(name, xs)
    ep = _ulp_err(p, ref)
    mism_cr = np.mean(p != ref.astype(np.float64))
    mism_glibc = np.mean(p != g)
    print(f"{name}: max {ep.max():.4f} ulp, != correctly rounded {mism_cr:.5f}, != glibc {mism_glibc:.5f}")
    assert ep.max() <= 0.51
    assert mism_cr <= 0.002 and mism_glibc <= 0.003


def test_pdm_special_values(orc):
    xs = np.array([0.0, -1.0, np.inf, np.nan, 5e-324, 1.0, 2.0, 0.5])
    p = orc.libm("pdm_log", xs)
    g = orc.libm("log", xs)
    assert np.array_equal(np.isnan(p), np.isnan(g)) and np.array_equal(p[~np.isnan(p)], g[~np.isnan(g)])
    xe = np.array([0.0, -800.0, 800.0, np.inf, -np.inf, np.nan, 1.0])
    p = orc.libm("pdm_exp", xe)
    g = orc.libm("exp", xe)
    assert np.array_equal(np.isnan(p), np.isnan(g)) and np.array_equal(p[~np.isnan(p)], g[~np.isnan(g)])
    assert orc.libm("pdm_exp", np.array([0.0]))[0] == 1.0
