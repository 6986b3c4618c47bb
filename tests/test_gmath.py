"""csrc/gmath.h (the device's restatement of the host glibc exp/log, the
libm the reference's material.cpp:135-150 calls), built for the host: equal
to glibc bit for bit.

The sweeps run 2^30 arguments per function (OpenMP inside the oracle
library), spread over the material's ranges (exp of plastic strains and of
2(eps_tr - eps_p); log of principal stretches near 1 and of 1/Fp_zz^2),
both log paths (|x - 1| < 2^-4 and the table path), the exp main range up to
|x| = 745, the rare paths (|x| < 2^-54, subnormal and huge results,
subnormal log arguments) and raw random bit patterns (every exponent, inf,
nan, negative)."""
import numpy as np
import pytest

EXP_SWEEPS = [  # (mode, lo, hi, n)   mode 0 uniform, 1 log-uniform |x|, 2 raw bits
    (0, -2.0, 2.0, 1 << 29),
    (0, -0.02, 0.02, 1 << 27),
    (0, -745.2, 709.9, 1 << 27),
    (1, 1e-300, 1e-5, 1 << 27),
    (2, 0.0, 0.0, 1 << 27),
]
LOG_SWEEPS = [
    (0, 0.5, 2.0, 1 << 29),
    (0, 0.9375, 1.0648, 1 << 28),
    (1, 1e-300, 1e300, 1 << 27),
    (1, 4.9e-324, 2.2e-308, 1 << 24),
    (2, 0.0, 0.0, 1 << 27),
]


def _total(sweeps):
    return sum(s[3] for s in sweeps)


@pytest.mark.parametrize("which,sweeps", [("exp", EXP_SWEEPS), ("log", LOG_SWEEPS)])
def test_gm_equals_glibc_bitwise(orc, which, sweeps):
    assert _total(sweeps) >= 1 << 30  # >= 2^30 arguments per function
    for k, (mode, lo, hi, n) in enumerate(sweeps):
        for seed in (101 + k, 202 + k):  # two independent streams of n / 2
            m, bad = orc.libm_sweep(which, n // 2, seed, mode, lo, hi)
            assert m == 0, f"{which}: {m} mismatches in sweep {k} (first at x = {bad!r})"


def test_gm_special_values(orc):
    xs = np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 5e-324, 2.2250738585072014e-308,
                   1.7976931348623157e308, 0.9375, 1.0647, 1 - 2 ** -53, 1 + 2 ** -52])
    for f in ("log", "exp"):
        g = orc.libm(f, xs)
        m = orc.libm("gm_" + f, xs)
        assert np.array_equal(np.isnan(g), np.isnan(m)), f
        assert np.array_equal(g[~np.isnan(g)].view(np.int64), m[~np.isnan(m)].view(np.int64)), f
    xe = np.array([709.78, 709.79, -708.4, -708.5, -745.1, -745.2, -1000.0, 1000.0, 512.0, -512.0,
                   1e-17, -1e-17, 2 ** -54, -(2 ** -54), 2 ** -55])
    g = orc.libm("exp", xe)
    m = orc.libm("gm_exp", xe)
    assert np.array_equal(g.view(np.int64), m.view(np.int64))


def test_fast_paths_on_their_domains(orc):
    """The branch-free forms the material kernels call: exp_fast (= exp_core)
    on |x| < 512 including the tiny range glibc special-cases (|x| < 2^-54,
    zeros, subnormals), log_core on every normal positive x (both paths and
    x == 1)."""
    rng = np.random.default_rng(5)
    tiny = np.concatenate([np.ldexp(rng.uniform(1, 2, 200000), rng.integers(-1074, -54, 200000)),
                           [0.0, -0.0, 5e-324, -5e-324, 2.0 ** -55, -(2.0 ** -55), np.nextafter(2.0 ** -54, 0)]])
    tiny = np.concatenate([tiny, -tiny])
    xe = np.concatenate([tiny, rng.uniform(-511.9, 511.9, 400000), rng.uniform(-1e-3, 1e-3, 200000)])
    g, m = orc.libm("exp", xe), orc.libm("gm_exp_fast", xe)
    assert np.array_equal(g.view(np.int64), m.view(np.int64))
    xl = np.concatenate([np.ldexp(rng.uniform(1, 2, 400000), rng.integers(-1021, 1023, 400000)),
                         rng.uniform(0.9, 1.1, 400000), [1.0, np.nextafter(1.0, 0), np.nextafter(1.0, 2),
                                                         2.2250738585072014e-308, 1.7976931348623157e308]])
    g, m = orc.libm("log", xl), orc.libm("gm_log_core", xl)
    assert np.array_equal(g.view(np.int64), m.view(np.int64))
