"""Pins the CPU oracle's material restatement to the reference's own
known-answer and property tests (test_material.cpp:144-239; the reference
ships no golden vectors and cannot be built here)."""
import numpy as np
import pytest

from paper_2307_16894_b200.api import PlasticityParams


def matrix_params():  # test_material.cpp:11-18
    return PlasticityParams(10.0, 0.3, 0.2, 5.0)


def elastic(p):
    return PlasticityParams(p.E, p.nu, 1e12, p.H)


def virgin(n=1):
    st = np.zeros((6, n))
    st[0] = st[3] = st[4] = 1.0
    return st


def lam_mu(p):
    return p.E * p.nu / ((1 + p.nu) * (1 - 2 * p.nu)), p.E / (2 * (1 + p.nu))


def mat(F):
    return np.array([[F[0], F[2]], [F[1], F[3]]])


def flat(M):
    return np.array([M[0, 0], M[1, 0], M[0, 1], M[1, 1]])


def test_stress_free_at_identity(orc):  # :144-149
    r = orc.material_batch(flat(np.eye(2))[:, None], virgin(), [matrix_params()])
    assert np.linalg.norm(r["P"][:, 0]) <= 1e-14


def test_equal_biaxial_closed_form(orc):  # :151-163
    p = elastic(matrix_params())
    c = 1.05
    r = orc.material_batch(flat(c * np.eye(2))[:, None], virgin(), [p])
    la, mu = lam_mu(p)
    sig = la * 2 * np.log(c) + 2 * mu * np.log(c)
    P = r["P"][:, 0]
    assert abs(P[0] - sig / c) <= 1e-12 and abs(P[3] - sig / c) <= 1e-12
    assert abs(P[1]) <= 1e-13 and abs(P[2]) <= 1e-13


def test_rotation_rotates_stress(orc):  # :182-193 objectivity
    p = elastic(matrix_params())
    f = np.array([[1.08, 0.03], [-0.02, 0.95]])
    th = 0.4
    R = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
    r = orc.material_batch(np.stack([flat(f), flat(R @ f)], 1), virgin(2), [p])
    P0, P1 = mat(r["P"][:, 0]), mat(r["P"][:, 1])
    assert np.linalg.norm(P1 - R @ P0) <= 1e-12


def test_plastic_flow_isochoric(orc):  # :195-208
    p = matrix_params()
    rng = np.random.default_rng(19)
    st = virgin()
    for _ in range(50):
        f = np.array([1 + rng.uniform(-.08, .08), rng.uniform(-.08, .08), rng.uniform(-.08, .08),
                      1 + rng.uniform(-.08, .08)])
        r = orc.material_batch(f[:, None], st, [p], tangent=False)
        st = r["st"]
        Fp = mat(st[:4, 0])
        assert abs(np.linalg.det(Fp) * st[4, 0] - 1.0) <= 1e-12
        assert st[5, 0] >= 0
    assert st[5, 0] > 0


def test_kkt_after_return(orc):  # :210-219
    p = matrix_params()
    f = flat(np.array([[1.08, 0.05], [0.0, 0.97]]))
    r = orc.material_batch(f[:, None], virgin(), [p])
    assert r["dgamma"][0] > 0
    la, mu = lam_mu(p)
    xi1 = r["st"][5, 0]
    f_new = r["mises"][0] - (p.sigma_y0 + p.H * xi1)
    assert abs(f_new) <= 1e-10 * p.sigma_y0
    assert abs(r["dgamma"][0] - r["f_trial"][0] / (3 * mu + p.H)) <= 1e-14


def test_tangent_matches_directional_differences(orc):  # :221-239
    p = matrix_params()
    s = orc.material_batch(flat(np.array([[1.06, 0.02], [0.01, 0.96]]))[:, None], virgin(), [p])["st"]
    f = flat(np.array([[1.09, 0.03], [0.02, 0.94]]))
    A = orc.material_batch(f[:, None], s, [p])["A"][:, 0].reshape(4, 4, order="F")
    rng = np.random.default_rng(23)
    for _ in range(10):
        d = rng.uniform(-1, 1, 4)
        d /= np.linalg.norm(d)
        h = 1e-6
        Fs = np.stack([f + h * d, f - h * d], 1)
        r = orc.material_batch(Fs, np.repeat(s, 2, axis=1), [p], tangent=False)
        fd = (r["P"][:, 0] - r["P"][:, 1]) / (2 * h)
        assert np.linalg.norm(A @ d - fd) <= 1e-5 * np.linalg.norm(fd) + 1e-8


def test_xi_never_hardens_yield_quirk(orc):
    """material.cpp:137-138 runs the inner return from SmallState{}: the
    accumulated xi does not raise the yield stress (replicated, not fixed)."""
    p = matrix_params()
    f = flat(np.array([[1.08, 0.05], [0.0, 0.97]]))
    st = virgin(2)
    st[5, 1] = 10.0  # huge accumulated plastic strain
    r = orc.material_batch(np.stack([f, f], 1), st, [p])
    assert r["dgamma"][0] == r["dgamma"][1] > 0
    assert np.array_equal(r["P"][:, 0], r["P"][:, 1])
    assert r["st"][5, 1] == 10.0 + r["dgamma"][1]


def test_inclusion_never_yields(orc):
    p = PlasticityParams(100.0, 0.3, 1e12, 5.0)
    rng = np.random.default_rng(17)
    F = np.eye(2).reshape(4, 1, order="F") + rng.uniform(-0.2, 0.2, (4, 100)) * np.array([1, 1, 1, 1])[:, None]
    F = F[:, (F[0] * F[3] - F[1] * F[2]) > 0.3]
    r = orc.material_batch(F, virgin(F.shape[1]), [p])
    assert np.all(r["dgamma"] == 0)
    assert np.all(r["st"][5] == 0)


def test_nonpositive_stretch_raises(orc):
    """material.cpp:128-130: a singular stretch (lambda_2 of C <= 0) raises
    SolveError; a reflection (det F < 0, C regular) does not."""
    F = np.array([[1.0, 0.0, 0.0, 0.0], [0.0, 0.0, 0.0, 0.0], [1.0, 0.0, 0.0, -0.5]]).T
    r = orc.material_batch(F, virgin(3), [matrix_params()])
    assert list(r["status"]) == [3, 3, 0]


def test_thread_count_does_not_change_results(orc):
    from paper_2307_16894_b200 import synth
    F, st = synth.config1_points(4096, 5)
    p = PlasticityParams(1.0, 0.3, 0.01, 0.1)
    a = orc.material_batch(F, st, [p], nthreads=1)
    b = orc.material_batch(F, st, [p], nthreads=4)
    for k in ("P", "A", "st"):
        assert np.array_equal(a[k], b[k])
