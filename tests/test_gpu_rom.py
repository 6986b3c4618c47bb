"""K3 parity: batched hyper-reduced online stage (config 3) vs the CPU oracle
(rom.cpp:16-200 restated).  Homogenised stress histories within 1e-8
relative per increment; Newton iteration counts per increment equal; the
bisection state machine is exercised by forcing failures (tight max_iter).
"""
import numpy as np
import pytest

from paper_2307_16894_b200 import synth

pytestmark = pytest.mark.gpu


def _mats():
    from paper_2307_16894_b200.api import inclusion_params, matrix_params
    return [matrix_params(), inclusion_params()]


@pytest.fixture(scope="module")
def setup(orc):
    from paper_2307_16894_b200 import api
    g = api.Rve(128, _mats())
    o = orc.Rve(128, _mats())
    model = synth.rom_model(g.export(), g.n_red, N=50, Q=400, seed=2029)
    rom = api.Rom(g, model["ids"], model["weights"], model["mode_grads"])
    return g, o, model, rom


def _solve(setup, n, K, seed, hm, opts_kw):
    import torch
    from paper_2307_16894_b200 import api
    g, o, model, rom = setup
    geom, sched = synth.rom_instances(n, K, seed, hm)
    T = lambda a: torch.from_numpy(a).cuda()
    opts = api.NewtonOpts(**opts_kw)
    rg = rom.solve(T(geom), T(sched), opts)
    torch.cuda.synchronize()
    rg = {k: v.cpu().numpy() for k, v in rg.items()}
    ro = o.rom_solve(model["ids"], model["weights"], model["mode_grads"], geom, sched,
                     eps_rel=opts.eps_rel, eps_abs=opts.eps_abs, max_iter=opts.max_iter,
                     max_bisect=opts.max_bisect)
    return rg, ro


def _check(rg, ro, tol=1e-8, iters_exact=True):
    assert np.array_equal(rg["status"], ro["status"]), (rg["status"], ro["status"])
    ok = ro["status"] == 0
    d = np.linalg.norm(rg["pbar"][ok] - ro["pbar"][ok], axis=-1)
    nrm = np.maximum(np.linalg.norm(ro["pbar"][ok], axis=-1), 1e-14)
    rel = d / nrm
    mism = int((rg["iters"][ok] != ro["iters"][ok]).sum())
    print(f"pbar max rel {rel.max():.3e}; iteration-count mismatches {mism}/{rg['iters'][ok].size}; "
          f"mean iters/increment {ro['iters'][ok].mean():.2f}")
    assert rel.max() <= tol
    if iters_exact:
        assert mism == 0


def test_config3_instances(setup):
    rg, ro = _solve(setup, 6, 20, 2030, 0.2, dict(eps_rel=1e-10, eps_abs=1e-12, max_iter=25))
    assert np.all(ro["status"] == 0)
    _check(rg, ro)


def test_bisection_path(setup):
    """One big increment with max_iter = 3 forces failed attempts -> recursive
    bisection (rom.cpp:152-175) to depths 1-3; histories and the summed
    iteration counts must match."""
    rg, ro = _solve(setup, 6, 1, 77, 0.2, dict(eps_rel=1e-10, eps_abs=1e-12, max_iter=3,
                                               max_bisect=5))
    assert ro["iters"].max() > 3  # bisection happened
    _check(rg, ro)


def test_bisection_exhausted_is_solveerror(setup):
    """max_iter = 0 with max_bisect = 1 cannot converge: every instance fails
    with SolveError like the reference's rethrow."""
    rg, ro = _solve(setup, 3, 2, 5, 0.2, dict(eps_rel=1e-10, eps_abs=1e-12, max_iter=0,
                                              max_bisect=1))
    assert np.all(ro["status"] == 3)
    assert np.array_equal(rg["status"], ro["status"])


def test_exact_limit_gpu_equals_full_order(orc):
    """test_rom.cpp:44-125 on the GPU: full periodic basis (N = n_red = 30)
    and full quadrature on a 4x4 cell => the batched ROM reproduces the
    full-order response (oracle FE Newton) to 1e-8."""
    import torch
    from paper_2307_16894_b200 import api
    from oracle.fe import exact_limit_model, fe_newton_pbar
    o = orc.Rve(4, _mats())
    t = o.export()
    ids, wts, mg = exact_limit_model(o, t)
    g = api.Rve(4, _mats())
    rom = api.Rom(g, ids, wts, mg)
    geom = (0.3, 0.2)
    H = np.array([0.06, 0.02, -0.03, -0.04])
    sched = np.array([[1, 0, 0, 1] + (k / 6) * H for k in range(1, 7)])
    fe = fe_newton_pbar(o, t, geom, sched)
    r = rom.solve(torch.tensor([geom], dtype=torch.float64).cuda(),
                  torch.from_numpy(sched[None].copy()).cuda(), api.NewtonOpts(eps_rel=1e-10))
    torch.cuda.synchronize()
    assert int(r["status"][0]) == 0
    err = np.abs(r["pbar"][0].cpu().numpy() - fe).max() / np.abs(fe).max()
    print(f"exact limit: GPU ROM vs FE max rel {err:.2e}")
    assert err <= 1e-8


def test_folding_morph_fails_only_its_instance(setup):
    """A geometry whose morph folds the mesh (det Fmu <= 0) raises SolveError
    in MorphOperator::derive (morph.cpp:116-119): that instance fails, the
    others are unaffected and match the oracle."""
    import torch
    from paper_2307_16894_b200 import api
    g, o, model, rom = setup
    geom, sched = synth.rom_instances(3, 3, 41, 0.1)
    geom[1] = (0.49, 0.49)  # folds the transition ring
    opts = api.NewtonOpts(eps_rel=1e-10, eps_abs=1e-12)
    T = lambda a: torch.from_numpy(a).cuda()
    rg = rom.solve(T(geom), T(sched), opts)
    rg = {k: v.cpu().numpy() for k, v in rg.items()}
    ro = o.rom_solve(model["ids"], model["weights"], model["mode_grads"], geom, sched, eps_rel=1e-10,
                     eps_abs=1e-12)
    assert list(ro["status"]) == [0, 3, 0]
    _check(rg, ro)
    with pytest.raises(api.SolveError):
        rom.ctx.check()


@pytest.mark.parametrize("N", [48, 49, 51, 80, 119])
def test_wide_bases(orc, N):
    """Bases other than N = 50.  N + 1 > 56 columns: the contraction runs one
    instance per CTA with up to 15 column tiles; N = 49 takes the
    remainder-packed kernel with ONE remainder row / column, N = 48 and 51 the
    column-tiled kernel next to it; the warp LU, the effective stiffness and
    the Newton logic are generic in N."""
    import torch
    from paper_2307_16894_b200 import api
    g = api.Rve(16, _mats())
    o = orc.Rve(16, _mats())
    model = synth.rom_model(g.export(), g.n_red, N=N, Q=150, seed=2040 + N)
    rom = api.Rom(g, model["ids"], model["weights"], model["mode_grads"])
    geom, sched = synth.rom_instances(3, 2, 2041, 0.12)
    opts = api.NewtonOpts(eps_rel=1e-10, eps_abs=1e-12)
    T = lambda a: torch.from_numpy(a).cuda()
    rg = rom.solve(T(geom), T(sched), opts, abar=True)
    rg = {k: v.cpu().numpy() for k, v in rg.items()}
    ro = o.rom_solve(model["ids"], model["weights"], model["mode_grads"], geom, sched, eps_rel=1e-10,
                     eps_abs=1e-12, abar=True)
    _check(rg, ro)
    rel = np.linalg.norm(rg["abar"] - ro["abar"], axis=-1) / np.maximum(1.0, np.linalg.norm(ro["abar"], axis=-1))
    print(f"N={N}: abar rel {rel.max():.2e}")
    assert rel.max() <= 1e-8


def test_fused_pipeline_variant():
    """The default pipeline evaluates the FD tangent and the contraction only
    for instances the residual check sends to a Newton update (k_rom_check /
    k_rom_solve).  PODECM_ROM_LAZY=0 selects the fused one (tangent at every
    point every iteration, k_rom_newton); the library reads the variable once
    per process, so this module runs again in a child process under it."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, PODECM_ROM_LAZY="0")
    r = subprocess.run([sys.executable, "-m", "pytest", str(Path(__file__)), "-x", "-q", "-m", "gpu",
                        "-k", "not fused_pipeline_variant", "-p", "no:cacheprovider"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("var,val", [("PODECM_ROM_LU", "smem"), ("PODECM_ROM_F", "fma")])
def test_kernel_variants_bit_identical(setup, monkeypatch, var, val):
    """The register-resident LU (k_rom_solve_reg<50>) against the shared-memory
    LU, and the DMMA F kernel (k_rom_F_mma) against the DFMA one: same
    pivots, same per-element FMA sequence (a DMMA accumulates as the
    sequential FMA chain), so a whole solve — with bisections — must agree
    byte for byte (pbar, iteration counts, status)."""
    import torch
    from paper_2307_16894_b200 import api
    g, o, model, rom = setup
    geom, sched = synth.rom_instances(96, 2, 77, 0.2)  # two big increments
    T = lambda a: torch.from_numpy(a).cuda()
    opts = api.NewtonOpts(eps_rel=1e-10, eps_abs=1e-12, max_iter=3, max_bisect=5)  # increments bisect
    monkeypatch.delenv(var, raising=False)
    a = {k: v.cpu().numpy() for k, v in rom.solve(T(geom), T(sched), opts).items()}
    monkeypatch.setenv(var, val)
    b = {k: v.cpu().numpy() for k, v in rom.solve(T(geom), T(sched), opts).items()}
    assert (a["iters"] > 3).any(), "no increment bisected"
    for k in ("pbar", "iters", "status"):
        assert np.array_equal(np.ascontiguousarray(a[k]).view(np.uint8), np.ascontiguousarray(b[k]).view(np.uint8)), k


def test_remainder_packed_contraction(setup, monkeypatch):
    """k_rom_contract_rp (N = 50: the 48 x 48 block of full DMMA tiles per
    instance, the two remainder rows and columns of both instances of a CTA
    packed into one 8-column tile) against the 56-wide kernel: the remainder
    rows are summed through the transposed tangent, so K differs by rounding
    there and nowhere else; whole solves — odd instance count, with
    bisections — agree to 1e-11 in pbar with equal iteration counts, and the
    packed form holds the oracle tolerance on its own."""
    import torch
    from paper_2307_16894_b200 import api
    g, o, model, rom = setup
    geom, sched = synth.rom_instances(97, 2, 78, 0.2)
    T = lambda a: torch.from_numpy(a).cuda()
    opts = api.NewtonOpts(eps_rel=1e-10, eps_abs=1e-12, max_iter=4, max_bisect=5)
    res = {}
    for mode in ("std", "rp"):
        monkeypatch.setenv("PODECM_ROM_CONTRACT", mode)
        res[mode] = {k: v.cpu().numpy() for k, v in rom.solve(T(geom), T(sched), opts).items()}
    a, b = res["std"], res["rp"]
    # the large-batch forms (two instances per CTA: 8 warps with 3 x 3 tile blocks by default, 12 warps
    # with 2 x 3 blocks under rp23) give every instance the bits of the one-instance form used above
    gl, sl = synth.rom_instances(4097, 1, 79, 0.2)
    big = {}
    for mode in ("rp", "rp23"):
        monkeypatch.setenv("PODECM_ROM_CONTRACT", mode)
        big[mode] = {k: v.cpu().numpy() for k, v in rom.solve(T(gl), T(sl), opts).items()}
    monkeypatch.setenv("PODECM_ROM_CONTRACT", "rp")
    small = {k: v.cpu().numpy() for k, v in rom.solve(T(gl[:33]), T(sl[:33]), opts).items()}
    for k in ("pbar", "iters", "status"):
        assert np.array_equal(big["rp"][k], big["rp23"][k]), k
        assert np.array_equal(big["rp"][k][:33], small[k]), k
    assert np.array_equal(a["status"], b["status"]) and np.array_equal(a["iters"], b["iters"])
    rel = np.abs(a["pbar"] - b["pbar"]).max() / np.abs(a["pbar"]).max()
    print(f"rp vs std: pbar max rel {rel:.2e}; bitwise equal: {np.array_equal(a['pbar'], b['pbar'])}")
    assert 0 < rel <= 1e-11 or np.array_equal(a["pbar"], b["pbar"])
    ro = o.rom_solve(model["ids"], model["weights"], model["mode_grads"], geom, sched, eps_rel=opts.eps_rel,
                     eps_abs=opts.eps_abs, max_iter=opts.max_iter, max_bisect=opts.max_bisect)
    _check(b, ro)


@pytest.mark.parametrize("N", [49, 50])
def test_packed_contraction_large_batch_small_cell(orc, N):
    """The two-instance packed contraction (3 x 3 tile blocks) at N = 49 (one
    remainder row / column) and N = 50 on a 16 x 16 cell, 4,097 instances (an
    odd count: the last CTA holds one instance): every instance has the bits
    of the one-instance form that a 33-instance sub-batch runs, and a spread
    sample meets the oracle tolerance with equal Newton counts."""
    import torch
    from paper_2307_16894_b200 import api
    g = api.Rve(16, _mats())
    o = orc.Rve(16, _mats())
    model = synth.rom_model(g.export(), g.n_red, N=N, Q=56, seed=2050 + N)
    rom = api.Rom(g, model["ids"], model["weights"], model["mode_grads"])
    geom, sched = synth.rom_instances(4097, 2, 2051, 0.12)
    opts = api.NewtonOpts(eps_rel=1e-10, eps_abs=1e-12)
    T = lambda a: torch.from_numpy(a).cuda()
    big = {k: v.cpu().numpy() for k, v in rom.solve(T(geom), T(sched), opts).items()}
    pick = np.unique(np.linspace(0, 4096, 33).astype(np.int64))
    small = {k: v.cpu().numpy() for k, v in rom.solve(T(geom[pick]), T(sched[pick]), opts).items()}
    for k in ("pbar", "iters", "status"):
        assert np.array_equal(big[k][pick], small[k]), k
    ro = o.rom_solve(model["ids"], model["weights"], model["mode_grads"], geom[pick], sched[pick], eps_rel=1e-10,
                     eps_abs=1e-12)
    _check(small, ro)
