"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front end of ``liboracle.so``, the CPU restatement of the reference
hot path (see oracle.hpp for the citations and the parity-pinning status).
Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this package; the product never does.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"          # faithful: glibc exp/log, like the reference
LIB_PDM = HERE / "liboracle_pdm.so"  # same algorithm with the device's portable exp/log
# The reference's own material.cpp / rom.cpp / store.cpp / mesh.cpp compiled
# unchanged against oracle/eigen_shim (oracle/ref/Makefile).  Built only where
# /root/reference exists (this container); the .so travels to the GPU box.
REF_LIB = HERE / "_ref" / "libpodecm_ref.so"
REF_SRC = Path("/root/reference/proj")
_libs = {}

P = C.c_void_p
L = C.c_long
D = C.c_double
I = C.c_int


def build() -> Path:
    r = subprocess.run(["make", "-C", str(HERE), "-s"], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")
    build_ref()
    return LIB


def build_ref() -> Path | None:
    """oracle/_ref from the reference's sources (only where they exist)."""
    if not (REF_SRC / "src" / "material.cpp").exists():
        return REF_LIB if REF_LIB.exists() else None
    r = subprocess.run(["make", "-C", str(HERE / "ref"), "-s", f"REF={REF_SRC}"], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle/_ref build failed:\n{r.stdout}\n{r.stderr}")
    return REF_LIB


_ref = None


def ref_available() -> bool:
    return REF_LIB.exists()


def ref_lib():
    global _ref
    if _ref is None:
        l = C.CDLL(str(REF_LIB))
        l.ref_last_error.restype = C.c_char_p
        l.ref_material_batch.restype = L
        l.ref_material_batch.argtypes = [L, P, P, P, P, P, P, P, D, I, P]
        l.ref_rom_solve.restype = L
        l.ref_rom_solve.argtypes = [I, P, P, I, I, I, P, P, P, L, P, P, P, I, D, D, I, P, P, P, P, P, P, I]
        l.ref_periodic_dof_map.restype = I
        l.ref_periodic_dof_map.argtypes = [I, P]
        l.ref_fingerprint.restype = C.c_ulonglong
        l.ref_fingerprint.argtypes = [I, P]
        l.ref_rom_model_save.restype = I
        l.ref_rom_model_save.argtypes = [C.c_char_p, C.c_ulonglong, I, I, D, L, I, P, I, P, P, P]
        l.ref_assemble.restype = I
        l.ref_assemble.argtypes = [I, P, P, I, P, P, P, P, P, P, P, I, P, P, P, P, P, P]
        l.ref_solve_rve.restype = I
        l.ref_solve_rve.argtypes = [I, P, P, I, P, P, P, P, P, I, D, D, I, P, P, P, P]
        l.ref_rom_model_load.restype = I
        l.ref_rom_model_load.argtypes = [C.c_char_p, C.POINTER(L), C.POINTER(I), C.POINTER(I),
                                         C.POINTER(C.c_ulonglong), C.POINTER(I), C.POINTER(I), C.POINTER(D),
                                         P, P, P, P]
        _ref = l
    return _ref


def ref_material_batch(F, st, mat, h_rel=1e-7, nthreads=0):
    """The reference's large_strain_update + large_strain_tangent per point
    (material.cpp compiled unchanged).  Failed points (status 3) are NaN."""
    F = np.ascontiguousarray(F, dtype=np.float64)
    st = np.ascontiguousarray(st, dtype=np.float64)
    n = F.shape[1]
    out = {"P": np.full((4, n), np.nan), "A": np.full((16, n), np.nan), "st": np.full((6, n), np.nan),
           "status": np.empty(n, np.int32), "extra": np.full((4, n), np.nan)}
    m = np.array([mat.E, mat.nu, mat.sigma_y0, mat.H], dtype=np.float64)
    ref_lib().ref_material_batch(n, _p(m), _p(F), _p(st), _p(out["P"]), _p(out["A"]), _p(out["st"]),
                                 _p(out["status"]), h_rel, nthreads, _p(out["extra"]))
    return out


def ref_rom_solve(n_cells, regions, mats, ids, weights, mode_grads, fmi_q, det_q, sched, eps_rel=1e-8,
                  eps_abs=1e-12, max_iter=25, abar=False, nthreads=0):
    """The reference's rom_solve (+ rom_effective_stiffness at the last step)
    on a structured Q4 cell.  fmi_q [n, Q, 4] / det_q [n, Q]: the morph at the
    ECM points; sched [n, K, 4]."""
    regions = np.ascontiguousarray(regions, dtype=np.int32)
    m = _mats(mats)
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    weights = np.ascontiguousarray(weights, dtype=np.float64)
    mg = np.ascontiguousarray(mode_grads, dtype=np.float64)
    fmi_q = np.ascontiguousarray(fmi_q, dtype=np.float64)
    det_q = np.ascontiguousarray(det_q, dtype=np.float64)
    sched = np.ascontiguousarray(sched, dtype=np.float64)
    Q, N = mg.shape[0], mg.shape[1]
    n, K = sched.shape[0], sched.shape[1]
    out = {"pbar": np.zeros((n, K, 4)), "iters": np.zeros((n, K), np.int32), "resid": np.zeros((n, K)),
           "a_final": np.zeros((n, N)), "status": np.zeros(n, np.int32)}
    ab = np.zeros((n, 16)) if abar else None
    ref_lib().ref_rom_solve(n_cells, _p(regions), _p(m), len(mats), N, Q, _p(ids), _p(weights), _p(mg), n,
                            _p(fmi_q), _p(det_q), _p(sched), K, eps_rel, eps_abs, max_iter, _p(out["pbar"]),
                            _p(out["iters"]), _p(out["resid"]), _p(out["a_final"]), _p(out["status"]), _p(ab),
                            nthreads)
    if abar:
        out["abar"] = ab
    return out


def ref_assemble(n_cells, tables, mats, fmi, det, st0, fbar, w_red, tangent=True):
    """The reference's assemble (microfem.cpp:56-130) of one instance on the Q4
    cell: tables = an exported Rve (regions, grad, w, row_ptr, col_idx);
    fmi [4][nq], det [nq], st0 [6][nq], fbar [4], w_red [n_red].  Returns
    (rc, dict f, K (on the CSR pattern), p_field [4][nq], st1 [6][nq])."""
    nq = tables["w"].shape[0]
    n_red = tables["row_ptr"].shape[0] - 1
    c = lambda a, t=np.float64: np.ascontiguousarray(a, dtype=t)
    out = {"f": np.zeros(n_red), "K": np.zeros(tables["col_idx"].shape[0]), "p_field": np.zeros((4, nq)),
           "st1": np.zeros((6, nq))}
    regs, m = c(tables["regions"], np.int32), _mats(mats)
    g, w, fm, dt, s0, fb, wr = (c(x) for x in (tables["grad"], tables["w"], fmi, det, st0, fbar, w_red))
    rp, ci = c(tables["row_ptr"], np.int32), c(tables["col_idx"], np.int32)
    rc = ref_lib().ref_assemble(n_cells, _p(regs), _p(m), len(mats), _p(g), _p(w), _p(fm), _p(dt), _p(s0), _p(fb),
                                _p(wr), int(tangent), _p(rp), _p(ci), _p(out["f"]), _p(out["K"]),
                                _p(out["p_field"]), _p(out["st1"]))
    return rc, out


def ref_solve_rve(n_cells, tables, mats, fmi, det, sched, eps_rel=1e-8, eps_abs=1e-12, max_iter=25):
    """The reference's solve_rve (microfem.cpp:213-238; dense-LU stand-in for
    SparseLU) of one instance: sched [K][4] -> (rc, pbar [K][4], iters [K],
    resid [K], w_final [n_red])."""
    c = lambda a, t=np.float64: np.ascontiguousarray(a, dtype=t)
    K = sched.shape[0]
    n_red = tables["row_ptr"].shape[0] - 1
    pbar, iters, resid, wf = np.zeros((K, 4)), np.zeros(K, np.int32), np.zeros(K), np.zeros(n_red)
    regs, g, w, fm, dt, sc = (c(tables["regions"], np.int32), c(tables["grad"]), c(tables["w"]), c(fmi), c(det),
                              c(sched))
    rc = ref_lib().ref_solve_rve(n_cells, _p(regs), _p(_mats(mats)), len(mats), _p(g), _p(w), _p(fm), _p(dt),
                                 _p(sc), K, eps_rel, eps_abs, max_iter, _p(pbar), _p(iters), _p(resid), _p(wf))
    return rc, {"pbar": pbar, "iters": iters, "resid": resid, "w_final": wf}


DROPIN_LIB = HERE / "_ref" / "libpodecm_dropin.so"
_dropin = None


def dropin_available() -> bool:
    return DROPIN_LIB.exists()


def dropin_lib():
    """The reference-signature drop-in (paper_2307_16894_b200/dropin) built
    against the reference's headers, with C test drivers (oracle/ref/
    dropin_check.cpp).  Runs the product's device path: GPU tests only."""
    global _dropin
    if _dropin is None:
        l = C.CDLL(str(DROPIN_LIB))
        l.dropin_material.argtypes = [L, P, P, P, P, P, P, P, P, I]
        l.dropin_assemble.restype = I
        l.dropin_assemble.argtypes = [I, P, P, I, P, P, P, P, P, P, P, P, P, P, P, P, P]
        l.dropin_rom_solve.argtypes = [I, P, P, I, P, P, I, I, P, P, P, L, P, P, P, I, D, D, I, P, P, P, P, P, I]
        _dropin = l
    return _dropin


def dropin_material(F, st, mat, per_call):
    F = np.ascontiguousarray(F, dtype=np.float64)
    st = np.ascontiguousarray(st, dtype=np.float64)
    n = F.shape[1]
    out = {"P": np.full((4, n), np.nan), "A": np.full((16, n), np.nan), "st": np.full((6, n), np.nan),
           "extra": np.full((4, n), np.nan), "status": np.empty(n, np.int32)}
    m = np.array([mat.E, mat.nu, mat.sigma_y0, mat.H], dtype=np.float64)
    dropin_lib().dropin_material(n, _p(m), _p(F), _p(st), _p(out["P"]), _p(out["A"]), _p(out["st"]),
                                 _p(out["extra"]), _p(out["status"]), int(per_call))
    return out


def dropin_assemble(n_cells, tables, mats, fmi, det, st0, fbar, w_red):
    nq = tables["w"].shape[0]
    n_red = tables["row_ptr"].shape[0] - 1
    c = lambda a, t=np.float64: np.ascontiguousarray(a, dtype=t)
    out = {"f": np.zeros(n_red), "K": np.zeros(tables["col_idx"].shape[0]), "p_field": np.zeros((4, nq)),
           "st1": np.zeros((6, nq))}
    regs, m = c(tables["regions"], np.int32), _mats(mats)
    g, w, fm, dt, s0, fb, wr = (c(x) for x in (tables["grad"], tables["w"], fmi, det, st0, fbar, w_red))
    rp, ci = c(tables["row_ptr"], np.int32), c(tables["col_idx"], np.int32)
    rc = dropin_lib().dropin_assemble(n_cells, _p(regs), _p(m), len(mats), _p(g), _p(w), _p(fm), _p(dt), _p(s0),
                                      _p(fb), _p(wr), _p(rp), _p(ci), _p(out["f"]), _p(out["K"]),
                                      _p(out["p_field"]), _p(out["st1"]))
    return rc, out


def dropin_rom_solve(n_cells, tables, mats, ids, weights, mode_grads, fmi_q, det_q, sched, eps_rel=1e-8,
                     eps_abs=1e-12, max_iter=25, per_call=True):
    c = lambda a, t=np.float64: np.ascontiguousarray(a, dtype=t)
    mg = c(mode_grads)
    Q, N = mg.shape[0], mg.shape[1]
    n, K = sched.shape[0], sched.shape[1]
    out = {"pbar": np.zeros((n, K, 4)), "iters": np.zeros((n, K), np.int32), "resid": np.zeros((n, K)),
           "a_hist": np.zeros((n, K, N)), "status": np.zeros(n, np.int32)}
    regs, m = c(tables["regions"], np.int32), _mats(mats)
    g, w, idc, wt, fm, dt, sc = (c(tables["grad"]), c(tables["w"]), c(ids, np.int32), c(weights), c(fmi_q), c(det_q),
                                 c(sched))
    dropin_lib().dropin_rom_solve(n_cells, _p(regs), _p(m), len(mats), _p(g), _p(w), N, Q, _p(idc), _p(wt), _p(mg), n,
                                  _p(fm), _p(dt), _p(sc), K, eps_rel, eps_abs, max_iter, _p(out["pbar"]),
                                  _p(out["iters"]), _p(out["resid"]), _p(out["a_hist"]), _p(out["status"]),
                                  int(per_call))
    return out


def ref_periodic_dof_map(n_cells):
    nd = np.empty((n_cells + 1) ** 2, np.int32)
    n_red = ref_lib().ref_periodic_dof_map(n_cells, _p(nd))
    if n_red < 0:
        raise RuntimeError(ref_lib().ref_last_error().decode())
    return nd, n_red


def ref_fingerprint(n_cells, regions) -> int:
    regions = np.ascontiguousarray(regions, dtype=np.int32)
    return int(ref_lib().ref_fingerprint(n_cells, _p(regions)))


def ref_rom_model_save(path, model) -> int:
    modes = np.asfortranarray(model["modes"], dtype=np.float64)
    ids = np.ascontiguousarray(model["ids"], dtype=np.int32)
    w = np.ascontiguousarray(model["weights"], dtype=np.float64)
    mg = np.ascontiguousarray(model["mode_grads"], dtype=np.float64)
    return ref_lib().ref_rom_model_save(str(path).encode(), int(model.get("mesh_tag", 0)), int(model.get("kind", 0)),
                                        int(model.get("n_stress_modes", 0)), float(model.get("ecm_eps", 0.0)),
                                        modes.shape[0], modes.shape[1], modes.ctypes.data_as(C.c_void_p),
                                        ids.shape[0], _p(ids), _p(w), _p(mg))


def ref_rom_model_load(path):
    """(rc, model dict or error message) via the reference's RomModel::load."""
    n_dof, N, Q, tag, kind, nsm, eps = L(), I(), I(), C.c_ulonglong(), I(), I(), D()
    l = ref_lib()
    args = [str(path).encode(), C.byref(n_dof), C.byref(N), C.byref(Q), C.byref(tag), C.byref(kind), C.byref(nsm),
            C.byref(eps)]
    rc = l.ref_rom_model_load(*args, None, None, None, None)
    if rc != 0:
        return rc, l.ref_last_error().decode()
    modes = np.empty((N.value, n_dof.value))  # column-major image
    ids = np.empty(Q.value, np.int32)
    w = np.empty(Q.value)
    mg = np.empty((Q.value, N.value, 4))
    rc = l.ref_rom_model_load(*args, _p(modes), _p(ids), _p(w), _p(mg))
    return rc, {"modes": modes.T, "ids": ids, "weights": w, "mode_grads": mg, "mesh_tag": tag.value,
                "kind": kind.value, "n_stress_modes": nsm.value, "ecm_eps": eps.value}


def lib(libm: str = "glibc"):
    if libm not in _libs:
        path = LIB if libm == "glibc" else LIB_PDM
        if not path.exists():
            build()
        l = C.CDLL(str(path))
        l.orc_material_batch.restype = L
        l.orc_material_batch.argtypes = [L, P, I, P, P, P, P, P, P, P, P, D, I]
        l.orc_rve_create.restype = P
        l.orc_rve_create.argtypes = [I, D, P, I]
        l.orc_rve_destroy.argtypes = [P]
        l.orc_rve_info.argtypes = [P, P]
        l.orc_rve_export.argtypes = [P] + [P] * 8
        l.orc_rve_morph.restype = I
        l.orc_rve_morph.argtypes = [P, D, D, P, P]
        l.orc_rve_assemble.restype = L
        l.orc_rve_assemble.argtypes = [P, L, P, P, P, P, P, P, P, P, P, I]
        l.orc_rom_set_init_resid.restype = None
        l.orc_rom_set_init_resid.argtypes = [P]
        l.orc_rom_solve.restype = L
        l.orc_rom_solve.argtypes = [P, I, I, P, P, P, L, P, P, I, D, D, I, I, P, P, P, P, P, P, I]
        l.orc_rom_effective_stiffness.restype = L
        l.orc_rom_effective_stiffness.argtypes = [P, I, I, P, P, P, L, P, P, P, P, P, P, I]
        l.orc_fe_solve.restype = L
        l.orc_fe_solve.argtypes = [P, L, P, P, I, D, D, I, I, P, P, P, P, P, P, P, I]
        l.orc_fe_effective_stiffness.restype = L
        l.orc_fe_effective_stiffness.argtypes = [P, L, P, P, P, P, P, P, I]
        l.orc_macro_qp_positions.restype = L
        l.orc_macro_qp_positions.argtypes = [I, I, D, D, P]
        l.orc_twoscale_run.restype = I
        l.orc_twoscale_run.argtypes = [P, I, I, D, D, D, I, D, D, I, D, D, P, P, P, P, P]
        l.orc_rom_engines_create.restype = P
        l.orc_rom_engines_create.argtypes = [P, I, I, P, P, P, L, P, P, D, D, I, I]
        l.orc_rom_engines_destroy.argtypes = [P]
        l.orc_rom_engines_respond.restype = L
        l.orc_rom_engines_respond.argtypes = [P, P, P, P, P, P, I]
        l.orc_rom_engines_commit.argtypes = [P]
        l.orc_rom_engines_out_of_range.argtypes = [P, P]
        l.orc_stress_snapshots.restype = L
        l.orc_stress_snapshots.argtypes = [P, P, L, P, I]
        l.orc_max_threads.restype = I
        l.orc_libm.argtypes = [I, L, P, P]
        l.orc_libm_sweep.restype = L
        l.orc_libm_sweep.argtypes = [I, L, C.c_ulonglong, I, D, D, P]
        _libs[libm] = l
    return _libs[libm]


def libm(which: str, x):
    """Host exp/log: 'exp'/'log' (glibc), 'pdm_exp'/'pdm_log' (portable
    variant) or 'gm_exp'/'gm_log' (csrc/gmath.h, the device's restatement of
    glibc, built for the host)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    code = {"exp": 0, "log": 1, "pdm_exp": 2, "pdm_log": 3, "gm_exp": 4, "gm_log": 5, "gm_exp_fast": 6,
            "gm_log_core": 7}[which]
    lib().orc_libm(code, x.size, _p(x), _p(out))
    return out


def libm_sweep(which: str, n: int, seed: int, mode: int, lo: float = 0.0, hi: float = 0.0):
    """gm:: vs glibc over n generated arguments (see orc_libm_sweep):
    returns (mismatch count, first mismatching argument or None)."""
    bad = C.c_double(0.0)
    m = lib().orc_libm_sweep({"exp": 0, "log": 1}[which], int(n), int(seed), int(mode), float(lo),
                             float(hi), C.byref(bad))
    return int(m), (bad.value if m else None)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _mats(mats):
    return np.ascontiguousarray([[m.E, m.nu, m.sigma_y0, m.H] for m in mats], dtype=np.float64)


def max_threads() -> int:
    """Host threads available to this process (not OpenMP's current setting,
    which a previous nthreads=1 call may have lowered)."""
    import os
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def material_batch(F, st, mats, region=None, h_rel=1e-7, tangent=True, nthreads=0, libm="glibc"):
    """large_strain_update + large_strain_tangent per point (material.cpp).
    libm="pdm" uses the device's portable exp/log (algorithm-only check)."""
    F = np.ascontiguousarray(F, dtype=np.float64)
    st = np.ascontiguousarray(st, dtype=np.float64)
    n = F.shape[1]
    P_ = np.empty((4, n))
    A = np.empty((16, n)) if tangent else None
    so = np.empty((6, n))
    ex = np.empty((4, n))
    status = np.empty(n, np.int32)
    m = _mats(mats)
    reg = None if region is None else np.ascontiguousarray(region, dtype=np.int32)
    lib(libm).orc_material_batch(n, _p(m), len(mats), _p(reg), _p(F), _p(st), _p(P_), _p(A), _p(so),
                                 _p(status), _p(ex), h_rel, nthreads)
    return {"P": P_, "A": A, "st": so, "status": status, "dgamma": ex[0], "f_trial": ex[1],
            "q_trial": ex[2], "mises": ex[3]}


class Rve:
    """Structured Q4 RveProblem restated on the CPU."""

    def __init__(self, n_cells, mats, r0=0.25, libm="glibc"):
        """libm="pdm": the device's portable exp/log instead of glibc's
        (separates the algorithm from the libm floor)."""
        m = _mats(mats)
        self.L = lib(libm)
        self.h = self.L.orc_rve_create(n_cells, r0, _p(m), len(mats))
        info = np.zeros(6, dtype=np.int64)
        self.L.orc_rve_info(self.h, _p(info))
        self.n_nodes, self.n_elems, self.n_qp, self.n_red, self.nnz, self.anchor = (int(x) for x in info)

    def export(self):
        t = {"nodes": np.empty((self.n_nodes, 2)), "elems": np.empty((self.n_elems, 4), np.int32),
             "regions": np.empty(self.n_elems, np.int32), "grad": np.empty((self.n_qp, 4, 2)),
             "w": np.empty(self.n_qp), "node_dof": np.empty(self.n_nodes, np.int32),
             "row_ptr": np.empty(self.n_red + 1, np.int32), "col_idx": np.empty(self.nnz, np.int32)}
        self.L.orc_rve_export(self.h, *(_p(t[k]) for k in ("nodes", "elems", "regions", "grad", "w",
                                                          "node_dof", "row_ptr", "col_idx")))
        return t

    def morph(self, a, b):
        fmi = np.empty((4, self.n_qp))
        det = np.empty(self.n_qp)
        rc = self.L.orc_rve_morph(self.h, a, b, _p(fmi), _p(det))
        return fmi, det, rc

    def assemble(self, geom, fbar, w_red, st0, tangent=True, states1=True, store_stress=False,
                 nthreads=0):
        n = geom.shape[0]
        geom = np.ascontiguousarray(geom, dtype=np.float64)
        fbar = np.ascontiguousarray(fbar, dtype=np.float64)
        w_red = np.ascontiguousarray(w_red, dtype=np.float64)
        st0 = np.ascontiguousarray(st0, dtype=np.float64)
        f = np.empty((n, self.n_red))
        K = np.empty((n, self.nnz)) if tangent else None
        s1 = np.empty((n, 6, self.n_qp)) if states1 else None
        pf = np.empty((n, 4, self.n_qp)) if store_stress else None
        status = np.empty(n, np.int32)
        self.L.orc_rve_assemble(self.h, n, _p(geom), _p(fbar), _p(w_red), _p(st0), _p(s1), _p(f), _p(K),
                               _p(pf), _p(status), nthreads)
        return {"f": f, "K": K, "st1": s1, "p_field": pf, "status": status}

    def stress_snapshots(self, U, nthreads=0):
        """Weighted stress snapshots W [L][n_qp][4] of nodal fields U (2n x L)."""
        U = np.asfortranarray(U, dtype=np.float64)
        L = U.shape[1]
        W = np.empty((L, self.n_qp, 4))
        fails = self.L.orc_stress_snapshots(self.h, U.ctypes.data_as(C.c_void_p), L, _p(W), nthreads)
        return W, int(fails)

    def rom_solve(self, ids, weights, mode_grads, geom, sched, eps_rel=1e-8, eps_abs=1e-12,
                  max_iter=25, max_bisect=5, nthreads=0, abar=False):
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        weights = np.ascontiguousarray(weights, dtype=np.float64)
        mg = np.ascontiguousarray(mode_grads, dtype=np.float64)
        geom = np.ascontiguousarray(geom, dtype=np.float64)
        sched = np.ascontiguousarray(sched, dtype=np.float64)
        Q, N = mg.shape[0], mg.shape[1]
        n, K = sched.shape[0], sched.shape[1]
        pbar = np.empty((n, K, 4))
        iters = np.empty((n, K), np.int32)
        resid = np.empty((n, K))
        af = np.empty((n, N))
        status = np.empty(n, np.int32)
        ab = np.zeros((n, 16)) if abar else None
        r0 = np.zeros((n, K))  # initial residual per increment (tolerance = max(eps_rel r0, eps_abs))
        self.L.orc_rom_set_init_resid(_p(r0))
        try:
            self.L.orc_rom_solve(self.h, N, Q, _p(ids), _p(weights), _p(mg), n, _p(geom), _p(sched), K,
                                eps_rel, eps_abs, max_iter, max_bisect, _p(pbar), _p(iters), _p(resid),
                                _p(af), _p(status), _p(ab) if abar else None, nthreads)
        finally:
            self.L.orc_rom_set_init_resid(None)
        out = {"pbar": pbar, "iters": iters, "resid": resid, "a_final": af, "status": status, "init_resid": r0}
        if abar:
            out["abar"] = ab
        return out

    def fe_solve(self, geom, sched, eps_rel=1e-8, eps_abs=1e-12, max_iter=25, max_bisect=5, nthreads=0,
                 history=False):
        """Full-order solve_rve (microfem.cpp:213-238) per instance: pbar
        [n, K, 4], iters [n, K], resid [n, K], w_final [n, n_red], status [n]."""
        geom = np.ascontiguousarray(geom, dtype=np.float64)
        sched = np.ascontiguousarray(sched, dtype=np.float64)
        n, K = sched.shape[0], sched.shape[1]
        pbar = np.empty((n, K, 4))
        iters = np.empty((n, K), np.int32)
        resid = np.empty((n, K))
        wf = np.empty((n, self.n_red))
        status = np.empty(n, np.int32)
        wh = np.zeros((n, K, self.n_red)) if history else None
        ph = np.zeros((n, K, 4, self.n_qp)) if history else None
        self.L.orc_fe_solve(self.h, n, _p(geom), _p(sched), K, eps_rel, eps_abs, max_iter, max_bisect, _p(pbar),
                            _p(iters), _p(resid), _p(wf), _p(status), _p(wh), _p(ph), nthreads)
        out = {"pbar": pbar, "iters": iters, "resid": resid, "w_final": wf, "status": status}
        if history:
            out.update(w_hist=wh, p_hist=ph)
        return out

    def fe_effective_stiffness(self, geom, st0, fbar, w, nthreads=0):
        """effective_stiffness (microfem.cpp:240-313): abar [n, 16], status [n]."""
        geom, st0, fbar, w = (np.ascontiguousarray(x, dtype=np.float64) for x in (geom, st0, fbar, w))
        n = geom.shape[0]
        abar = np.zeros((n, 16))
        status = np.empty(n, np.int32)
        self.L.orc_fe_effective_stiffness(self.h, n, _p(geom), _p(st0), _p(fbar), _p(w), _p(abar), _p(status),
                                          nthreads)
        return abar, status

    def rom_effective_stiffness(self, ids, weights, mode_grads, geom, st0, fbar, a, nthreads=0):
        """rom_effective_stiffness (rom.cpp:202-241): abar [n, 16] (Tensor4
        storage r + 4c), status [n]."""
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        weights = np.ascontiguousarray(weights, dtype=np.float64)
        mg = np.ascontiguousarray(mode_grads, dtype=np.float64)
        geom, st0, fbar, a = (np.ascontiguousarray(x, dtype=np.float64) for x in (geom, st0, fbar, a))
        Q, N = mg.shape[0], mg.shape[1]
        n = geom.shape[0]
        abar = np.zeros((n, 16))
        status = np.empty(n, np.int32)
        self.L.orc_rom_effective_stiffness(self.h, N, Q, _p(ids), _p(weights), _p(mg), n, _p(geom), _p(st0),
                                          _p(fbar), _p(a), _p(abar), _p(status), nthreads)
        return abar, status

    def rom_sensitivity(self, ids, weights, mode_grads, geom, sched, h, **kw):
        """rom_sensitivity (rom.cpp:243-263) on the analytic geometry (a, b):
        central differences of the final pbar, step h * max(1, |param|).
        Returns grad [n, 2, 4] and status [n]."""
        geom = np.ascontiguousarray(geom, dtype=np.float64)
        sched = np.ascontiguousarray(sched, dtype=np.float64)
        n = geom.shape[0]
        grad = np.empty((n, 2, 4))
        status = np.zeros(n, np.int32)
        for k in range(2):
            step = h * np.maximum(1.0, np.abs(geom[:, k]))
            lo, hi = geom.copy(), geom.copy()
            lo[:, k] -= step
            hi[:, k] += step
            rl = self.rom_solve(ids, weights, mode_grads, lo, sched, **kw)
            rh = self.rom_solve(ids, weights, mode_grads, hi, sched, **kw)
            grad[:, k, :] = (rh["pbar"][:, -1, :] - rl["pbar"][:, -1, :]) / (2.0 * step)[:, None]
            status |= rl["status"] | rh["status"]
        return grad, np.where(status != 0, 3, 0).astype(np.int32)

    def __del__(self):
        try:
            if self.h:
                self.L.orc_rve_destroy(self.h)
                self.h = None
        except Exception:
            pass


class RomEngines:
    """Batch of RomMicroEngine (twoscale.cpp:53-96) on the oracle: respond /
    commit / out_of_range, one engine per geometry (a, b)."""

    def __init__(self, rve: "Rve", ids, weights, mode_grads, geom, bounds=None, eps_rel=1e-8,
                 eps_abs=1e-12, max_iter=25, max_bisect=5):
        self._keep = [np.ascontiguousarray(ids, dtype=np.int32), np.ascontiguousarray(weights, dtype=np.float64),
                      np.ascontiguousarray(mode_grads, dtype=np.float64)]
        ids, weights, mg = self._keep
        geom = np.ascontiguousarray(geom, dtype=np.float64)
        self.n = geom.shape[0]
        self.N = mg.shape[1]
        b = None if bounds is None else np.ascontiguousarray(bounds, dtype=np.float64).reshape(6)
        self.rve = rve
        self.h = self.rve.L.orc_rom_engines_create(rve.h, self.N, ids.shape[0], _p(ids), _p(weights), _p(mg), self.n,
                                              _p(geom), _p(b), eps_rel, eps_abs, max_iter, max_bisect)

    def respond(self, fbar, abar=False, nthreads=0):
        fbar = np.ascontiguousarray(fbar, dtype=np.float64)
        pbar = np.empty((self.n, 4))
        ab = np.empty((self.n, 16)) if abar else None
        iters = np.empty(self.n, np.int32)
        status = np.empty(self.n, np.int32)
        self.rve.L.orc_rom_engines_respond(self.h, _p(fbar), _p(pbar), _p(ab), _p(iters), _p(status), nthreads)
        out = {"pbar": pbar, "iters": iters, "status": status}
        if abar:
            out["abar"] = ab
        return out

    def commit(self):
        self.rve.L.orc_rom_engines_commit(self.h)

    def out_of_range(self):
        out = np.empty(self.n, np.int32)
        self.rve.L.orc_rom_engines_out_of_range(self.h, _p(out))
        return out

    def __del__(self):
        try:
            if self.h:
                self.rve.L.orc_rom_engines_destroy(self.h)
                self.h = None
        except Exception:
            pass


def macro_qp_positions(nx, ny, width=2.0, height=1.0):
    n = lib().orc_macro_qp_positions(nx, ny, width, height, None)
    x = np.empty((n, 2))
    lib().orc_macro_qp_positions(nx, ny, width, height, _p(x))
    return x


def run_twoscale(nx=5, ny=3, width=2.0, height=1.0, peak=0.2, steps=50, eps_rel=1e-8, eps_abs=1e-12, max_iter=25,
                 engines: "RomEngines | None" = None, E=1.0, nu=0.3):
    """run_twoscale (twoscale.cpp:131-242) with the oracle's RomMicroEngines or
    LinearElasticEngine(E, nu).  Returns the result dict and the status (0/3)."""
    n_nodes = (2 * nx + 1) * (2 * ny + 1) - nx * ny
    lf, comp, uf = np.zeros(steps), np.zeros(steps), np.zeros(2 * n_nodes)
    it = np.zeros(steps, np.int32)
    rn = C.c_double()
    L = engines.rve.L if engines is not None else lib()
    st = L.orc_twoscale_run(engines.h if engines is not None else None, nx, ny, width, height, peak, steps, eps_rel,
                            eps_abs, max_iter, E, nu, _p(lf), _p(comp), _p(it), _p(uf), C.byref(rn))
    return {"load_factor": lf, "compliance": comp, "iters": it, "u_final": uf, "residual_norm": rn.value}, st
