"""Host-side mirror of the reference interfaces for the hot path.

Names and argument meaning follow /root/reference/proj/include/podecm:
``PlasticityParams`` (material.hpp:9-17), ``large_strain_update`` +
``large_strain_tangent`` (material.hpp:69-75) batched as
:func:`material_batch`, ``RveProblem``/``assemble`` (microfem.hpp:16-77) as
:class:`Rve` / :meth:`Rve.assemble`, ``RomModel``/``rom_solve``
(rom.hpp:15-88) as :class:`Rom` / :meth:`Rom.solve`.  Errors surface as the
reference's exception kinds (``SolveError``, ``ConfigError``).

Device memory, streams and tensors come from PyTorch (plumbing only); every
computation runs in the sm_100a kernels of ``libpodecm_cuda.so`` through the
C-ABI.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import ConfigError, SolveError, podecm_ecm_opts, podecm_newton, podecm_params

__all__ = ["PlasticityParams", "NewtonOpts", "Context", "material_batch", "Rve", "Rom",
           "pod", "EcmOpts", "ecm_mode_grads", "ecm_stress_snapshots", "ecm_select",
           "ConfigError", "SolveError", "matrix_params", "inclusion_params"]


@dataclass(frozen=True)
class PlasticityParams:
    """material.hpp:9-17 (defaults: E=1, nu=0.3, elastic sigma_y0=1e300, H=0)."""
    E: float = 1.0
    nu: float = 0.3
    sigma_y0: float = 1e300
    H: float = 0.0

    def c(self) -> podecm_params:
        return podecm_params(self.E, self.nu, self.sigma_y0, self.H)


def matrix_params() -> PlasticityParams:
    """BASELINE config-0 matrix phase: E=1, nu=0.3, sigma_y=0.01, H=0.1."""
    return PlasticityParams(1.0, 0.3, 0.01, 0.1)


def inclusion_params() -> PlasticityParams:
    """BASELINE config-0 inclusion: E=10, nu=0.3, elastic."""
    return PlasticityParams(10.0, 0.3, 1e300, 0.0)


@dataclass
class NewtonOpts:
    """microfem.hpp:45-56 plus the bisection depth of rom.hpp:66-73."""
    eps_rel: float = 1e-8
    eps_abs: float = 1e-12
    max_iter: int = 25
    force_ref: float = 0.0
    max_bisect: int = 5

    def c(self) -> podecm_newton:
        return podecm_newton(self.eps_rel, self.eps_abs, self.force_ref, self.max_iter,
                             self.max_bisect)


def _mats(mats) -> tuple:
    arr = (podecm_params * len(mats))(*[m.c() for m in mats])
    return arr, len(mats)


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ConfigError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ConfigError("expected a contiguous tensor")
    return C.c_void_p(t.data_ptr())


def _f64(t: torch.Tensor, shape, name: str) -> torch.Tensor:
    if t.dtype != torch.float64 or tuple(t.shape) != tuple(shape):
        raise ConfigError(f"{name}: expected float64 {tuple(shape)}, got {t.dtype} {tuple(t.shape)}")
    return t


class Context:
    """One C-ABI context per device (podecm_ctx)."""

    _default: dict = {}

    def __init__(self, device: int = 0):
        if not torch.cuda.is_available():
            raise _lib.CudaError("no CUDA device: the hot path has no CPU fallback")
        self.lib = _lib.load()
        self.device = device
        torch.cuda.set_device(device)
        h = C.c_void_p()
        _lib.raise_for(self.lib.podecm_ctx_create(device, C.byref(h)), None, "podecm_ctx_create")
        self.h = h

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = Context(device)
        return cls._default[device]

    def stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def check(self) -> None:
        """Synchronise and raise SolveError if any item failed (podecm_check)."""
        _lib.raise_for(self.lib.podecm_check(self.h, self.stream()), self.h, "podecm_check")

    def launches(self) -> int:
        return int(self.lib.podecm_launch_count(self.h))

    def set_timing(self, on: bool) -> None:
        """Per-kernel CUDA-event timing inside the library (bench only)."""
        self.lib.podecm_set_timing(self.h, 1 if on else 0)

    def timings(self) -> dict:
        """{kernel name: (total ms, launches)} since the previous call."""
        buf = C.create_string_buffer(4096)
        ms = (C.c_double * 64)()
        cnt = (C.c_int64 * 64)()
        n = self.lib.podecm_get_timings(self.h, buf, 4096, ms, cnt, 64)
        names = buf.value.decode().split("\n")[:n]
        return {nm: (ms[k], int(cnt[k])) for k, nm in enumerate(names)}

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.podecm_ctx_destroy(self.h)
                self.h = None
        except Exception:
            pass


def material_batch(F: torch.Tensor, st: torch.Tensor, mats, region: torch.Tensor | None = None,
                   h_rel: float = 1e-7, tangent: bool = True, state: bool = True,
                   ctx: Context | None = None, out: dict | None = None):
    """Batched large_strain_update + large_strain_tangent (material.hpp:69-75).

    F: [4, n] float64 (flatten order), st: [6, n] (Fp00, Fp10, Fp01, Fp11,
    Fp_zz, xi).  Returns dict P [4, n], A [16, n] (plane r + 4c), st [6, n],
    status [n] int32.  Raises nothing per point: check ``status`` or call
    ``ctx.check()`` for the reference's throw-on-first-failure behaviour.
    """
    ctx = ctx or Context.default(F.device.index or 0)
    n = F.shape[1]
    _f64(F, (4, n), "F")
    _f64(st, (6, n), "st")
    o = out or {}
    P = o.get("P") if o.get("P") is not None else torch.empty((4, n), dtype=torch.float64, device=F.device)
    A = (o.get("A") if o.get("A") is not None else torch.empty((16, n), dtype=torch.float64, device=F.device)) if tangent else None
    S = (o.get("st") if o.get("st") is not None else torch.empty((6, n), dtype=torch.float64, device=F.device)) if state else None
    status = o.get("status") if o.get("status") is not None else torch.empty(n, dtype=torch.int32, device=F.device)
    arr, nm = _mats(mats)
    rc = ctx.lib.podecm_material_batch(ctx.h, ctx.stream(), n, arr, nm, _ptr(region), _ptr(F),
                                       _ptr(st), _ptr(P), _ptr(A), _ptr(S), _ptr(status), h_rel)
    _lib.raise_for(rc, ctx.h, "podecm_material_batch")
    return {"P": P, "A": A, "st": S, "status": status}


class Rve:
    """RveProblem (microfem.hpp:16-30) of the structured Q4 unit cell."""

    def __init__(self, n_cells: int, mats, r0: float = 0.25, ctx: Context | None = None):
        self.ctx = ctx or Context.default()
        self.lib = self.ctx.lib
        arr, nm = _mats(mats)
        h = C.c_void_p()
        _lib.raise_for(self.lib.podecm_rve_create_q4(self.ctx.h, n_cells, r0, arr, nm, C.byref(h)),
                       self.ctx.h, "podecm_rve_create_q4")
        self.h = h
        self.mats = list(mats)
        self.n_cells = n_cells
        self.r0 = r0
        info = (C.c_int64 * 6)()
        self.lib.podecm_rve_info(h, info)
        self.n_nodes, self.n_elems, self.n_qp, self.n_red, self.nnz, self.anchor = (int(x) for x in info)
        self.n_trip = int(self.lib.podecm_rve_n_triplets(h))

    def export(self) -> dict:
        import numpy as np
        t = {
            "nodes": np.empty((self.n_nodes, 2)), "elems": np.empty((self.n_elems, 4), np.int32),
            "regions": np.empty(self.n_elems, np.int32), "grad": np.empty((self.n_qp, 4, 2)),
            "w": np.empty(self.n_qp), "node_dof": np.empty(self.n_nodes, np.int32),
            "row_ptr": np.empty(self.n_red + 1, np.int32), "col_idx": np.empty(self.nnz, np.int32),
            "slot_ptr": np.empty(self.nnz + 1, np.int32), "slot_terms": np.empty(self.n_trip, np.int32),
        }
        p = lambda a: a.ctypes.data_as(C.c_void_p)
        self.lib.podecm_rve_export(self.h, *(p(t[k]) for k in ("nodes", "elems", "regions", "grad", "w",
                                                                "node_dof", "row_ptr", "col_idx",
                                                                "slot_ptr", "slot_terms")))
        return t

    def fingerprint(self) -> int:
        """Mesh::fingerprint (mesh.cpp:158-180) of this cell (non-Tri6 kind byte 1)."""
        return int(self.lib.podecm_rve_fingerprint(self.h))

    def morph(self, geom: torch.Tensor):
        """Analytic morph at every qp: (fmu_inv [n,4,nqp], det [n,nqp], status)."""
        n = geom.shape[0]
        _f64(geom, (n, 2), "geom")
        fmi = torch.empty((n, 4, self.n_qp), dtype=torch.float64, device=geom.device)
        det = torch.empty((n, self.n_qp), dtype=torch.float64, device=geom.device)
        status = torch.empty(n, dtype=torch.int32, device=geom.device)
        rc = self.lib.podecm_rve_morph(self.ctx.h, self.ctx.stream(), self.h, n, _ptr(geom), _ptr(fmi),
                                       _ptr(det), _ptr(status))
        _lib.raise_for(rc, self.ctx.h, "podecm_rve_morph")
        return fmi, det, status

    def assemble(self, fbar: torch.Tensor, w_red: torch.Tensor, st0: torch.Tensor,
                 geom: torch.Tensor | None = None, morph: torch.Tensor | None = None,
                 tangent: bool = True, states1: bool = True, store_stress: bool = False,
                 out: dict | None = None, store_tangent_field: bool = False) -> dict:
        """Batched assemble (microfem.cpp:56-130): f [n, n_red], K values
        [n, nnz] (CSR pattern of :meth:`export`), st1 [n, 6, nqp], p_field,
        and with store_tangent_field the FD tangent per qp, a_field [n, 16, nqp]."""
        n = fbar.shape[0]
        dev = fbar.device
        _f64(fbar, (n, 4), "fbar")
        _f64(w_red, (n, self.n_red), "w_red")
        _f64(st0, (n, 6, self.n_qp), "st0")
        if geom is not None:
            _f64(geom, (n, 2), "geom")
        if morph is not None:
            _f64(morph, (n, 5, self.n_qp), "morph")
        o = out or {}
        mk = lambda k, shape: o[k] if o.get(k) is not None else torch.empty(shape, dtype=torch.float64, device=dev)
        f = mk("f", (n, self.n_red))
        K = mk("K", (n, self.nnz)) if tangent else None
        S1 = mk("st1", (n, 6, self.n_qp)) if states1 else None
        PF = mk("p_field", (n, 4, self.n_qp)) if store_stress else None
        status = o["status"] if o.get("status") is not None else torch.empty(n, dtype=torch.int32, device=dev)
        AF = mk("a_field", (n, 16, self.n_qp)) if store_tangent_field else None
        rc = self.lib.podecm_assemble_batch_ex(self.ctx.h, self.ctx.stream(), self.h, n, _ptr(geom),
                                               _ptr(morph), _ptr(fbar), _ptr(w_red), _ptr(st0), _ptr(S1),
                                               _ptr(f), _ptr(K), _ptr(PF), _ptr(status), _ptr(AF))
        _lib.raise_for(rc, self.ctx.h, "podecm_assemble_batch")
        r = {"f": f, "K": K, "st1": S1, "p_field": PF, "status": status}
        if store_tangent_field:
            r["a_field"] = AF
        return r

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.podecm_rve_destroy(self.h)
                self.h = None
        except Exception:
            pass


class Rom:
    """RomModel (rom.hpp:15-30) bound to an Rve: ECM ids, weights, mode_grads."""

    def __init__(self, rve: Rve, ids, weights, mode_grads):
        import numpy as np
        self.rve = rve
        self.ctx = rve.ctx
        self.lib = rve.lib
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        weights = np.ascontiguousarray(weights, dtype=np.float64)
        mode_grads = np.ascontiguousarray(mode_grads, dtype=np.float64)
        self.Q = ids.shape[0]
        self.N = mode_grads.shape[1]
        if mode_grads.shape != (self.Q, self.N, 4) or weights.shape != (self.Q,):
            raise ConfigError("rom: inconsistent ids/weights/mode_grads shapes")
        p = lambda a: a.ctypes.data_as(C.c_void_p)
        h = C.c_void_p()
        _lib.raise_for(self.lib.podecm_rom_create(self.ctx.h, rve.h, self.N, self.Q, p(ids), p(weights),
                                                  p(mode_grads), C.byref(h)),
                       self.ctx.h, "podecm_rom_create")
        self.h = h

    def solve(self, geom: torch.Tensor, sched: torch.Tensor, opts: NewtonOpts | None = None,
              out: dict | None = None, abar: bool = False) -> dict:
        """Batched rom_solve (rom.cpp:177-200): pbar [n, K, 4] history,
        iters [n, K], resid [n, K], a_final [n, N], status [n].  abar=True adds
        run_online's effective stiffness at the last increment
        (pipeline.cpp:456-483): abar [n, 16], Tensor4 storage r + 4c.

        Lazy tangent (default): the reference assembles K with the FD tangent
        at every Newton check (rom.cpp:132), also at the iterate that then
        meets the tolerance, and discards it there; this pipeline skips that
        tangent.  The one observable difference: if an FD evaluation at such a
        converged iterate hit a non-positive elastic stretch, the reference
        would fail the attempt and bisect while this pipeline accepts the
        step.  PODECM_ROM_LAZY=0 selects the strict order (every check with
        its tangent); tests/test_gpu_rom.py runs the module both ways."""
        opts = opts or NewtonOpts()
        n, K = sched.shape[0], sched.shape[1]
        dev = sched.device
        _f64(geom, (n, 2), "geom")
        _f64(sched, (n, K, 4), "sched")
        o = out or {}
        pbar = o.get("pbar") if o.get("pbar") is not None else torch.empty((n, K, 4), dtype=torch.float64, device=dev)
        iters = o.get("iters") if o.get("iters") is not None else torch.empty((n, K), dtype=torch.int32, device=dev)
        resid = o.get("resid") if o.get("resid") is not None else torch.empty((n, K), dtype=torch.float64, device=dev)
        af = o.get("a_final") if o.get("a_final") is not None else torch.empty((n, self.N), dtype=torch.float64, device=dev)
        status = o.get("status") if o.get("status") is not None else torch.empty(n, dtype=torch.int32, device=dev)
        ab = torch.zeros((n, 16), dtype=torch.float64, device=dev) if abar else None
        oc = opts.c()
        rc = self.lib.podecm_rom_solve_batch_ex(self.ctx.h, self.ctx.stream(), self.h, n, _ptr(geom),
                                                _ptr(sched), K, C.byref(oc), _ptr(pbar), _ptr(iters),
                                                _ptr(resid), _ptr(af), _ptr(status), _ptr(ab))
        _lib.raise_for(rc, self.ctx.h, "podecm_rom_solve_batch")
        self.global_iterations = int(self.lib.podecm_rom_global_iterations(self.h))
        r = {"pbar": pbar, "iters": iters, "resid": resid, "a_final": af, "status": status}
        if abar:
            r["abar"] = ab
        return r

    def effective_stiffness(self, geom: torch.Tensor, st0: torch.Tensor, fbar: torch.Tensor,
                            a: torch.Tensor) -> dict:
        """Batched rom_effective_stiffness (rom.cpp:202-241): history st0
        [n, 6, Q] at the ECM points, fbar [n, 4], reduced coordinates a [n, N]
        -> abar [n, 16] (Tensor4 storage r + 4c), status [n]."""
        n = geom.shape[0]
        _f64(geom, (n, 2), "geom")
        _f64(st0, (n, 6, self.Q), "st0")
        _f64(fbar, (n, 4), "fbar")
        _f64(a, (n, self.N), "a")
        abar = torch.zeros((n, 16), dtype=torch.float64, device=geom.device)
        status = torch.empty(n, dtype=torch.int32, device=geom.device)
        rc = self.lib.podecm_rom_effective_stiffness_batch(self.ctx.h, self.ctx.stream(), self.h, n, _ptr(geom),
                                                           _ptr(st0), _ptr(fbar), _ptr(a), _ptr(abar),
                                                           _ptr(status))
        _lib.raise_for(rc, self.ctx.h, "podecm_rom_effective_stiffness_batch")
        return {"abar": abar, "status": status}

    def sensitivity(self, geom: torch.Tensor, sched: torch.Tensor, opts: NewtonOpts | None = None,
                    h: float = 1e-4) -> dict:
        """Batched rom_sensitivity (rom.cpp:243-263) over the analytic
        geometry (a, b): grad [n, 2, 4] = d pbar_final / d (a, b), status [n]."""
        opts = opts or NewtonOpts()
        n, K = sched.shape[0], sched.shape[1]
        _f64(geom, (n, 2), "geom")
        _f64(sched, (n, K, 4), "sched")
        grad = torch.zeros((n, 2, 4), dtype=torch.float64, device=geom.device)
        status = torch.empty(n, dtype=torch.int32, device=geom.device)
        oc = opts.c()
        rc = self.lib.podecm_rom_sensitivity_batch(self.ctx.h, self.ctx.stream(), self.h, n, _ptr(geom),
                                                   _ptr(sched), K, C.byref(oc), float(h), _ptr(grad),
                                                   _ptr(status))
        _lib.raise_for(rc, self.ctx.h, "podecm_rom_sensitivity_batch")
        return {"grad": grad, "status": status}

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.podecm_rom_destroy(self.h)
                self.h = None
        except Exception:
            pass


# ---------------------------------------------------------------- POD / ECM --
def pod(S_cm: torch.Tensor, max_modes: int, tol_rel: float = 1e-10, gram_diag=None,
        ctx: Context | None = None):
    """pod_diag (podkit.cpp:117-127) of a column-major snapshot matrix given as
    its transpose ``S_cm`` [n_snap, n_dof] (row s = snapshot s, contiguous).
    Returns (modes^T [kept, n_dof], eigenvalues [n_snap] descending)."""
    ctx = ctx or Context.default(S_cm.device.index or 0)
    n_snap, n_dof = S_cm.shape
    C_ = torch.empty((n_snap, n_snap), dtype=torch.float64, device=S_cm.device)
    rc = ctx.lib.podecm_pod_gram(ctx.h, ctx.stream(), _ptr(S_cm), n_dof, n_snap, _ptr(gram_diag), _ptr(C_))
    _lib.raise_for(rc, ctx.h, "podecm_pod_gram")
    modes = torch.empty((max_modes, n_dof), dtype=torch.float64, device=S_cm.device)
    ev = torch.empty(n_snap, dtype=torch.float64, device=S_cm.device)
    kept = C.c_int()
    rc = ctx.lib.podecm_pod_modes(ctx.h, ctx.stream(), _ptr(S_cm), n_dof, n_snap, _ptr(C_),
                                  _ptr(gram_diag), max_modes, tol_rel, _ptr(modes), _ptr(ev), C.byref(kept))
    _lib.raise_for(rc, ctx.h, "podecm_pod_modes")
    return modes[: kept.value], ev


def _gram_peer(ctx: "Context", S_local: torch.Tensor, n_snap: int, world: int, rank: int) -> torch.Tensor:
    """The summed Gram sum_k S_k^T S_k by the peer-memory path: each rank's
    DMMA GEMM stores its partial straight into the row owners' receive slots
    (podecm_pod_gram_peer, CUDA IPC mappings: NVLink stores across GPUs), the
    owner sums its slots in rank order (podecm_pod_gram_reduce) and every rank
    pulls the reduced rows of the other owners (podecm_peer_copy).  Host-side
    barriers separate the phases, so no kernel ever waits on another rank's.
    Returns the full n_snap^2 Gram on this rank's device."""
    import torch.distributed as dist
    n_loc = S_local.shape[1]
    row0 = [n_snap * o // world for o in range(world + 1)]
    rows = row0[rank + 1] - row0[rank]
    L = ctx.lib

    def alloc(nbytes):
        p = C.c_void_p()
        _lib.raise_for(L.podecm_dev_alloc(ctx.h, nbytes, C.byref(p)), ctx.h, "podecm_dev_alloc")
        return p

    def share(p):
        h = (C.c_ubyte * 64)()
        _lib.raise_for(L.podecm_ipc_handle(ctx.h, p, C.cast(h, C.c_void_p)), ctx.h, "podecm_ipc_handle")
        hs = [None] * world
        dist.all_gather_object(hs, bytes(h))
        out = []
        for o in range(world):
            if o == rank:
                out.append(p)
                continue
            q = C.c_void_p()
            hb = (C.c_ubyte * 64).from_buffer_copy(hs[o])
            _lib.raise_for(L.podecm_ipc_open(ctx.h, C.cast(hb, C.c_void_p), C.byref(q)), ctx.h, "podecm_ipc_open")
            out.append(q)
        return out

    recv = alloc(world * rows * n_snap * 8)  # [world][rows][n_snap]: the partials of this rank's rows
    gfull = alloc(n_snap * n_snap * 8)
    recv_all, g_all = share(recv), share(gfull)
    try:
        ptrs = (C.c_void_p * world)(*[p.value for p in recv_all])
        r0 = (C.c_int64 * (world + 1))(*row0)
        rc = L.podecm_pod_gram_peer(ctx.h, ctx.stream(), _ptr(S_local), n_loc, n_snap, None,
                                    C.cast(ptrs, C.c_void_p), rank, world, C.cast(r0, C.c_void_p))
        _lib.raise_for(rc, ctx.h, "podecm_pod_gram_peer")
        torch.cuda.synchronize(S_local.device)
        dist.barrier()  # every partial has landed in its owner's slots
        rc = L.podecm_pod_gram_reduce(ctx.h, ctx.stream(), recv, world, rows, n_snap,
                                      C.c_void_p(gfull.value + row0[rank] * n_snap * 8))
        _lib.raise_for(rc, ctx.h, "podecm_pod_gram_reduce")
        torch.cuda.synchronize(S_local.device)
        dist.barrier()  # every owner's rows are reduced
        for o in range(world):
            if o != rank:
                off = row0[o] * n_snap * 8
                rc = L.podecm_peer_copy(ctx.h, ctx.stream(), C.c_void_p(gfull.value + off),
                                        C.c_void_p(g_all[o].value + off), (row0[o + 1] - row0[o]) * n_snap)
                _lib.raise_for(rc, ctx.h, "podecm_peer_copy")
        G = torch.empty((n_snap, n_snap), dtype=torch.float64, device=S_local.device)
        rc = L.podecm_peer_copy(ctx.h, ctx.stream(), _ptr(G), gfull, n_snap * n_snap)
        _lib.raise_for(rc, ctx.h, "podecm_peer_copy")
        torch.cuda.synchronize(S_local.device)
        dist.barrier()  # nobody reads a peer buffer any more
    finally:
        for o in range(world):
            if o != rank:
                L.podecm_ipc_close(recv_all[o])
                L.podecm_ipc_close(g_all[o])
        L.podecm_dev_free(recv)
        L.podecm_dev_free(gfull)
    return G


def pod_sharded(S_local: torch.Tensor, max_modes: int, tol_rel: float = 1e-10, ctx: Context | None = None,
                exchange: str = "peer"):
    """Row-sharded pod_diag: ``S_local`` [n_snap, n_local] holds
    this rank's contiguous dof rows of the snapshot matrix (same layout as
    pod()).  The summed Gram sum_k S_k^T S_k: ``exchange="peer"`` (default) by
    the GEMM fused with its reduce-scatter over peer memory (_gram_peer), or
    ``"collective"`` by a local Gram and one SUM all-reduce (NCCL, or gloo on a
    host copy).  Then the eigenproblem and S_k v / sqrt(lambda) on every rank,
    an all-gather of the mode rows and the MGS pass (podkit.cpp:75-86) on the
    whole basis.  Returns (modes^T [kept, n_dof], eigenvalues), the same on
    every rank."""
    import torch.distributed as dist
    ctx = ctx or Context.default(S_local.device.index or 0)
    n_snap, n_loc = S_local.shape
    dev = S_local.device
    world = dist.get_world_size() if dist.is_initialized() else 1
    if world > 1 and exchange == "peer":
        C_ = _gram_peer(ctx, S_local, n_snap, world, dist.get_rank())
    else:
        C_ = torch.empty((n_snap, n_snap), dtype=torch.float64, device=dev)
        rc = ctx.lib.podecm_pod_gram(ctx.h, ctx.stream(), _ptr(S_local), n_loc, n_snap, None, _ptr(C_))
        _lib.raise_for(rc, ctx.h, "podecm_pod_gram")
    if world > 1 and exchange != "peer":
        if "nccl" in str(dist.get_backend()):
            dist.all_reduce(C_)
        else:  # host backend (gloo): reduce a host copy
            h = C_.cpu()
            dist.all_reduce(h)
            C_.copy_(h)
    modes_l = torch.empty((max_modes, n_loc), dtype=torch.float64, device=dev)
    ev = torch.empty(n_snap, dtype=torch.float64, device=dev)
    kept = C.c_int()
    rc = ctx.lib.podecm_pod_modes_ex(ctx.h, ctx.stream(), _ptr(S_local), n_loc, n_snap, _ptr(C_), None, max_modes,
                                     tol_rel, _ptr(modes_l), _ptr(ev), C.byref(kept), 0)
    _lib.raise_for(rc, ctx.h, "podecm_pod_modes_ex")
    k = kept.value
    if world > 1:
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather_object(sizes, int(n_loc))
        mx = max(sizes)
        pad = torch.zeros((k, mx), dtype=torch.float64, device=dev)
        pad[:, :n_loc] = modes_l[:k]
        if "nccl" in str(dist.get_backend()):
            parts = [torch.empty_like(pad) for _ in range(world)]
            dist.all_gather(parts, pad)
        else:
            hp = pad.cpu()
            hparts = [torch.empty_like(hp) for _ in range(world)]
            dist.all_gather(hparts, hp)
            parts = [p.to(dev) for p in hparts]
        full = torch.cat([p[:, :n] for p, n in zip(parts, sizes)], dim=1).contiguous()
    else:
        full = modes_l[:k].contiguous()
    rc = ctx.lib.podecm_pod_mgs(ctx.h, ctx.stream(), _ptr(full), full.shape[1], k, None)
    _lib.raise_for(rc, ctx.h, "podecm_pod_mgs")
    return full, ev


@dataclass
class EcmOpts:
    """EcmOpts (ecm.hpp:28-32) + stop_at_count (configs 3/4 stop at a count)."""
    eps: float = 0.01
    volume_row: bool = True
    max_points: int = 0
    stop_at_count: bool = False

    def c(self) -> podecm_ecm_opts:
        return podecm_ecm_opts(self.eps, int(self.volume_row), self.max_points, int(self.stop_at_count))


def ecm_mode_grads(rve: Rve, modes_t: torch.Tensor) -> torch.Tensor:
    """H [n_qp, N, 4] from nodal modes given as modes^T [N, 2 n_nodes]."""
    N = modes_t.shape[0]
    H = torch.empty((rve.n_qp, N, 4), dtype=torch.float64, device=modes_t.device)
    rc = rve.lib.podecm_ecm_mode_grads(rve.ctx.h, rve.ctx.stream(), rve.h, _ptr(modes_t), N, _ptr(H))
    _lib.raise_for(rc, rve.ctx.h, "podecm_ecm_mode_grads")
    return H


def ecm_stress_snapshots(rve: Rve, U_t: torch.Tensor):
    """W [L, n_qp, 4] of snapshots U^T [L, 2 n_nodes]; returns (W, status)."""
    L = U_t.shape[0]
    W = torch.empty((L, rve.n_qp, 4), dtype=torch.float64, device=U_t.device)
    st = torch.zeros(1, dtype=torch.int32, device=U_t.device)
    rc = rve.lib.podecm_ecm_stress_snapshots(rve.ctx.h, rve.ctx.stream(), rve.h, _ptr(U_t), L, _ptr(W), _ptr(st))
    _lib.raise_for(rc, rve.ctx.h, "podecm_ecm_stress_snapshots")
    return W, st


def ecm_select(rve: Rve, H: torch.Tensor, W: torch.Tensor, opts: EcmOpts):
    """ecm_select (ecm.cpp:132-204) on the factored integrand.  Returns
    (ids ascending, weights, residual_rel, iterations)."""
    import numpy as np
    nq, N = H.shape[0], H.shape[1]
    L = W.shape[0]
    cap = opts.max_points if opts.max_points > 0 else nq
    ids = np.empty(cap, np.int32)
    w = np.empty(cap)
    n = C.c_int()
    rr = C.c_double()
    it = C.c_int()
    oc = opts.c()
    rc = rve.lib.podecm_ecm_select(rve.ctx.h, rve.ctx.stream(), rve.h, _ptr(H), N, _ptr(W), L, C.byref(oc),
                                   ids.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p),
                                   C.byref(n), C.byref(rr), C.byref(it))
    _lib.raise_for(rc, rve.ctx.h, "podecm_ecm_select")
    return ids[: n.value].copy(), w[: n.value].copy(), rr.value, it.value


def ecm_select_sharded(rve: Rve, H_local: torch.Tensor, W_local: torch.Tensor, q0: int, opts: EcmOpts):
    """The greedy of ecm_select over this rank's candidate shard [q0, q0 +
    nq_local) of the cell: H_local [nq_local, N, 4], W_local
    [L, nq_local, 4].  The exchanges (rhs all-reduce, per-iteration (score,
    index) argmax with the first-index rule, the selected column's
    broadcast) run over torch.distributed; the refit is replicated.  Returns
    ecm_select's tuple (global ids), the same on every rank."""
    import numpy as np
    from . import shard
    nql, N = H_local.shape[0], H_local.shape[1]
    L = W_local.shape[0]
    cap = opts.max_points if opts.max_points > 0 else rve.n_qp
    ids = np.empty(cap, np.int32)
    w = np.empty(cap)
    n = C.c_int()
    rr = C.c_double()
    it = C.c_int()
    oc = opts.c()
    comm = shard.ecm_comm(q0, nql)
    rc = rve.lib.podecm_ecm_select_sharded(rve.ctx.h, rve.ctx.stream(), rve.h, _ptr(H_local), N, _ptr(W_local), L,
                                           C.byref(comm), C.byref(oc), ids.ctypes.data_as(C.c_void_p),
                                           w.ctypes.data_as(C.c_void_p), C.byref(n), C.byref(rr), C.byref(it))
    _lib.raise_for(rc, rve.ctx.h, "podecm_ecm_select_sharded")
    return ids[: n.value].copy(), w[: n.value].copy(), rr.value, it.value


class RomEngines:
    """n RomMicroEngine instances (twoscale.hpp:55-80) on the device, one per
    macro Gauss point: respond() evaluates all of them for a batch of trial
    macro gradients from their committed histories, commit() accepts the
    trials.  geom [n, 2] (a, b); stretch_bounds [(lo, hi)] * 3 for
    (F00, F11, F01) or None."""

    def __init__(self, rom: Rom, geom: torch.Tensor, stretch_bounds=None):
        import numpy as np
        self.rom = rom
        self.ctx = rom.ctx
        self.lib = rom.lib
        self.n = geom.shape[0]
        _f64(geom, (self.n, 2), "geom")
        b = None
        if stretch_bounds is not None:
            b = np.ascontiguousarray(stretch_bounds, dtype=np.float64).reshape(6)
        h = C.c_void_p()
        rc = self.lib.podecm_rom_engines_create(self.ctx.h, rom.h, self.n, _ptr(geom),
                                                None if b is None else b.ctypes.data_as(C.c_void_p), C.byref(h))
        _lib.raise_for(rc, self.ctx.h, "podecm_rom_engines_create")
        self.h = h

    def respond(self, fbar: torch.Tensor, opts: NewtonOpts | None = None, abar: bool = False) -> dict:
        """MicroEngine::respond for every engine: pbar [n, 4], abar [n, 16]
        (Tensor4 storage r + 4c) if requested, iters [n], status [n]."""
        opts = opts or NewtonOpts()
        _f64(fbar, (self.n, 4), "fbar")
        dev = fbar.device
        pbar = torch.zeros((self.n, 4), dtype=torch.float64, device=dev)
        ab = torch.zeros((self.n, 16), dtype=torch.float64, device=dev) if abar else None
        iters = torch.zeros(self.n, dtype=torch.int32, device=dev)
        status = torch.empty(self.n, dtype=torch.int32, device=dev)
        oc = opts.c()
        rc = self.lib.podecm_rom_engines_respond(self.ctx.h, self.ctx.stream(), self.h, _ptr(fbar), C.byref(oc),
                                                 _ptr(pbar), _ptr(ab), _ptr(iters), _ptr(status))
        _lib.raise_for(rc, self.ctx.h, "podecm_rom_engines_respond")
        out = {"pbar": pbar, "iters": iters, "status": status}
        if abar:
            out["abar"] = ab
        return out

    def commit(self) -> None:
        _lib.raise_for(self.lib.podecm_rom_engines_commit(self.ctx.h, self.ctx.stream(), self.h), self.ctx.h,
                       "podecm_rom_engines_commit")

    def out_of_range(self) -> torch.Tensor:
        out = torch.empty(self.n, dtype=torch.int32, device="cuda")
        _lib.raise_for(self.lib.podecm_rom_engines_out_of_range(self.ctx.h, self.ctx.stream(), self.h, _ptr(out)),
                       self.ctx.h, "podecm_rom_engines_out_of_range")
        return out

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.podecm_rom_engines_destroy(self.h)
                self.h = None
        except Exception:
            pass


class FullOrder:
    """Full-order solve_rve (microfem.cpp:142-238) on the GPU for a batch of
    instances of one Rve: batched assembly + batched sparse LU refactorisation."""

    def __init__(self, rve: Rve):
        self.rve = rve
        self.ctx = rve.ctx
        self.lib = rve.lib
        h = C.c_void_p()
        _lib.raise_for(self.lib.podecm_fe_create(self.ctx.h, rve.h, C.byref(h)), self.ctx.h, "podecm_fe_create")
        self.h = h

    def solve(self, geom: torch.Tensor, sched: torch.Tensor, opts: NewtonOpts | None = None,
              history: bool = False) -> dict:
        """pbar [n, K, 4], iters [n, K], resid [n, K], w_final [n, n_red], status [n];
        history=True adds w_hist [n, K, n_red] and p_hist [n, K, 4, n_qp]."""
        opts = opts or NewtonOpts()
        n, K = sched.shape[0], sched.shape[1]
        dev = sched.device
        _f64(geom, (n, 2), "geom")
        _f64(sched, (n, K, 4), "sched")
        z = lambda shape, dt=torch.float64: torch.zeros(shape, dtype=dt, device=dev)
        pbar, iters, resid = z((n, K, 4)), z((n, K), torch.int32), z((n, K))
        wf, status = z((n, self.rve.n_red)), z(n, torch.int32)
        wh = z((n, K, self.rve.n_red)) if history else None
        ph = z((n, K, 4, self.rve.n_qp)) if history else None
        oc = opts.c()
        rc = self.lib.podecm_fe_solve_batch_ex(self.ctx.h, self.ctx.stream(), self.h, n, _ptr(geom), _ptr(sched), K,
                                               C.byref(oc), _ptr(pbar), _ptr(iters), _ptr(resid), _ptr(wf),
                                               _ptr(status), _ptr(wh), _ptr(ph))
        _lib.raise_for(rc, self.ctx.h, "podecm_fe_solve_batch")
        self.global_iterations = int(self.lib.podecm_fe_global_iterations(self.h))
        out = {"pbar": pbar, "iters": iters, "resid": resid, "w_final": wf, "status": status}
        if history:
            out.update(w_hist=wh, p_hist=ph)
        return out

    def collect_snapshots(self, geom: torch.Tensor, sched: torch.Tensor, opts: NewtonOpts | None = None) -> dict:
        """collect_snapshots (pipeline.cpp:157-188) for the training samples
        geom [S, 2] with schedules sched [S, K, 4]: disp [2 n_nodes, S K]
        (expanded fluctuations, sample-major columns), stress [4 n_qp, S K]
        (weighted_stress_field, column entries q*4 + c), newton_iters [S K],
        steps_per_sample [S].  A failed sample raises SolveError like the
        reference."""
        r = self.solve(geom, sched, opts, history=True)
        if int((r["status"] != 0).sum().item()):
            bad = int(torch.nonzero(r["status"] != 0)[0].item())
            raise SolveError(f"training sample {bad}: cell Newton did not converge")
        S, K = sched.shape[0], sched.shape[1]
        rv = self.rve
        nd = torch.as_tensor(rv.export()["node_dof"], device=geom.device, dtype=torch.int64)
        w = r["w_hist"].reshape(S * K, rv.n_red)
        disp = torch.zeros((S * K, rv.n_nodes, 2), dtype=torch.float64, device=geom.device)
        m = nd >= 0  # DofMap::expand (mesh.cpp:390-400): the anchor stays zero
        disp[:, m, 0] = w[:, nd[m]]
        disp[:, m, 1] = w[:, nd[m] + 1]
        geom_k = geom.repeat_interleave(K, dim=0).contiguous()
        W = torch.empty((S * K, rv.n_qp, 4), dtype=torch.float64, device=geom.device)
        pf = r["p_hist"].reshape(S * K, 4, rv.n_qp).contiguous()
        rc = self.lib.podecm_weighted_stress_field(self.ctx.h, self.ctx.stream(), rv.h, S * K, _ptr(geom_k),
                                                   _ptr(pf), _ptr(W))
        _lib.raise_for(rc, self.ctx.h, "podecm_weighted_stress_field")
        return {"disp": disp.reshape(S * K, 2 * rv.n_nodes).T, "stress": W.reshape(S * K, 4 * rv.n_qp).T,
                "newton_iters": r["iters"].reshape(-1), "steps_per_sample": torch.full((S,), K, dtype=torch.int64)}

    def effective_stiffness(self, geom: torch.Tensor, st0: torch.Tensor, fbar: torch.Tensor,
                            w: torch.Tensor) -> dict:
        """effective_stiffness (microfem.cpp:240-313): history st0 [n, 6, n_qp],
        fbar [n, 4], fluctuation w [n, n_red] -> abar [n, 16] (Tensor4 storage
        r + 4c), status [n]."""
        n = geom.shape[0]
        _f64(geom, (n, 2), "geom")
        _f64(st0, (n, 6, self.rve.n_qp), "st0")
        _f64(fbar, (n, 4), "fbar")
        _f64(w, (n, self.rve.n_red), "w")
        abar = torch.zeros((n, 16), dtype=torch.float64, device=geom.device)
        status = torch.zeros(n, dtype=torch.int32, device=geom.device)
        rc = self.lib.podecm_fe_effective_stiffness_batch(self.ctx.h, self.ctx.stream(), self.h, n, _ptr(geom),
                                                          _ptr(st0), _ptr(fbar), _ptr(w), _ptr(abar), _ptr(status))
        _lib.raise_for(rc, self.ctx.h, "podecm_fe_effective_stiffness_batch")
        return {"abar": abar, "status": status}

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.podecm_fe_destroy(self.h)
                self.h = None
        except Exception:
            pass


# ---- FE2 macro driver -------------------------------------
@dataclass
class MacroConfig:
    """MacroConfig (twoscale.hpp:82-94): nx x ny Quad8 plate, bottom clamped,
    parabolic top traction ramped up to peak over steps/2 and back."""
    nx: int = 5
    ny: int = 3
    width: float = 2.0
    height: float = 1.0
    peak_traction: float = 0.2
    steps: int = 50
    newton: NewtonOpts | None = None

    def c(self) -> _lib.podecm_macro_cfg:
        nw = (self.newton or NewtonOpts()).c()
        return _lib.podecm_macro_cfg(self.nx, self.ny, self.width, self.height, self.peak_traction, self.steps, nw)

    def info(self) -> dict:
        out = (C.c_int64 * 4)()
        cc = self.c()
        _lib.raise_for(_lib.load().podecm_macro_info(C.byref(cc), out), None, "podecm_macro_info")
        return dict(zip(("n_nodes", "n_elems", "n_qp", "n_red"), (int(v) for v in out)))

    def qp_positions(self):
        import numpy as np
        x = np.empty((self.info()["n_qp"], 2))
        cc = self.c()
        _lib.raise_for(_lib.load().podecm_macro_qp_positions(C.byref(cc), x.ctypes.data_as(C.c_void_p)), None,
                       "podecm_macro_qp_positions")
        return x


def run_twoscale(cfg: MacroConfig, engines: "RomEngines | None" = None, micro_opts: NewtonOpts | None = None,
                 E: float = 1.0, nu: float = 0.3, ctx: Context | None = None) -> dict:
    """run_twoscale (twoscale.cpp:131-242) with the batched ROM engines of the
    macro Gauss points, or LinearElasticEngine(E, nu) when engines is None.
    Returns load_factor, compliance, iters [steps], u_final [2 n_nodes],
    residual_norm, micro_evals."""
    import numpy as np
    ctx = engines.ctx if engines is not None else (ctx or Context.default())
    inf = cfg.info()
    lf, comp = np.zeros(cfg.steps), np.zeros(cfg.steps)
    it = np.zeros(cfg.steps, np.int32)
    uf = np.zeros(2 * inf["n_nodes"])
    rn, ev = C.c_double(), C.c_int64()
    cc = cfg.c()
    mo = (micro_opts or NewtonOpts()).c()
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    rc = ctx.lib.podecm_twoscale_run(ctx.h, ctx.stream(), C.byref(cc), engines.h if engines is not None else None,
                                     C.byref(mo), E, nu, p(lf), p(comp), p(it), p(uf), C.byref(rn), C.byref(ev))
    _lib.raise_for(rc, ctx.h, "podecm_twoscale_run")
    return {"load_factor": lf, "compliance": comp, "iters": it, "u_final": uf, "residual_norm": rn.value,
            "micro_evals": ev.value}


# ---- interchange formats --------------------------------
FNV_SEED = 14695981039346656037


def rom_model_save(path, model: dict) -> None:
    """RomModel::save (rom.cpp:265-289) into a PODECM1 container.  ``model``:
    modes [n_dof, N] (numpy), ids [Q], weights [Q], mode_grads [Q, N, 4],
    optional mesh_tag, kind, n_stress_modes, ecm_eps."""
    import numpy as np
    lib = _lib.load()
    modes = np.asfortranarray(model["modes"], dtype=np.float64)
    ids = np.ascontiguousarray(model["ids"], dtype=np.int32)
    w = np.ascontiguousarray(model["weights"], dtype=np.float64)
    mg = np.ascontiguousarray(model["mode_grads"], dtype=np.float64)
    n_dof, N = modes.shape
    Q = ids.shape[0]
    if mg.shape != (Q, N, 4) or w.shape != (Q,):
        raise ConfigError("rom_model_save: inconsistent ids/weights/mode_grads shapes")
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    rc = lib.podecm_rom_model_save(str(path).encode(), int(model.get("mesh_tag", 0)), int(model.get("kind", 0)),
                                   int(model.get("n_stress_modes", 0)), float(model.get("ecm_eps", 0.0)), n_dof, N,
                                   p(modes), Q, p(ids), p(w), p(mg))
    _lib.raise_for(rc, None, "rom_model_save")


def rom_model_load(path) -> dict:
    """RomModel::load (rom.cpp:291-327): the arrays of rom_model_save plus
    mesh_tag, kind, n_stress_modes, ecm_eps.  Raises IoError / FormatError
    like the reference."""
    import numpy as np
    lib = _lib.load()
    n_dof, N, Q = C.c_int64(), C.c_int32(), C.c_int32()
    tag, kind, nsm, eps = C.c_uint64(), C.c_int32(), C.c_int32(), C.c_double()
    rc = lib.podecm_rom_model_info(str(path).encode(), C.byref(n_dof), C.byref(N), C.byref(Q), C.byref(tag),
                                   C.byref(kind), C.byref(nsm), C.byref(eps))
    _lib.raise_for(rc, None, "rom_model_load")
    modes = np.empty((N.value, n_dof.value))  # column-major image
    ids = np.empty(Q.value, np.int32)
    w = np.empty(Q.value)
    mg = np.empty((Q.value, N.value, 4))
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    rc = lib.podecm_rom_model_read(str(path).encode(), p(modes), p(ids), p(w), p(mg))
    _lib.raise_for(rc, None, "rom_model_load")
    return {"modes": modes.T, "ids": ids, "weights": w, "mode_grads": mg, "mesh_tag": tag.value,
            "kind": kind.value, "n_stress_modes": nsm.value, "ecm_eps": eps.value}


def fnv1a64(data: bytes, seed: int = FNV_SEED) -> int:
    """FNV-1a 64 (store.hpp:52-54) as the library computes it."""
    buf = C.create_string_buffer(bytes(data), len(data))
    return int(_lib.load().podecm_fnv1a64(buf, len(data), seed))
