"""ctypes binding of the C-ABI in include/podecm_cuda.h.

The product path has exactly one implementation: the sm_100a kernels in
``libpodecm_cuda.so``.  There is no CPU fallback — if the library is missing
or no CUDA device is present, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libpodecm_cuda.so"

_lib = None

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
D = C.c_double


class podecm_params(C.Structure):
    _fields_ = [("E", D), ("nu", D), ("sigma_y0", D), ("H", D)]


class podecm_ecm_opts(C.Structure):
    _fields_ = [("eps", D), ("volume_row", I32), ("max_points", I32), ("stop_at_count", I32)]


ECM_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), I64)
ECM_ARGMAX = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(I64), C.POINTER(C.c_int))
ECM_BCAST = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), I64, C.c_int)


class podecm_ecm_comm(C.Structure):
    _fields_ = [("user", C.c_void_p), ("q0", I64), ("nq_local", I64), ("allreduce_sum", ECM_ALLREDUCE),
                ("argmax", ECM_ARGMAX), ("bcast", ECM_BCAST)]


class podecm_newton(C.Structure):
    _fields_ = [("eps_rel", D), ("eps_abs", D), ("force_ref", D), ("max_iter", I32),
                ("max_bisect", I32)]


class podecm_macro_cfg(C.Structure):
    _fields_ = [("nx", I32), ("ny", I32), ("width", D), ("height", D), ("peak_traction", D), ("steps", I32),
                ("newton", podecm_newton)]


_SIGS = {
    "podecm_ctx_create": (C.c_int, [C.c_int, C.POINTER(P)]),
    "podecm_ctx_destroy": (None, [P]),
    "podecm_last_error": (C.c_char_p, [P]),
    "podecm_check": (C.c_int, [P, P]),
    "podecm_launch_count": (I64, [P]),
    "podecm_set_timing": (None, [P, C.c_int]),
    "podecm_get_timings": (C.c_int, [P, C.c_char_p, C.c_int, P, P, C.c_int]),
    "podecm_material_batch": (C.c_int, [P, P, I64, C.POINTER(podecm_params), C.c_int, P, P, P, P,
                                        P, P, P, D]),
    "podecm_material_batch_ex": (C.c_int, [P, P, I64, C.POINTER(podecm_params), C.c_int, P, P, P, P,
                                           P, P, P, D, P]),
    "podecm_rve_create_q4": (C.c_int, [P, C.c_int, D, C.POINTER(podecm_params), C.c_int,
                                       C.POINTER(P)]),
    "podecm_rve_create_q4_regions": (C.c_int, [P, C.c_int, D, P, C.POINTER(podecm_params), C.c_int,
                                               C.POINTER(P)]),
    "podecm_rve_destroy": (None, [P]),
    "podecm_rve_info": (C.c_int, [P, C.POINTER(I64)]),
    "podecm_rve_export": (C.c_int, [P, P, P, P, P, P, P, P, P, P, P]),
    "podecm_rve_n_triplets": (I64, [P]),
    "podecm_rve_morph": (C.c_int, [P, P, P, I64, P, P, P, P]),
    "podecm_assemble_batch": (C.c_int, [P, P, P, I64, P, P, P, P, P, P, P, P, P, P]),
    "podecm_rom_create": (C.c_int, [P, P, C.c_int, C.c_int, P, P, P, C.POINTER(P)]),
    "podecm_rom_destroy": (None, [P]),
    "podecm_rom_global_iterations": (I64, [P]),
    "podecm_pod_gram": (C.c_int, [P, P, P, I64, C.c_int, P, P]),
    "podecm_pod_modes": (C.c_int, [P, P, P, I64, C.c_int, P, P, C.c_int, D, P, P, C.POINTER(C.c_int)]),
    "podecm_pod_modes_ex": (C.c_int, [P, P, P, I64, C.c_int, P, P, C.c_int, D, P, P, C.POINTER(C.c_int),
                                       C.c_int]),
    "podecm_pod_mgs": (C.c_int, [P, P, P, I64, C.c_int, P]),
    "podecm_pod_gram_peer": (C.c_int, [P, P, P, I64, C.c_int, P, P, C.c_int, C.c_int, P]),
    "podecm_pod_gram_reduce": (C.c_int, [P, P, P, C.c_int, I64, C.c_int, P]),
    "podecm_peer_copy": (C.c_int, [P, P, P, P, I64]),
    "podecm_dev_alloc": (C.c_int, [P, I64, C.POINTER(P)]),
    "podecm_dev_free": (None, [P]),
    "podecm_ipc_handle": (C.c_int, [P, P, P]),
    "podecm_ipc_open": (C.c_int, [P, P, C.POINTER(P)]),
    "podecm_ipc_close": (None, [P]),
    "podecm_ecm_select_sharded": (C.c_int, [P, P, P, P, C.c_int, P, I64, P, C.POINTER(podecm_ecm_opts), P, P,
                                            C.POINTER(C.c_int), C.POINTER(D), C.POINTER(C.c_int)]),
    "podecm_ecm_mode_grads": (C.c_int, [P, P, P, P, C.c_int, P]),
    "podecm_ecm_stress_snapshots": (C.c_int, [P, P, P, P, I64, P, P]),
    "podecm_ecm_select": (C.c_int, [P, P, P, P, C.c_int, P, I64, C.POINTER(podecm_ecm_opts), P, P,
                                    C.POINTER(C.c_int), C.POINTER(D), C.POINTER(C.c_int)]),
    "podecm_probe_fp64": (C.c_int, [P, P, C.c_int, C.c_int, P, C.POINTER(D)]),
    "podecm_probe_math": (C.c_int, [P, P, C.c_int, I64, P, P, P]),
    "podecm_rom_solve_batch": (C.c_int, [P, P, P, I64, P, P, C.c_int, C.POINTER(podecm_newton),
                                         P, P, P, P, P]),
    "podecm_rom_solve_batch_ex": (C.c_int, [P, P, P, I64, P, P, C.c_int, C.POINTER(podecm_newton),
                                            P, P, P, P, P, P]),
    "podecm_rom_solve_batch_morph": (C.c_int, [P, P, P, I64, P, P, C.c_int, C.POINTER(podecm_newton),
                                               P, P, P, P, P, P, P]),
    "podecm_rom_effective_stiffness_batch": (C.c_int, [P, P, P, I64, P, P, P, P, P, P]),
    "podecm_rom_sensitivity_batch": (C.c_int, [P, P, P, I64, P, P, C.c_int, C.POINTER(podecm_newton),
                                               D, P, P]),
    "podecm_rom_engines_create": (C.c_int, [P, P, I64, P, P, C.POINTER(P)]),
    "podecm_rom_engines_destroy": (None, [P]),
    "podecm_rom_engines_respond": (C.c_int, [P, P, P, P, C.POINTER(podecm_newton), P, P, P, P]),
    "podecm_rom_engines_commit": (C.c_int, [P, P, P]),
    "podecm_rom_engines_out_of_range": (C.c_int, [P, P, P, P]),
    "podecm_assemble_batch_ex": (C.c_int, [P, P, P, I64, P, P, P, P, P, P, P, P, P, P, P]),
    "podecm_fe_solve_batch_ex": (C.c_int, [P, P, P, I64, P, P, C.c_int, C.POINTER(podecm_newton), P, P, P, P, P,
                                           P, P]),
    "podecm_weighted_stress_field": (C.c_int, [P, P, P, I64, P, P, P]),
    "podecm_fe_effective_stiffness_batch": (C.c_int, [P, P, P, I64, P, P, P, P, P, P]),
    "podecm_fe_create": (C.c_int, [P, P, C.POINTER(P)]),
    "podecm_fe_destroy": (None, [P]),
    "podecm_fe_global_iterations": (I64, [P]),
    "podecm_fe_solve_batch": (C.c_int, [P, P, P, I64, P, P, C.c_int, C.POINTER(podecm_newton), P, P, P, P, P]),
    "podecm_macro_info": (C.c_int, [C.POINTER(podecm_macro_cfg), C.POINTER(I64)]),
    "podecm_macro_qp_positions": (C.c_int, [C.POINTER(podecm_macro_cfg), P]),
    "podecm_twoscale_run": (C.c_int, [P, P, C.POINTER(podecm_macro_cfg), P, C.POINTER(podecm_newton), D, D, P, P,
                                      P, P, C.POINTER(D), C.POINTER(I64)]),
    "podecm_store_last_error": (C.c_char_p, []),
    "podecm_fnv1a64": (C.c_uint64, [P, C.c_uint64, C.c_uint64]),
    "podecm_rve_fingerprint": (C.c_uint64, [P]),
    "podecm_rom_model_save": (C.c_int, [C.c_char_p, C.c_uint64, I32, I32, D, I64, I32, P, I32, P, P, P]),
    "podecm_rom_model_info": (C.c_int, [C.c_char_p, C.POINTER(I64), C.POINTER(I32), C.POINTER(I32),
                                        C.POINTER(C.c_uint64), C.POINTER(I32), C.POINTER(I32), C.POINTER(D)]),
    "podecm_rom_model_read": (C.c_int, [C.c_char_p, P, P, P, P]),
}

# every symbol include/podecm_cuda.h declares (checked by tests on CPU)
EXPORTED = tuple(_SIGS)


class PodecmError(RuntimeError):
    pass


class ConfigError(PodecmError):
    """Reference ConfigError (types.hpp:60-63); C-ABI code 2."""


class SolveError(PodecmError):
    """Reference SolveError (types.hpp:65-68); C-ABI code 3."""


class CudaError(PodecmError):
    """C-ABI code 4."""


class IoError(PodecmError):
    """Reference IoError (types.hpp:50-53); C-ABI code 5."""


class FormatError(PodecmError):
    """Reference FormatError (types.hpp:55-58); C-ABI code 6."""


def load(path: Path | str | None = None):
    """Load the library (without touching the GPU) and bind every signature."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise PodecmError(f"{p} is missing: run `python -m paper_2307_16894_b200._build` "
                          "(the CUDA path has no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def raise_for(rc: int, ctx=None, what: str = "") -> None:
    if rc == 0:
        return
    msg = what
    if ctx:
        m = load().podecm_last_error(ctx)
        msg = f"{what}: {m.decode() if m else ''}"
    if rc == 2:
        raise ConfigError(msg)
    if rc == 3:
        raise SolveError(msg)
    if rc == 4:
        raise CudaError(msg)
    if rc in (5, 6):
        m = load().podecm_store_last_error()
        msg = f"{what}: {m.decode() if m else ''}"
        raise (IoError if rc == 5 else FormatError)(msg)
    raise PodecmError(f"{msg} (code {rc})")
