"""ctypes loader and signatures for libtopt.so (the C ABI in include/topt.h).

Argument marshalling only: every step of the hot path runs in the library's CUDA
kernels.  There is no fallback: if the shared library is missing or fails to
load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# TOPT_LIB selects another build of the same ABI (tests: lib/libtopt_stress.so, the race-stress /
# bounds-checked build); the default is the release library
LIB_PATH = os.environ.get("TOPT_LIB") or os.path.join(HERE, "lib", "libtopt.so")

NSCALARS = 16
S_OBJ, S_DIST, S_REG, S_GRAD_INF, S_GS, S_SLV, S_SLS = range(7)
OK = 0
STATUS = {0: "OK", -1: "INVALID_ARG", -2: "UNSUPPORTED", -3: "CUDA", -4: "NCCL", -5: "WORKSPACE",
          -6: "HALO"}


class Params(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_int32),
        ("n", ctypes.c_int32 * 3),
        ("nt", ctypes.c_int32),
        ("model", ctypes.c_int32),
        ("reg_order", ctypes.c_int32),
        ("alpha", ctypes.c_double),
        ("window", ctypes.c_int32),
        ("sigma", ctypes.c_int32),
        ("tau", ctypes.c_int32),
        ("method", ctypes.c_int32),
        ("ordering", ctypes.c_int32),
        ("max_iter", ctypes.c_int32),
        ("eps_rel", ctypes.c_double),
        ("armijo_c", ctypes.c_double),
        ("max_backtracks", ctypes.c_int32),
    ]


class Report(ctypes.Structure):
    _fields_ = [
        ("obj", ctypes.c_double), ("dist", ctypes.c_double), ("reg", ctypes.c_double),
        ("grad_inf", ctypes.c_double), ("grad_inf0", ctypes.c_double), ("rho", ctypes.c_double),
        ("iters", ctypes.c_int32), ("grad_evals", ctypes.c_int32), ("obj_evals", ctypes.c_int32),
        ("pde_solves", ctypes.c_int32), ("exit", ctypes.c_int32), ("ngmres_steps", ctypes.c_int32),
        ("t_total", ctypes.c_double), ("t_pde", ctypes.c_double), ("t_ls", ctypes.c_double),
        ("t_q", ctypes.c_double), ("t_f", ctypes.c_double), ("dist0", ctypes.c_double),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


# name -> (restype, argtypes); mirrors include/topt.h
_P = ctypes.c_void_p
_I = ctypes.c_int32
SIGNATURES = {
    "topt_abi_version": (ctypes.c_int32, []),
    "topt_last_error": (ctypes.c_char_p, []),
    "topt_get_unique_id": (_I, [ctypes.c_void_p]),
    "topt_create": (_I, [ctypes.POINTER(Params), _I, _I, _P, _I, ctypes.POINTER(_P)]),
    "topt_destroy": (_I, [_P]),
    "topt_workspace_size": (_I, [_P, ctypes.POINTER(ctypes.c_size_t)]),
    "topt_bind_workspace": (_I, [_P, _P, ctypes.c_size_t]),
    "topt_local_slab": (_I, [_P, ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    "topt_set_transport": (_I, [_P, _I]),
    "topt_get_transport": (_I, [_P]),
    "topt_linear_ngmres": (_I, [_P, _P, ctypes.c_double, _P, _I, ctypes.POINTER(ctypes.c_double), _P]),
    "topt_set_peer_workspaces": (_I, [_P, ctypes.POINTER(_P), _I]),
    "topt_solve": (_I, [_P, _P, _P, _P, ctypes.POINTER(Report), _P]),
    "topt_set_step_replay": (_I, [_P, ctypes.POINTER(ctypes.c_double), _I]),
    "topt_eval_gradient": (_I, [_P, _P, _P, _P, _P, _P, _P, _P]),
    "topt_eval_gradient_host": (_I, [_P, _P, _P, _P, _P, _P, _P]),
    "topt_eval_gradient_host_async": (_I, [_P, _P, _P, _P, _P, _P, _P]),
    "topt_flow_map": (_I, [_P, _P, _P, _P, _P]),
    "topt_objective": (_I, [_P, _P, _P, _P, _P, _P]),
    "topt_feet": (_I, [_P, _P, _P, _P, _P]),
    "topt_forward": (_I, [_P, _P, _P, _P, _P]),
    "topt_get_adjoint": (_I, [_P, _P, _P, _P]),
    "topt_derivative": (_I, [_P, _P, _I, _P, _P]),
    "topt_apply_precond": (_I, [_P, _P, _P, _P]),
    "topt_leray": (_I, [_P, _P, _P, _P]),
    "topt_multidot": (_I, [_P, _P, ctypes.POINTER(_P), _I, _P, _P]),
    "topt_mix": (_I, [_P, _P, ctypes.POINTER(_P), ctypes.POINTER(ctypes.c_double), _I, _P, _P]),
    "topt_profile": (_I, [_P, _I]),
    "topt_set_graphs": (_I, [_P, _I]),
    "topt_kernel_stats": (_I, [_P, _I, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_double),
                               ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]),
    "topt_launch_count": (ctypes.c_int64, []),
}


class ToptError(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    if not os.path.exists(path):
        raise ImportError(
            f"libtopt.so not found at {path}; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = load()


def check(status: int, what: str = ""):
    if status != OK:
        msg = LIB.topt_last_error().decode(errors="replace")
        raise ToptError(f"{what}: {STATUS.get(status, status)}: {msg}")
