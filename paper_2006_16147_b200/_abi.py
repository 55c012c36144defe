"""ctypes binding of include/amg_b200.h — argument marshalling only.

Every step of the solve path runs in libamg_b200.so (sm_100a kernels + the C++
setup).  There is no Python or CPU fallback: if the library is missing this
module raises at import time.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AMG_LIB_PATH") or os.path.join(_HERE, "libamg_b200.so")  # override: experiments

AMG_OK, AMG_ERR_ARG, AMG_ERR_NOT_SPD, AMG_ERR_CUDA, AMG_ERR_NCCL, AMG_ERR_OOM = 0, 1, 2, 3, 4, 5
AMG_NOT_CONVERGED, AMG_ERR_BREAKDOWN = 6, 7
FORMATS = {0: "sell32", 1: "csr_vector", 2: "dense_inverse", 3: "sdia32", 4: "sell32_sigma"}


class amg_config_t(C.Structure):
    _fields_ = [("sweeps_per_level", C.c_int32), ("smooth_prolongator", C.c_int32),
                ("prol_omega_scale", C.c_double), ("max_coarse_size", C.c_int64),
                ("max_levels", C.c_int32), ("min_coarsening_ratio", C.c_double),
                ("pre_sweeps", C.c_int32), ("post_sweeps", C.c_int32),
                ("replicate_below_bytes", C.c_int64), ("setup_threads", C.c_int32),
                ("use_graphs", C.c_int32), ("emulate_ranks", C.c_int32),
                ("krylov", C.c_int32), ("coarse_solver", C.c_int32), ("coarse_maxit", C.c_int32),
                ("coarse_rtol", C.c_double), ("cycle", C.c_int32), ("setup_device", C.c_int32),
                ("tail_rows", C.c_int64), ("smoother", C.c_int32), ("invk_fill", C.c_int32),
                ("tail_bytes", C.c_int64), ("invk_l1", C.c_int32), ("invk_blocks", C.c_int32),
                ("invk_dense_cut", C.c_int32), ("coarse_prec", C.c_int32), ("setup_distributed", C.c_int32)]


class amg_report_t(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("nlevels", C.c_int32),
                ("status", C.c_int32), ("final_relres", C.c_double), ("setup_s", C.c_double),
                ("solve_s", C.c_double), ("opc", C.c_double), ("avg_cr", C.c_double),
                ("vcycle_bytes_model", C.c_double), ("iteration_bytes_model", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                      f"g.build()'` (no CPU fallback exists)")

lib = C.CDLL(LIB_PATH)
_vp = C.c_void_p
_i64p = C.POINTER(C.c_int64)
_SIG = {
    "amg_config_default": (None, [C.POINTER(amg_config_t)]),
    "amg_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, _vp, C.POINTER(_vp)]),
    "amg_ctx_destroy": (C.c_int, [_vp]),
    "amg_hierarchy_build": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, _vp, _vp, _vp, _vp,
                                      C.POINTER(amg_config_t), C.POINTER(_vp)]),
    "amg_hierarchy_destroy": (C.c_int, [_vp]),
    "amg_solve": (C.c_int, [_vp, _vp, _vp, C.c_double, C.c_int32, C.POINTER(amg_report_t)]),
    "amg_solve_host": (C.c_int, [_vp, _vp, _vp, C.c_double, C.c_int32, C.POINTER(amg_report_t)]),
    "amg_solve_host_batch": (C.c_int, [_vp, C.c_int32, _vp, _vp, C.c_double, C.c_int32, _vp]),
    "amg_precond_apply": (C.c_int, [_vp, _vp, _vp]),
    "amg_num_levels": (C.c_int, [_vp, C.POINTER(C.c_int32)]),
    "amg_solve_graph_mode": (C.c_int, [_vp, C.POINTER(C.c_int32)]),
    "amg_comm_transport": (C.c_int, [_vp, C.POINTER(C.c_int32)]),
    "amg_level_info": (C.c_int, [_vp, C.c_int32, _i64p, _i64p, _i64p, _i64p, _i64p,
                                 C.POINTER(C.c_int32)]),
    "amg_level_aggregates": (C.c_int, [_vp, C.c_int32, _vp]),
    "amg_hierarchy_report": (C.c_int, [_vp, C.POINTER(amg_report_t)]),
    "amg_profile_vcycle": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, _vp, _vp, _vp,
                                     C.POINTER(C.c_int32)]),
    "amg_profile_iteration": (C.c_int, [_vp, _vp, _vp, C.c_int32, C.c_int32, _vp, _vp, _vp, _vp,
                                        C.POINTER(C.c_int32)]),
    "amg_last_error": (C.c_char_p, []),
    "amg_nccl_unique_id": (C.c_int, [_vp]),
    "amg_host_hierarchy_build": (C.c_int, [C.c_int64, _vp, _vp, _vp, _vp, C.POINTER(amg_config_t),
                                           C.POINTER(_vp)]),
    "amg_host_hierarchy_destroy": (C.c_int, [_vp]),
    "amg_host_num_levels": (C.c_int, [_vp, C.POINTER(C.c_int32)]),
    "amg_host_level_sizes": (C.c_int, [_vp, C.c_int32, _i64p, _i64p, _i64p, C.POINTER(C.c_double)]),
    "amg_host_level_aggregates": (C.c_int, [_vp, C.c_int32, _vp]),
    "amg_host_level_matrix": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, _vp, _vp]),
    "amg_host_partition": (C.c_int, [_vp, C.c_int32, _vp, C.c_int64]),
    "amg_host_dist_build": (C.c_int, [C.c_int64, _vp, _vp, _vp, _vp, C.POINTER(amg_config_t), C.c_int32,
                                      C.c_int64, C.POINTER(_vp)]),
    "amg_host_dist_build_rank": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, _vp, _vp, _vp, _vp,
                                           C.POINTER(amg_config_t), C.c_int32, C.c_int32, C.c_int64,
                                           _vp, _vp, C.POINTER(_vp)]),
    "amg_host_plan_level": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp]),
    "amg_host_plan_array": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, _vp]),
}
for _name, (_res, _args) in _SIG.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIG)

# amg_exchange_fn (include/amg_b200.h): the distributed setup's transport callback
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                          C.c_void_p, C.c_void_p)


class AmgError(RuntimeError):
    def __init__(self, code, where):
        msg = lib.amg_last_error().decode(errors="replace")
        super().__init__(f"{where} failed with status {code}: {msg}")
        self.code = code


def check(code, where, ok=(AMG_OK,)):
    if code not in ok:
        raise AmgError(code, where)
    return code


# thin same-name wrappers -------------------------------------------------------
def amg_config_default() -> amg_config_t:
    c = amg_config_t()
    lib.amg_config_default(C.byref(c))
    return c


def amg_last_error() -> str:
    return lib.amg_last_error().decode(errors="replace")


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib.amg_nccl_unique_id(buf), "amg_nccl_unique_id")
    return buf.raw
