"""B200-native AMG-PCG solve path of arxiv 2006.16147 (AMG4PSBLAS).

Public API (same names as the C ABI in include/amg_b200.h):

    ctx = Context(device=0)
    h = Hierarchy(ctx, A, cfg=None, w=None)       # amg_hierarchy_build
    x, rep = h.solve(b, rtol=1e-6, maxit=500)     # amg_solve (torch CUDA tensors)
    x, rep = h.solve_host(b_np)                   # amg_solve_host (host buffers)
    z = h.precond_apply(r)                        # amg_precond_apply (one V-cycle)
    h.level_aggregates(l), h.level_info(l), h.report(), h.profile_vcycle(n)

Everything runs in libamg_b200.so; this package only marshals arguments.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from ._abi import (AMG_ERR_BREAKDOWN, AMG_NOT_CONVERGED, AMG_OK, AmgError, amg_config_default,  # noqa: F401
                   amg_config_t, amg_last_error, amg_report_t, check, lib, nccl_unique_id)

__all__ = ["Context", "Hierarchy", "amg_config_default", "AmgError", "lib"]


def make_config(**kw) -> amg_config_t:
    c = amg_config_default()
    for k, v in kw.items():
        if not hasattr(c, k):
            raise KeyError(k)
        setattr(c, k, v)
    return c


class Context:
    """amg_ctx_create / amg_ctx_destroy.  stream=None lets the library own a stream."""

    def __init__(self, device: int = 0, rank: int = 0, nranks: int = 1, nccl_uid: bytes | None = None,
                 stream: int | None = None):
        self.h = C.c_void_p()
        uid = C.create_string_buffer(nccl_uid, 128) if nccl_uid else None
        check(lib.amg_ctx_create(device, rank, nranks, uid, C.c_void_p(stream) if stream else None,
                                 C.byref(self.h)), "amg_ctx_create")
        self.device, self.rank, self.nranks = device, rank, nranks

    def close(self):
        if self.h:
            lib.amg_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _ptr(a):
    return C.c_void_p(a.ctypes.data)


class Hierarchy:
    """amg_hierarchy_build and the solve-phase calls on the built hierarchy."""

    def __init__(self, ctx: Context, A, cfg: amg_config_t | None = None, w=None):
        self.ctx = ctx
        self.h = C.c_void_p()
        rp = np.ascontiguousarray(A.rowptr, dtype=np.int64)
        ci = np.ascontiguousarray(A.colind, dtype=np.int64)
        v = np.ascontiguousarray(A.values, dtype=np.float64)
        wv = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
        self.cfg = cfg if cfg is not None else amg_config_default()
        check(lib.amg_hierarchy_build(ctx.h, A.n_global, A.row_begin, A.row_end, _ptr(rp), _ptr(ci),
                                      _ptr(v), _ptr(wv) if wv is not None else None, C.byref(self.cfg),
                                      C.byref(self.h)), "amg_hierarchy_build")
        self.n_local = A.row_end - A.row_begin

    def close(self):
        if self.h:
            lib.amg_hierarchy_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------- inspection
    @property
    def nlevels(self) -> int:
        n = C.c_int32()
        check(lib.amg_num_levels(self.h, C.byref(n)), "amg_num_levels")
        return n.value

    def level_info(self, l: int) -> dict:
        vals = [C.c_int64() for _ in range(5)]
        f = C.c_int32()
        check(lib.amg_level_info(self.h, l, *[C.byref(x) for x in vals], C.byref(f)), "amg_level_info")
        n, nnzA, nnzP, rb, re = (x.value for x in vals)
        return dict(n=n, nnzA=nnzA, nnzP=nnzP, row_begin=rb, row_end=re, format=_abi.FORMATS[f.value])

    def sizes(self):
        return [self.level_info(l)["n"] for l in range(self.nlevels)]

    def level_aggregates(self, l: int) -> np.ndarray:
        info = self.level_info(l)
        out = np.zeros(info["row_end"] - info["row_begin"], dtype=np.int64)
        check(lib.amg_level_aggregates(self.h, l, _ptr(out)), "amg_level_aggregates")
        return out

    def graph_mode(self) -> str:
        """amg_solve_graph_mode: 'while' (one graph per solve), 'iter' (one per iteration) or 'eager'."""
        m = C.c_int32()
        check(lib.amg_solve_graph_mode(self.h, C.byref(m)), "amg_solve_graph_mode")
        return ("while", "iter", "eager")[m.value]

    def transport(self) -> str:
        """amg_comm_transport: 'none', 'copies', 'nccl' or 'lsa' (peer memory)."""
        t = C.c_int32()
        check(lib.amg_comm_transport(self.h, C.byref(t)), "amg_comm_transport")
        return ("none", "copies", "nccl", "lsa")[t.value]

    def report(self) -> dict:
        r = amg_report_t()
        check(lib.amg_hierarchy_report(self.h, C.byref(r)), "amg_hierarchy_report")
        return r.as_dict()

    # ------------------------------------------------------------- solve phase
    def solve(self, b, x=None, rtol: float = 1e-6, maxit: int = 500):
        """amg_solve on CUDA tensors (fp64, this rank's rows)."""
        import torch
        if not (b.dtype == torch.float64 and b.is_cuda and b.is_contiguous() and b.numel() == self.n_local):
            raise ValueError(f"b must be a contiguous float64 CUDA tensor of {self.n_local} entries")
        if x is None:
            x = torch.empty_like(b)
        elif not (x.dtype == torch.float64 and x.is_cuda and x.is_contiguous() and x.numel() == self.n_local):
            raise ValueError(f"x must be a contiguous float64 CUDA tensor of {self.n_local} entries")
        torch.cuda.current_stream(b.device).synchronize()
        rep = amg_report_t()
        code = lib.amg_solve(self.h, C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()), float(rtol),
                             int(maxit), C.byref(rep))
        check(code, "amg_solve", ok=(AMG_OK, AMG_NOT_CONVERGED))
        return x, rep.as_dict()

    def solve_raw(self, b_ptr: int, x_ptr: int, rtol: float = 1e-6, maxit: int = 500) -> dict:
        rep = amg_report_t()
        code = lib.amg_solve(self.h, C.c_void_p(b_ptr), C.c_void_p(x_ptr), float(rtol), int(maxit),
                             C.byref(rep))
        check(code, "amg_solve", ok=(AMG_OK, AMG_NOT_CONVERGED))
        return rep.as_dict()

    def solve_host(self, b: np.ndarray, x: np.ndarray | None = None, rtol: float = 1e-6, maxit: int = 500):
        """amg_solve_host: host buffers, H2D/D2H copies inside the call."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        if b.shape != (self.n_local,):
            raise ValueError(f"b must have shape ({self.n_local},), got {b.shape}")
        if x is None:
            x = np.empty_like(b)
        elif not (isinstance(x, np.ndarray) and x.dtype == np.float64 and x.flags.c_contiguous
                  and x.shape == b.shape and x.flags.writeable):
            raise ValueError("x must be a writeable C-contiguous float64 array of b's shape")
        rep = amg_report_t()
        code = lib.amg_solve_host(self.h, _ptr(b), _ptr(x), float(rtol), int(maxit), C.byref(rep))
        check(code, "amg_solve_host", ok=(AMG_OK, AMG_NOT_CONVERGED))
        return x, rep.as_dict()

    def solve_host_batch(self, B: np.ndarray, X: np.ndarray | None = None, rtol: float = 1e-6,
                         maxit: int = 500):
        """amg_solve_host_batch: nrhs solves on host buffers (rows of B, C-contiguous), copies
        pipelined with the solves (pin B and X, e.g. torch.empty(...).pin_memory(), for overlap)."""
        if not (isinstance(B, np.ndarray) and B.dtype == np.float64 and B.flags.c_contiguous):
            B = np.ascontiguousarray(B, dtype=np.float64)
        if B.ndim not in (1, 2) or B.shape[-1] != self.n_local:
            raise ValueError(f"B must have shape (n,) or (nrhs, n) with n = {self.n_local}, got {B.shape}")
        nrhs = B.shape[0] if B.ndim == 2 else 1
        if X is None:
            X = np.empty_like(B)
        elif not (isinstance(X, np.ndarray) and X.dtype == np.float64 and X.flags.c_contiguous
                  and X.shape == B.shape and X.flags.writeable):
            raise ValueError("X must be a writeable C-contiguous float64 array of B's shape")
        reps = (amg_report_t * max(1, nrhs))()
        code = lib.amg_solve_host_batch(self.h, int(nrhs), _ptr(B), _ptr(X), float(rtol), int(maxit),
                                        C.cast(reps, C.c_void_p))
        check(code, "amg_solve_host_batch", ok=(AMG_OK, AMG_NOT_CONVERGED))
        return X, [reps[k].as_dict() for k in range(nrhs)]

    def precond_apply(self, r, z=None):
        """amg_precond_apply: one V-cycle z = B r on CUDA tensors."""
        import torch
        if not (r.dtype == torch.float64 and r.is_cuda and r.is_contiguous() and r.numel() == self.n_local):
            raise ValueError(f"r must be a contiguous float64 CUDA tensor of {self.n_local} entries")
        if z is None:
            z = torch.empty_like(r)
        elif not (z.dtype == torch.float64 and z.is_cuda and z.is_contiguous() and z.numel() == self.n_local):
            raise ValueError(f"z must be a contiguous float64 CUDA tensor of {self.n_local} entries")
        torch.cuda.current_stream(r.device).synchronize()
        check(lib.amg_precond_apply(self.h, C.c_void_p(r.data_ptr()), C.c_void_p(z.data_ptr())),
              "amg_precond_apply")
        return z

    def profile_vcycle(self, napply: int = 10, cap: int = 256):
        ms = np.zeros(cap)
        by = np.zeros(cap)
        sb = np.zeros(cap)
        names = (C.c_char_p * cap)()
        cnt = C.c_int32()
        check(lib.amg_profile_vcycle(self.h, napply, cap, _ptr(ms), _ptr(by), _ptr(sb), names, C.byref(cnt)),
              "amg_profile_vcycle")
        k = min(cnt.value, cap)
        return [dict(name=names[i].decode(), ms=float(ms[i]), bytes=float(by[i]), stored_bytes=float(sb[i]))
                for i in range(k)]

    def profile_iteration(self, b, napply: int = 10, cap: int = 512):
        """amg_profile_iteration: per-kernel device times of whole solver iterations (b: CUDA tensor;
        a scratch x is used)."""
        import torch
        if not (b.dtype == torch.float64 and b.is_cuda and b.is_contiguous() and b.numel() == self.n_local):
            raise ValueError(f"b must be a contiguous float64 CUDA tensor of {self.n_local} entries")
        x = torch.empty_like(b)
        torch.cuda.current_stream(b.device).synchronize()
        ms = np.zeros(cap)
        by = np.zeros(cap)
        sb = np.zeros(cap)
        names = (C.c_char_p * cap)()
        cnt = C.c_int32()
        check(lib.amg_profile_iteration(self.h, C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()), napply, cap,
                                        _ptr(ms), _ptr(by), _ptr(sb), names, C.byref(cnt)), "amg_profile_iteration")
        k = min(cnt.value, cap)
        return [dict(name=names[i].decode(), ms=float(ms[i]), bytes=float(by[i]), stored_bytes=float(sb[i]))
                for i in range(k)]
