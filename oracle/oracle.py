"""ctypes wrapper of oracle/liboracle.so — TEST INFRASTRUCTURE ONLY (see oracle.h)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

OR_OK, OR_ERR_ARG, OR_ERR_NOT_SPD, OR_NOT_CONVERGED, OR_BREAKDOWN = 0, 1, 2, 6, 7

__all__ = ["build_oracle", "OracleCSR", "OracleHierarchy", "lib", "edge_weights",
           "greedy_matching", "aggregates", "pairwise_sweep", "dinv_a_inf_norm",
           "l1_jacobi_inv", "rap", "smooth_prolongator", "spmv",
           "OR_OK", "OR_ERR_ARG", "OR_ERR_NOT_SPD", "OR_NOT_CONVERGED", "OR_BREAKDOWN"]


def build_oracle(force: bool = False) -> str:
    """Compile the oracle (plain C, -O2 -ffp-contract=off, no BLAS)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
                               "-o", _SO, src, "-lm"])
    return _SO


_lib = None
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_vp = C.c_void_p


def lib():
    global _lib
    if _lib is not None:
        return _lib
    L = C.CDLL(build_oracle())
    sig = {
        "or_csr_new_copy": (_vp, [C.c_int64, C.c_int64, _i64p, _i64p, _f64p]),
        "or_csr_dims": (None, [_vp, _i64p]),
        "or_csr_export": (None, [_vp, _i64p, _i64p, _f64p]),
        "or_csr_free": (None, [_vp]),
        "or_spmv": (None, [_vp, _f64p, _f64p]),
        "or_rap": (_vp, [_vp, _vp, _vp]),
        "or_mirror_drop": (None, [_vp]),
        "or_edge_weights": (C.c_int64, [_vp, _f64p, _i64p, _i64p, _f64p]),
        "or_greedy_matching": (None, [C.c_int64, C.c_int64, _i64p, _i64p, _f64p, _i64p]),
        "or_aggregates": (C.c_int64, [C.c_int64, _i64p, _i64p]),
        "or_pairwise_sweep": (_vp, [_vp, _f64p, _f64p, _i64p, _f64p, C.POINTER(C.c_int64)]),
        "or_dinv_a_inf_norm": (C.c_double, [_vp]),
        "or_prolongator_csr": (_vp, [C.c_int64, C.c_int64, _i64p, _f64p]),
        "or_smooth_prolongator": (_vp, [_vp, _vp, C.c_double]),
        "or_l1_jacobi_inv": (None, [_vp, _f64p]),
        "or_build": (_vp, [_vp, _vp, C.c_int32, C.c_int32, C.c_double, C.c_int64, C.c_int32,
                           C.c_double, C.c_int32, C.c_int32, C.POINTER(C.c_int32)]),
        "or_free": (None, [_vp]),
        "or_nlevels": (C.c_int32, [_vp]),
        "or_level_A": (_vp, [_vp, C.c_int32]),
        "or_level_P": (_vp, [_vp, C.c_int32]),
        "or_level_n": (C.c_int64, [_vp, C.c_int32]),
        "or_level_agg": (None, [_vp, C.c_int32, _i64p]),
        "or_level_pval": (None, [_vp, C.c_int32, _f64p]),
        "or_level_w": (None, [_vp, C.c_int32, _f64p]),
        "or_level_m": (None, [_vp, C.c_int32, _f64p]),
        "or_level_omega": (C.c_double, [_vp, C.c_int32]),
        "or_level_sweeps": (C.c_int32, [_vp, C.c_int32]),
        "or_opc": (C.c_double, [_vp]),
        "or_avg_cr": (C.c_double, [_vp]),
        "or_vcycle": (None, [_vp, _f64p, _f64p]),
        "or_pcg": (C.c_int32, [_vp, _f64p, _f64p, C.c_double, C.c_int32,
                               C.POINTER(C.c_int32), C.POINTER(C.c_double),
                               C.POINTER(C.c_double), _vp]),
        "or_fcg": (C.c_int32, [_vp, _f64p, _f64p, C.c_double, C.c_int32,
                               C.POINTER(C.c_int32), C.POINTER(C.c_double),
                               C.POINTER(C.c_double), _vp]),
        "or_set_coarse_cg": (None, [_vp, C.c_int32, C.c_double, C.c_int32]),
        "or_set_smoother_ex": (C.c_int32, [_vp, C.c_int32, C.c_int32, C.c_int32, _vp, C.c_int32, _vp]),
        "or_set_coarse_prec": (None, [_vp, C.c_int32]),
        "or_level_visits": (C.c_int64, [_vp, C.c_int32]),
        "or_set_threads": (None, [C.c_int32]),
        "or_set_cycle": (None, [_vp, C.c_int32]),
        "or_set_smoother": (C.c_int32, [_vp, C.c_int32, C.c_int32]),
        "or_level_invk": (_vp, [_vp, C.c_int32, C.c_int32]),
        "or_coarse_visits": (C.c_int64, [_vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _cf(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleCSR:
    """Owning handle of an oracle CSR matrix."""

    def __init__(self, handle, owned=True):
        self.h = handle
        self.owned = owned

    @classmethod
    def from_arrays(cls, nrows, ncols, rowptr, colind, values):
        L = lib()
        return cls(L.or_csr_new_copy(int(nrows), int(ncols), _c64(rowptr), _c64(colind),
                                     _cf(values)))

    @classmethod
    def from_scipy(cls, M):
        M = M.tocsr()
        M.sort_indices()
        return cls.from_arrays(M.shape[0], M.shape[1], M.indptr, M.indices, M.data)

    @classmethod
    def from_inputs(cls, A):
        """From an inputs.problems.CSR holding all rows."""
        assert A.row_begin == 0 and A.row_end == A.n_global
        return cls.from_arrays(A.n_global, A.n_global, A.rowptr, A.colind, A.values)

    def dims(self):
        d = np.zeros(3, np.int64)
        lib().or_csr_dims(self.h, d)
        return int(d[0]), int(d[1]), int(d[2])

    def arrays(self):
        nr, nc, nnz = self.dims()
        rp = np.zeros(nr + 1, np.int64)
        ci = np.zeros(max(nnz, 1), np.int64)
        v = np.zeros(max(nnz, 1), np.float64)
        lib().or_csr_export(self.h, rp, ci, v)
        return rp, ci[:nnz], v[:nnz]

    def to_scipy(self):
        import scipy.sparse as sp
        nr, nc, _ = self.dims()
        rp, ci, v = self.arrays()
        return sp.csr_matrix((v, ci, rp), shape=(nr, nc))

    def __del__(self):
        if self.owned and self.h and _lib is not None:
            _lib.or_csr_free(self.h)
            self.h = None


def spmv(A: OracleCSR, x):
    nr, _, _ = A.dims()
    y = np.zeros(nr)
    lib().or_spmv(A.h, _cf(x), y)
    return y


def rap(X: OracleCSR, A: OracleCSR, Y: OracleCSR, mirror=True) -> OracleCSR:
    C_ = OracleCSR(lib().or_rap(X.h, A.h, Y.h))
    if mirror:
        lib().or_mirror_drop(C_.h)
    return C_


def edge_weights(A: OracleCSR, w):
    _, _, nnz = A.dims()
    ei = np.zeros(max(nnz, 1), np.int64)
    ej = np.zeros(max(nnz, 1), np.int64)
    c = np.zeros(max(nnz, 1))
    ne = lib().or_edge_weights(A.h, _cf(w), ei, ej, c)
    return ei[:ne], ej[:ne], c[:ne]


def greedy_matching(n, ei, ej, c):
    mate = np.zeros(max(n, 1), np.int64)
    lib().or_greedy_matching(int(n), len(ei), _c64(ei), _c64(ej), _cf(c), mate)
    return mate[:n]


def aggregates(n, mate):
    agg = np.zeros(max(n, 1), np.int64)
    nc = lib().or_aggregates(int(n), _c64(mate), agg)
    return int(nc), agg[:n]


def pairwise_sweep(A: OracleCSR, w):
    n, _, _ = A.dims()
    wn = np.zeros(n)
    agg = np.zeros(n, np.int64)
    pv = np.zeros(n)
    nc = C.c_int64(0)
    An = OracleCSR(lib().or_pairwise_sweep(A.h, _cf(w), wn, agg, pv, C.byref(nc)))
    nc = nc.value
    return An, wn[:nc], agg, pv, nc


def dinv_a_inf_norm(A: OracleCSR) -> float:
    return lib().or_dinv_a_inf_norm(A.h)


def l1_jacobi_inv(A: OracleCSR):
    n, _, _ = A.dims()
    m = np.zeros(n)
    lib().or_l1_jacobi_inv(A.h, m)
    return m


def smooth_prolongator(A: OracleCSR, n, nc, agg, pval, omega) -> OracleCSR:
    P = OracleCSR(lib().or_prolongator_csr(int(n), int(nc), _c64(agg), _cf(pval)))
    return OracleCSR(lib().or_smooth_prolongator(A.h, P.h, float(omega)))


class OracleHierarchy:
    """Hierarchy built by the oracle."""

    def __init__(self, A, w=None, sweeps_per_level=3, smooth_prolongator=1,
                 prol_omega_scale=4.0 / 3.0, max_coarse_size=200, max_levels=20,
                 min_coarsening_ratio=1.2, pre_sweeps=1, post_sweeps=1):
        L = lib()
        if not isinstance(A, OracleCSR):
            A = OracleCSR.from_inputs(A) if hasattr(A, "row_begin") else OracleCSR.from_scipy(A)
        self._A0 = A
        self.n = A.dims()[0]
        st = C.c_int32(0)
        wp = None
        if w is not None:
            self._w = _cf(w)
            wp = self._w.ctypes.data_as(C.c_void_p)
        self.h = L.or_build(A.h, wp, sweeps_per_level, smooth_prolongator, prol_omega_scale,
                            max_coarse_size, max_levels, min_coarsening_ratio, pre_sweeps,
                            post_sweeps, C.byref(st))
        self.status = st.value
        if not self.h:
            raise ValueError(f"oracle build failed with status {self.status}")

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.or_free(self.h)
            self.h = None

    @property
    def nlevels(self) -> int:
        return lib().or_nlevels(self.h)

    def level_n(self, l):
        return lib().or_level_n(self.h, l)

    def sizes(self):
        return [self.level_n(l) for l in range(self.nlevels)]

    def A(self, l) -> OracleCSR:
        return OracleCSR(lib().or_level_A(self.h, l), owned=False)

    def P(self, l) -> OracleCSR:
        return OracleCSR(lib().or_level_P(self.h, l), owned=False)

    def agg(self, l):
        a = np.zeros(self.level_n(l), np.int64)
        lib().or_level_agg(self.h, l, a)
        return a

    def pval(self, l):
        a = np.zeros(self.level_n(l))
        lib().or_level_pval(self.h, l, a)
        return a

    def w(self, l):
        a = np.zeros(self.level_n(l))
        lib().or_level_w(self.h, l, a)
        return a

    def m(self, l):
        a = np.zeros(self.level_n(l))
        lib().or_level_m(self.h, l, a)
        return a

    def omega(self, l):
        return lib().or_level_omega(self.h, l)

    def sweeps(self, l):
        return lib().or_level_sweeps(self.h, l)

    def nnz(self, l):
        return self.A(l).dims()[2]

    @property
    def opc(self):
        return lib().or_opc(self.h)

    @property
    def avg_cr(self):
        return lib().or_avg_cr(self.h)

    def vcycle(self, r):
        z = np.zeros(self.n)
        lib().or_vcycle(self.h, _cf(r), z)
        return z

    def set_coarse_cg(self, on=True, rtol=1e-4, maxit=30):
        """Coarsest level by l1-Jacobi PCG instead of Cholesky."""
        lib().or_set_coarse_cg(self.h, int(on), float(rtol), int(maxit))

    def set_cycle(self, kind="V"):
        """'V' (Eq. 3.1) or 'K' (K-cycle: two FCG(1) iterations per intermediate level)."""
        lib().or_set_cycle(self.h, {"V": 0, "K": 1}[kind])

    def set_smoother(self, kind="l1jacobi", fill=1, blocks=None, l1=False, fill_per_level=None):
        """'l1jacobi' or 'invk' (`fill` levels in the inversion).
        blocks: level-0 row bounds [0, b1, ..., n] of the parallel block-Jacobi setting (HINVK on
        the diagonal blocks); l1=True: l1-INVK (A_pp + D_l1,p)."""
        nb = 1 if blocks is None else len(blocks) - 1
        self._bounds = None if blocks is None else np.ascontiguousarray(blocks, dtype=np.int64)
        self._fills = None if fill_per_level is None else np.ascontiguousarray(fill_per_level, dtype=np.int32)
        st = lib().or_set_smoother_ex(
            self.h, {"l1jacobi": 0, "invk": 1}[kind], int(fill), nb,
            None if self._bounds is None else self._bounds.ctypes.data_as(C.c_void_p), int(bool(l1)),
            None if self._fills is None else self._fills.ctypes.data_as(C.c_void_p))
        if st != OR_OK:
            raise RuntimeError(f"or_set_smoother failed with status {st}")

    def set_coarse_prec(self, kind="l1jacobi"):
        """Coarse CG preconditioner: 'l1jacobi' (VA3S5CS1) or 'invk' (VA3S3CS1).
        Call before set_smoother, which builds the coarsest level's factors."""
        lib().or_set_coarse_prec(self.h, {"l1jacobi": 0, "invk": 1}[kind])

    def level_visits(self, l):
        """Cycle applications rooted at level l since the build."""
        return lib().or_level_visits(self.h, int(l))

    @staticmethod
    def set_threads(t):
        """Solve-phase threads: 1 = sequential parity reference; > 1 = OpenMP (timing only)."""
        lib().or_set_threads(int(t))

    def invk(self, l, which):
        """which = 0: D^{-1} W; 1: Z = W^T (INVK factors of level l, borrowed)."""
        return OracleCSR(lib().or_level_invk(self.h, l, which), owned=False)

    @property
    def coarse_visits(self):
        return lib().or_coarse_visits(self.h)

    def fcg(self, b, rtol=1e-6, maxit=500, history=False):
        return self.pcg(b, rtol, maxit, history, _fn="or_fcg")

    def pcg(self, b, rtol=1e-6, maxit=500, history=False, _fn="or_pcg"):
        x = np.zeros(self.n)
        it = C.c_int32(0)
        rr = C.c_double(0)
        tr = C.c_double(0)
        hist = np.zeros(maxit + 1) if history else None
        st = getattr(lib(), _fn)(self.h, _cf(b), x, float(rtol), int(maxit), C.byref(it), C.byref(rr),
                                 C.byref(tr), hist.ctypes.data_as(C.c_void_p) if history else None)
        out = dict(status=st, iterations=it.value, relres=rr.value, true_relres=tr.value)
        if history:
            out["history"] = hist[:it.value + 1]
        return x, out
