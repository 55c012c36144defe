"""CPU-side checks of the product library (no GPU needed):

  * libamg_b200.so loads and exports every function declared in include/amg_b200.h;
  * its host setup (parallel locally-dominant matching, row-parallel canonical
    SpGEMM — an implementation independent of oracle/) reproduces the oracle's
    aggregate maps bit-exactly at every level, and (a stronger diagnostic) the
    coarse operators A_l and smoothed prolongators P-bar_l bit for bit;
  * argument validation and error codes.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
from inputs import config_problem, diagonal_spd, islands, jump27, poisson7, random_spd, uniform01

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def amg():
    import paper_2006_16147_b200 as amg
    return amg


def declared_functions():
    src = open(os.path.join(ROOT, "include", "amg_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+char\s*\*|int|void)\s+(amg_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol(amg):
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(amg.lib, n), n
    from paper_2006_16147_b200 import _abi
    assert set(_abi.EXPORTED) <= set(names)


def test_config_default_matches_header(amg):
    c = amg.amg_config_default()
    assert (c.sweeps_per_level, c.smooth_prolongator, c.max_coarse_size, c.max_levels) == (3, 1, 200, 20)
    assert c.prol_omega_scale == 4.0 / 3.0 and c.min_coarsening_ratio == 1.2
    assert (c.pre_sweeps, c.post_sweeps, c.use_graphs) == (1, 1, 1)
    # the paper's GPU method is opt-in: PCG + direct coarsest by default (readings R1, R2)
    assert (c.krylov, c.coarse_solver, c.coarse_maxit, c.coarse_rtol) == (0, 0, 30, 1e-4)
    assert c.cycle == 0  # V-cycle by default (the north_star path); K-cycle opt-in (NEXT-4)
    assert c.setup_device == 1  # GPU setup (NEXT-1), bit-identical to the host build
    assert c.tail_rows == 0  # persistent cooperative tail: experimental, off by default (slower)
    assert (c.smoother, c.invk_fill) == (0, 1)  # l1-Jacobi by default; INVK opt-in (NEXT-3)


def test_config_struct_layout_matches_header(amg):
    # every field the header declares, in order, is in the ctypes mirror
    import re
    txt = open(os.path.join(ROOT, "include", "amg_b200.h")).read()
    body = txt[txt.index("typedef struct {"):txt.index("} amg_config_t;")]
    fields = re.findall(r"^\s*(?:int32_t|int64_t|double)\s+(\w+);", body, re.M)
    from paper_2006_16147_b200 import _abi
    assert fields == [f for f, _ in _abi.amg_config_t._fields_]


class HostH:
    """Wrapper of the amg_host_* inspection entry points."""

    def __init__(self, amg, A, w=None, **cfg):
        L = amg.lib
        self.L = L
        self.h = C.c_void_p()
        c = amg.make_config(**dict({"setup_device": 0}, **cfg))  # host build unless asked (CPU box)
        self._keep = [np.ascontiguousarray(A.rowptr, np.int64), np.ascontiguousarray(A.colind, np.int64),
                      np.ascontiguousarray(A.values, np.float64)]
        wp = None
        if w is not None:
            self._keep.append(np.ascontiguousarray(w, np.float64))
            wp = C.c_void_p(self._keep[-1].ctypes.data)
        L.amg_host_hierarchy_build.argtypes = [C.c_int64] + [C.c_void_p] * 4 + [C.c_void_p, C.c_void_p]
        self.code = L.amg_host_hierarchy_build(A.n_global, *[C.c_void_p(a.ctypes.data) for a in self._keep[:3]],
                                               wp, C.byref(c), C.byref(self.h))

    def __del__(self):
        if self.h:
            self.L.amg_host_hierarchy_destroy(self.h)

    @property
    def nlevels(self):
        n = C.c_int32()
        self.L.amg_host_num_levels(self.h, C.byref(n))
        return n.value

    def sizes(self, l):
        n, a, p = C.c_int64(), C.c_int64(), C.c_int64()
        om = C.c_double()
        self.L.amg_host_level_sizes(self.h, l, C.byref(n), C.byref(a), C.byref(p), C.byref(om))
        return n.value, a.value, p.value, om.value

    def agg(self, l):
        n = self.sizes(l)[0]
        out = np.zeros(n, np.int64)
        assert self.L.amg_host_level_aggregates(self.h, l, C.c_void_p(out.ctypes.data)) == 0
        return out

    def matrix(self, l, which):
        n, nnzA, nnzP, _ = self.sizes(l)
        nnz = nnzA if which == 0 else nnzP
        rp = np.zeros(n + 1, np.int64)
        ci = np.zeros(max(nnz, 1), np.int64)
        v = np.zeros(max(nnz, 1))
        assert self.L.amg_host_level_matrix(self.h, l, which, C.c_void_p(rp.ctypes.data),
                                            C.c_void_p(ci.ctypes.data), C.c_void_p(v.ctypes.data)) == 0
        return rp, ci[:nnz], v[:nnz]


def _compare(amg, A, w=None, **cfg):
    hl = HostH(amg, A, w=w, **cfg)
    assert hl.code == 0, amg.amg_last_error()
    ho = O.OracleHierarchy(A, w=w, **cfg)
    assert hl.nlevels == ho.nlevels
    for l in range(ho.nlevels):
        assert hl.sizes(l)[0] == ho.level_n(l)
        rp, ci, v = hl.matrix(l, 0)
        orp, oci, ov = ho.A(l).arrays()
        assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
        assert np.array_equal(v.view(np.int64), ov.view(np.int64)), f"A_{l} values differ bitwise"
        if l + 1 < ho.nlevels:
            assert np.array_equal(hl.agg(l), ho.agg(l)), f"aggregates differ at level {l}"
            assert hl.sizes(l)[3] == ho.omega(l)
            rp, ci, v = hl.matrix(l, 1)
            orp, oci, ov = ho.P(l).arrays()
            assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
            assert np.array_equal(v.view(np.int64), ov.view(np.int64)), f"P_{l} values differ bitwise"
    return hl, ho


@pytest.mark.parametrize("case", ["c1", "aniso_32", "jump_16", "ragged", "unsmoothed_20", "random_w",
                                  "omega_text", "m4_sweeps", "c4_like_24x24x48", "irregular_hubs",
                                  "irregular_narrow", "line_1d", "plane_2d", "diagonal", "n1", "islands",
                                  "pair_mcs1"])
def test_host_setup_bit_exact_vs_oracle(amg, case):
    w, cfg = None, {}
    if case == "c1":
        A = config_problem(1)[0]
    elif case == "aniso_32":
        A = poisson7(32, 32, 32, (1, 1, 0.01))
        cfg = dict(pre_sweeps=2, post_sweeps=2)
    elif case == "jump_16":
        A = jump27(16)
    elif case == "ragged":
        A = poisson7(17, 13, 11)
    elif case == "unsmoothed_20":
        A = poisson7(20, 20, 20)
        cfg = dict(smooth_prolongator=0)
    elif case == "random_w":
        A = poisson7(14, 12, 10)
        w = 0.5 + uniform01(99, A.n_global)
    elif case == "omega_text":
        A = poisson7(16, 16, 16)
        cfg = dict(prol_omega_scale=1.0)
    elif case == "m4_sweeps":
        A = poisson7(24, 24, 24)
        cfg = dict(sweeps_per_level=4, max_coarse_size=20)
    elif case == "irregular_hubs":  # ragged rows 3..312 entries, long-range hub couplings
        A = random_spd(6000, hubs=3)
    elif case == "irregular_narrow":
        A = random_spd(3000, deg=3, window=5)
    elif case == "line_1d":  # 1-D chain: pairs only, cr 2 per sweep
        A = poisson7(1000, 1, 1)
    elif case == "plane_2d":
        A = poisson7(40, 30, 1)
    elif case == "diagonal":  # no couplings: nothing to match, single level
        A = diagonal_spd(300)
    elif case == "n1":
        A = diagonal_spd(1)
    elif case == "islands":  # two components + isolated rows, interleaved: coarsening stalls at 43
        A = islands()
        cfg = dict(max_coarse_size=20)
    elif case == "pair_mcs1":  # 2 rows, max_coarse_size 1: a 1-row coarsest level
        A = poisson7(2, 1, 1)
        cfg = dict(max_coarse_size=1)
    else:
        A = poisson7(24, 24, 48)
        cfg = dict(max_coarse_size=400)
    _compare(amg, A, w=w, **cfg)


@pytest.mark.slow
def test_host_setup_reproduces_tableSM_80cube(amg):
    """The library's own setup also reproduces Table SM:
    80^3, unsmoothed 3 sweeps -> nl = 5, cr = 8 per level, coarsest 125."""
    A = poisson7(80, 80, 80)
    hl = HostH(amg, A, smooth_prolongator=0)
    assert hl.code == 0
    sizes = [hl.sizes(l)[0] for l in range(hl.nlevels)]
    assert sizes == [512000, 64000, 8000, 1000, 125]


@pytest.mark.slow
def test_host_setup_bit_exact_c2(amg):
    """Full config 2 (128^3): every level's aggregates, A_l and P-bar_l bit-exact."""
    A = config_problem(2)[0]
    _compare(amg, A)


def test_host_setup_errors(amg):
    A = poisson7(4, 4, 4)
    A.values = A.values.copy()
    A.values[1] = -2.0
    assert HostH(amg, A).code == 1  # asymmetric
    A = poisson7(4, 4, 4)
    A.values = -A.values
    assert HostH(amg, A).code == 2  # non-positive diagonal
    A = poisson7(4, 4, 4)
    assert HostH(amg, A, w=np.zeros(64)).code == 2  # w == 0
    A = poisson7(4, 4, 4)
    assert HostH(amg, A, pre_sweeps=0).code == 1
    A = poisson7(4, 4, 4)
    A.colind = A.colind.copy()
    A.colind[0], A.colind[1] = A.colind[1], A.colind[0]  # unsorted row
    assert HostH(amg, A).code == 1


def test_null_handles_and_bad_arguments_are_status_codes(amg):
    """Every entry point answers a NULL handle / NULL output / bad argument with
    AMG_ERR_ARG (1) and a message, never a crash (include/amg_b200.h: status codes
    only, no exceptions across the ABI)."""
    L = amg.lib
    null = C.c_void_p()
    i32, i64, f64 = C.c_int32(), C.c_int64(), C.c_double()
    from paper_2006_16147_b200 import _abi
    rep = C.byref(_abi.amg_report_t())
    buf = np.zeros(16)
    p = C.c_void_p(buf.ctypes.data)
    calls = {
        "amg_solve": lambda: L.amg_solve(null, p, p, C.c_double(1e-6), C.c_int32(10), rep),
        "amg_solve_host": lambda: L.amg_solve_host(null, p, p, C.c_double(1e-6), C.c_int32(10), rep),
        "amg_precond_apply": lambda: L.amg_precond_apply(null, p, p),
        "amg_num_levels": lambda: L.amg_num_levels(null, C.byref(i32)),
        "amg_solve_graph_mode": lambda: L.amg_solve_graph_mode(null, C.byref(i32)),
        "amg_comm_transport": lambda: L.amg_comm_transport(null, C.byref(i32)),
        "amg_level_info": lambda: L.amg_level_info(null, 0, C.byref(i64), C.byref(i64), C.byref(i64),
                                                   C.byref(i64), C.byref(i64), C.byref(i32)),
        "amg_level_aggregates": lambda: L.amg_level_aggregates(null, 0, p),
        "amg_hierarchy_report": lambda: L.amg_hierarchy_report(null, rep),
        "amg_host_num_levels": lambda: L.amg_host_num_levels(null, C.byref(i32)),
        "amg_host_level_sizes": lambda: L.amg_host_level_sizes(null, 0, C.byref(i64), C.byref(i64),
                                                               C.byref(i64), C.byref(f64)),
        "amg_host_level_aggregates": lambda: L.amg_host_level_aggregates(null, 0, p),
    }
    for name, call in calls.items():
        assert call() == 1, name
        assert amg.amg_last_error(), name
    # a valid host hierarchy rejects out-of-range levels and a bad matrix selector
    h = HostH(amg, poisson7(6, 6, 6))
    assert h.code == 0
    nl = h.nlevels
    assert L.amg_host_level_sizes(h.h, nl, C.byref(i64), C.byref(i64), C.byref(i64), C.byref(f64)) == 1
    assert L.amg_host_level_aggregates(h.h, nl - 1, p) == 1  # the coarsest has no aggregates
    assert L.amg_host_level_matrix(h.h, 0, 7, p, p, p) == 1
