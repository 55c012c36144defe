"""Dump hierarchy operators A_l (and the restriction/prolongation of level 0) as
binary CSR files for tools/spmv_lab3.cu: int64 n, int64 nnz, int32 rowptr[n+1],
int32 col[nnz], f64 val[nnz].

  python tools/dump_levels.py OUTDIR c2          # 128^3 7-point, levels 1..4
  python tools/dump_levels.py OUTDIR c5 192      # 27-point jump, N^3, levels 1..3
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_16147_b200 as amg  # noqa: E402
from inputs import config_problem, jump27  # noqa: E402


def write(path, rp, ci, v):
    with open(path, "wb") as f:
        np.array([len(rp) - 1, len(ci)], np.int64).tofile(f)
        rp.astype(np.int32).tofile(f)
        ci.astype(np.int32).tofile(f)
        v.astype(np.float64).tofile(f)


def main():
    out, which = sys.argv[1], sys.argv[2]
    os.makedirs(out, exist_ok=True)
    if which == "c2":
        A = config_problem(2)[0]
        levels = range(1, 5)
    else:
        N = int(sys.argv[3]) if len(sys.argv) > 3 else 192
        A = jump27(N)
        levels = range(1, 4)
    L = amg.lib
    h = C.c_void_p()
    cfg = amg.make_config(setup_device=int(os.environ.get("SETUP_DEVICE", "1")))
    keep = [np.ascontiguousarray(A.rowptr, np.int64), np.ascontiguousarray(A.colind, np.int64),
            np.ascontiguousarray(A.values, np.float64)]
    L.amg_host_hierarchy_build.argtypes = [C.c_int64] + [C.c_void_p] * 4 + [C.c_void_p, C.c_void_p]
    st = L.amg_host_hierarchy_build(A.n_global, *[C.c_void_p(a.ctypes.data) for a in keep], None,
                                    C.byref(cfg), C.byref(h))
    assert st == 0, amg.amg_last_error()
    nl = C.c_int32()
    L.amg_host_num_levels(h, C.byref(nl))
    for l in ([0] if os.environ.get("DUMP_P") else []):  # P-bar_0 (prolongation) as well
        n, a, p = C.c_int64(), C.c_int64(), C.c_int64()
        om = C.c_double()
        L.amg_host_level_sizes(h, l, C.byref(n), C.byref(a), C.byref(p), C.byref(om))
        rp = np.zeros(n.value + 1, np.int64)
        ci = np.zeros(max(p.value, 1), np.int64)
        v = np.zeros(max(p.value, 1))
        assert L.amg_host_level_matrix(h, l, 1, C.c_void_p(rp.ctypes.data), C.c_void_p(ci.ctypes.data),
                                       C.c_void_p(v.ctypes.data)) == 0
        path = os.path.join(out, f"{which}_P{l}.csr")
        write(path, rp, ci[:p.value], v[:p.value])
        print(path, n.value, p.value, p.value / n.value)
    for l in levels:
        if l >= nl.value:
            break
        n, a, p = C.c_int64(), C.c_int64(), C.c_int64()
        om = C.c_double()
        L.amg_host_level_sizes(h, l, C.byref(n), C.byref(a), C.byref(p), C.byref(om))
        rp = np.zeros(n.value + 1, np.int64)
        ci = np.zeros(max(a.value, 1), np.int64)
        v = np.zeros(max(a.value, 1))
        assert L.amg_host_level_matrix(h, l, 0, C.c_void_p(rp.ctypes.data), C.c_void_p(ci.ctypes.data),
                                       C.c_void_p(v.ctypes.data)) == 0
        path = os.path.join(out, f"{which}_A{l}.csr")
        write(path, rp, ci[:a.value], v[:a.value])
        print(path, n.value, a.value, a.value / n.value)
    L.amg_host_hierarchy_destroy(h)


if __name__ == "__main__":
    main()
