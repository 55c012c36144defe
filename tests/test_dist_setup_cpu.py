"""Distributed hierarchy setup against the
single-process build, on CPU.

amg_host_dist_build runs np ranks (threads of one process, an in-process transport): each rank
holds only its row block of every level, matches with cross-rank pointer exchanges, gathers the
remote rows the Galerkin products need, all-reduces omega, and builds its own plan.  The bar is
bit-identity with amg_host_hierarchy_build + amg_host_partition: every level's A_l, P-bar_l,
aggregate map and omega, and every rank's plan (windows, halo lists, local operators in window
frames, l1 diagonal) -- and hence, by the single build's tests, the oracle's aggregate maps.
"""
import ctypes as C
import os

import numpy as np
import pytest

from inputs import config_problem, islands, jump27, poisson7, random_spd, uniform01


def _amg():
    import paper_2006_16147_b200 as amg
    return amg


def _ptrs(A):
    rp = np.ascontiguousarray(A.rowptr, dtype=np.int64)
    ci = np.ascontiguousarray(A.colind, dtype=np.int64)
    v = np.ascontiguousarray(A.values, dtype=np.float64)
    return (rp, ci, v), (A.n_global, C.c_void_p(rp.ctypes.data), C.c_void_p(ci.ctypes.data), C.c_void_p(v.ctypes.data))


def _build(A, cfg, w=None, nranks=None, rep=64 << 20):
    amg = _amg()
    keep, args = _ptrs(A)
    wv = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
    wp = None if wv is None else C.c_void_p(wv.ctypes.data)
    h = C.c_void_p()
    if nranks is None:
        amg.check(amg.lib.amg_host_hierarchy_build(*args, wp, C.byref(cfg), C.byref(h)), "host build")
    else:
        amg.check(amg.lib.amg_host_dist_build(*args, wp, C.byref(cfg), nranks, rep, C.byref(h)), "dist build")
    return h


def _levels(h):
    amg = _amg()
    nl = C.c_int32()
    amg.lib.amg_host_num_levels(h, C.byref(nl))
    out = []
    for l in range(nl.value):
        n, na, npp, om = C.c_int64(), C.c_int64(), C.c_int64(), C.c_double()
        amg.lib.amg_host_level_sizes(h, l, C.byref(n), C.byref(na), C.byref(npp), C.byref(om))
        mats = []
        for which, nz in ((0, na.value), (1, npp.value)):
            if which == 1 and l + 1 == nl.value:
                continue
            rp, ci, v = np.zeros(n.value + 1, np.int64), np.zeros(nz, np.int64), np.zeros(nz)
            amg.lib.amg_host_level_matrix(h, l, which, C.c_void_p(rp.ctypes.data), C.c_void_p(ci.ctypes.data),
                                          C.c_void_p(v.ctypes.data))
            mats.append((rp, ci, v))
        agg = None
        if l + 1 < nl.value:
            agg = np.zeros(n.value, np.int64)
            amg.lib.amg_host_level_aggregates(h, l, C.c_void_p(agg.ctypes.data))
        out.append(dict(n=n.value, omega=om.value, mats=mats, agg=agg))
    return out


def _plans(h, nr, nl):
    amg = _amg()
    out = []
    for r in range(nr):
        for l in range(nl):
            info = np.zeros(16, np.int64)
            amg.check(amg.lib.amg_host_plan_level(h, r, l, C.c_void_p(info.ctypes.data)), "plan level")
            rec = [info.copy()]
            win, comp, rst = info[7] - info[6], info[5] - info[4], info[9] - info[8]
            sizes = {0: nr + 1, 1: info[10], 2: nr + 1, 3: info[11], 4: comp + 1, 5: info[12], 6: info[12],
                     7: comp + 1, 8: info[13], 9: info[13], 10: rst + 1, 11: info[14], 12: info[14], 13: win}
            for which in range(14):
                if which in (7, 8, 9, 10, 11, 12) and l == nl - 1:
                    continue
                dt = np.float64 if which in (6, 9, 12, 13) else np.int64
                a = np.zeros(max(1, int(sizes[which])), dt)
                amg.check(amg.lib.amg_host_plan_array(h, r, l, which, C.c_void_p(a.ctypes.data)), "plan array")
                rec.append(a)
            out.append(rec)
    return out


def _case(name):
    if name == "c4_32x32x64":          # config-4 analogue, z-slabs
        return config_problem(4, grid=(32, 32, 64))[0], {}, None
    if name == "c4_24x24x96_np8":
        return config_problem(4, grid=(24, 24, 96))[0], {}, None
    if name == "c5_jump27_24":         # config-5 analogue: 27-point jump coefficients
        return jump27(24), {}, None
    if name == "c3_aniso_2x2":
        return config_problem(3, grid=(24, 24, 24))[0], dict(pre_sweeps=2, post_sweeps=2), None
    if name == "unsmoothed_va4":        # 4 sweeps per level, unsmoothed
        return poisson7(32, 32, 32), dict(smooth_prolongator=0, sweeps_per_level=4), None
    if name == "random_w":              # non-constant w (PAPER.md:133 restriction of w)
        A = poisson7(20, 18, 17)
        return A, {}, 0.5 + uniform01(77, A.n_global)
    if name == "irregular_hubs":        # hub rows couple every rank with every rank
        return random_spd(5000, hubs=3), {}, None
    if name == "ragged_rows":           # np does not divide n; uneven blocks
        return poisson7(17, 13, 11), {}, None
    if name == "islands":               # disconnected + isolated rows interleaved; coarsening stalls
        return islands(), dict(max_coarse_size=20), None
    raise KeyError(name)


CASES = [("c4_32x32x64", 2), ("c4_32x32x64", 4), ("c4_24x24x96_np8", 8), ("c5_jump27_24", 3),
         ("c3_aniso_2x2", 2), ("unsmoothed_va4", 4), ("random_w", 3), ("irregular_hubs", 3), ("ragged_rows", 5),
         ("islands", 4)]


@pytest.mark.parametrize("name,nr", CASES)
def test_distributed_build_equals_single_process_build(name, nr):
    amg = _amg()
    A, kw, w = _case(name)
    cfg = amg.make_config(setup_device=0, **kw)
    Ls = _levels(_build(A, cfg, w))
    Ld = _levels(_build(A, cfg, w, nranks=nr))
    assert [L["n"] for L in Ls] == [L["n"] for L in Ld]
    for l, (a, b) in enumerate(zip(Ls, Ld)):
        assert a["omega"] == b["omega"], l
        for (rp, ci, v), (rp2, ci2, v2) in zip(a["mats"], b["mats"]):
            assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2), l
            assert np.array_equal(v.view(np.int64), v2.view(np.int64)), l   # bit for bit
        if a["agg"] is not None:
            assert np.array_equal(a["agg"], b["agg"]), l


@pytest.mark.parametrize("name,nr,rep", [("c4_32x32x64", 4, 0), ("c4_32x32x64", 2, 1 << 20),
                                         ("c5_jump27_24", 3, 0), ("irregular_hubs", 3, 1 << 16),
                                         ("c3_aniso_2x2", 2, 0), ("ragged_rows", 5, 0)])
def test_distributed_plans_equal_partition_of_the_single_build(name, nr, rep):
    amg = _amg()
    A, kw, w = _case(name)
    cfg = amg.make_config(setup_device=0, **kw)
    hs = _build(A, cfg, w)
    n = A.n_global
    b = np.array([n * g // nr for g in range(nr + 1)], np.int64)
    amg.check(amg.lib.amg_host_partition(hs, nr, C.c_void_p(b.ctypes.data), rep), "partition")
    hd = _build(A, cfg, w, nranks=nr, rep=rep)
    nl = len(_levels(hs))
    Ps, Pd = _plans(hs, nr, nl), _plans(hd, nr, nl)
    for k, (x, y) in enumerate(zip(Ps, Pd)):
        for j, (p, q) in enumerate(zip(x, y)):
            assert np.array_equal(p.view(np.int64) if p.dtype == np.float64 else p,
                                  q.view(np.int64) if q.dtype == np.float64 else q), (k // nl, k % nl, j)


def test_distributed_build_rejects_bad_input():
    amg = _amg()
    A = poisson7(6, 6, 6)
    A.values = A.values.copy()
    A.values[1] = -2.0   # asymmetric
    with pytest.raises(amg.AmgError):
        _build(A, amg.make_config(setup_device=0), nranks=2)


# ------------------------------------------------------------ one process per rank (gloo)
def _gloo_rank(rank, world, port, q):
    """One rank of the distributed setup in its own process, the transport being
    torch.distributed all_to_all over gloo; compares its plan with partition() of the
    single-process build of the same matrix (each process builds that reference itself)."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        amg = _amg()
        A, kw, w = _case("c5_jump27_24")
        cfg = amg.make_config(setup_device=0, **kw)
        n = A.n_global
        b = [n * g // world for g in range(world + 1)]
        r0, r1 = b[rank], b[rank + 1]
        rp = np.ascontiguousarray(A.rowptr[r0:r1 + 1] - A.rowptr[r0], np.int64)
        ci = np.ascontiguousarray(A.colind[A.rowptr[r0]:A.rowptr[r1]], np.int64)
        v = np.ascontiguousarray(A.values[A.rowptr[r0]:A.rowptr[r1]], np.float64)
        state = {}

        def exchange(user, phase, sc, rc, sbuf, rbuf):
            try:
                if phase == 0:
                    send = torch.tensor([sc[k] for k in range(world)], dtype=torch.int64)
                    recv = torch.zeros(world, dtype=torch.int64)
                    dist.all_to_all_single(recv, send)
                    for k in range(world):
                        rc[k] = int(recv[k])
                    state["sc"], state["rc"] = send.tolist(), recv.tolist()
                else:
                    ns, nr = sum(state["sc"]), sum(state["rc"])
                    send = torch.frombuffer(C.string_at(sbuf, ns), dtype=torch.uint8) if ns else \
                        torch.zeros(0, dtype=torch.uint8)
                    recv = torch.zeros(nr, dtype=torch.uint8)
                    dist.all_to_all_single(recv, send, output_split_sizes=state["rc"],
                                           input_split_sizes=state["sc"])
                    if nr:
                        C.memmove(rbuf, recv.numpy().ctypes.data, nr)
                return 0
            except Exception as e:  # pragma: no cover - reported through the status code
                state["err"] = repr(e)
                return 1

        cb = amg._abi.EXCHANGE_FN(exchange)
        h = C.c_void_p()
        code = amg.lib.amg_host_dist_build_rank(n, r0, r1, C.c_void_p(rp.ctypes.data), C.c_void_p(ci.ctypes.data),
                                                C.c_void_p(v.ctypes.data), None, C.byref(cfg), world, rank, 0,
                                                C.cast(cb, C.c_void_p), None, C.byref(h))
        assert code == 0, (amg.amg_last_error(), state.get("err"))
        hs = _build(A, cfg)
        bb = np.array(b, np.int64)
        amg.check(amg.lib.amg_host_partition(hs, world, C.c_void_p(bb.ctypes.data), 0), "partition")
        nl = len(_levels(hs))
        mine = _plans_of_rank(h, rank, world, nl)
        ref = _plans_of_rank(hs, rank, world, nl)
        same = all(np.array_equal(p.view(np.int64) if p.dtype == np.float64 else p,
                                  r.view(np.int64) if r.dtype == np.float64 else r)
                   for x, y in zip(mine, ref) for p, r in zip(x, y))
        q.put((rank, same, nl))
    finally:
        dist.destroy_process_group()


def _plans_of_rank(h, r, nr, nl):
    return _plans_one(h, r, nr, nl)


def _plans_one(h, r, nr, nl):
    amg = _amg()
    out = []
    for l in range(nl):
        info = np.zeros(16, np.int64)
        amg.check(amg.lib.amg_host_plan_level(h, r, l, C.c_void_p(info.ctypes.data)), "plan level")
        rec = [info.copy()]
        win, comp, rst = info[7] - info[6], info[5] - info[4], info[9] - info[8]
        sizes = {0: nr + 1, 1: info[10], 2: nr + 1, 3: info[11], 4: comp + 1, 5: info[12], 6: info[12],
                 7: comp + 1, 8: info[13], 9: info[13], 10: rst + 1, 11: info[14], 12: info[14], 13: win}
        for which in range(14):
            if which in (7, 8, 9, 10, 11, 12) and l == nl - 1:
                continue
            dt = np.float64 if which in (6, 9, 12, 13) else np.int64
            a = np.zeros(max(1, int(sizes[which])), dt)
            amg.check(amg.lib.amg_host_plan_array(h, r, l, which, C.c_void_p(a.ctypes.data)), "plan array")
            rec.append(a)
        out.append(rec)
    return out


@pytest.mark.slow
def test_gloo_world2_distributed_setup_equals_partition():
    """Two processes (torch.distributed over gloo): each builds only its own rows and plan through
    amg_host_dist_build_rank; both plans equal partition() of the single-process build bit for bit."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[0] for r in res] == [0, 1] and all(r[1] for r in res) and res[0][2] >= 3
