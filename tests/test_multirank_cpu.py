"""Multi-rank host logic on CPU (SURVEY.md §4 layer 4; §8e).

* The partition plan built by the library (amg_host_partition): owned blocks per
  level follow the minimum-member rule (R18), local operators are exact row
  slices of the global ones in the window frame, halo lists are exactly the
  referenced non-owned ids, and send lists mirror the peers' receive lists.
* A world-size-2 `gloo` run executes the distributed V-cycle schedule of the
  CUDA path (the same exchange points: input halo, residual halo before the
  restriction, coarse-correction halo before the prolongation, x halo before each
  post-sweep, gather at the first replicated level) with numpy local operators
  and torch.distributed send/recv, and compares the result with the oracle's
  V-cycle.  This checks the plan and the exchange schedule; the GPU kernels of
  the same schedule are checked in tests/test_gpu_multirank.py (loopback).
"""
import ctypes as C
import os

import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O
from inputs import jump27, poisson7, uniform_pm1


def _amg():
    import paper_2006_16147_b200 as amg
    return amg


class Plan:
    def __init__(self, A, np_, bounds=None, rep_bytes=64 << 20, **cfg):
        amg = _amg()
        self.L = amg.lib
        c = amg.make_config(**dict({"setup_device": 0}, **cfg))  # host build (CPU box)
        self.keep = [np.ascontiguousarray(A.rowptr, np.int64), np.ascontiguousarray(A.colind, np.int64),
                     np.ascontiguousarray(A.values, np.float64)]
        self.h = C.c_void_p()
        code = self.L.amg_host_hierarchy_build(A.n_global, *[C.c_void_p(a.ctypes.data) for a in self.keep], None,
                                               C.byref(c), C.byref(self.h))
        assert code == 0, amg.amg_last_error()
        n = A.n_global
        if bounds is None:
            bounds = [n * g // np_ for g in range(np_ + 1)]
        self.bounds = np.array(bounds, np.int64)
        self.code = self.L.amg_host_partition(self.h, np_, C.c_void_p(self.bounds.ctypes.data), rep_bytes)
        self.np = np_
        nl = C.c_int32()
        self.L.amg_host_num_levels(self.h, C.byref(nl))
        self.nl = nl.value

    def __del__(self):
        if self.h:
            self.L.amg_host_hierarchy_destroy(self.h)

    def info(self, g, l):
        a = np.zeros(16, np.int64)
        assert self.L.amg_host_plan_level(self.h, g, l, C.c_void_p(a.ctypes.data)) == 0
        keys = ["replicated", "n", "own_begin", "own_end", "comp_begin", "comp_end", "win_begin", "win_end",
                "rst_begin", "rst_end", "n_recv", "n_send", "nnzA", "nnzP", "nnzR"]
        return dict(zip(keys, [int(v) for v in a[:15]]))

    def arr(self, g, l, which, n, dtype=np.int64):
        out = np.zeros(max(n, 1), dtype)
        assert self.L.amg_host_plan_array(self.h, g, l, which, C.c_void_p(out.ctypes.data)) == 0
        return out[:n]

    def local_ops(self, g, l):
        I = self.info(g, l)
        ops = {}
        nrows = {"A": I["comp_end"] - I["comp_begin"], "P": I["comp_end"] - I["comp_begin"],
                 "R": I["rst_end"] - I["rst_begin"]}
        for name, base, nnz in (("A", 4, I["nnzA"]), ("P", 7, I["nnzP"]), ("R", 10, I["nnzR"])):
            if name != "A" and l == self.nl - 1:
                continue
            rp = self.arr(g, l, base, nrows[name] + 1)
            ci = self.arr(g, l, base + 1, nnz)
            v = self.arr(g, l, base + 2, nnz, np.float64)
            ops[name] = (rp, ci, v)
        ops["m"] = self.arr(g, l, 13, I["win_end"] - I["win_begin"], np.float64)
        ops["recv_off"] = self.arr(g, l, 0, self.np + 1)
        ops["recv_ids"] = self.arr(g, l, 1, I["n_recv"])
        ops["send_off"] = self.arr(g, l, 2, self.np + 1)
        ops["send_ids"] = self.arr(g, l, 3, I["n_send"])
        return I, ops


def _csr(rp, ci, v, ncols):
    return sp.csr_matrix((v, ci, rp), shape=(len(rp) - 1, ncols))


CASES = {
    "c4_like_slabs": lambda: poisson7(16, 16, 32),
    "aniso": lambda: poisson7(16, 16, 16, (1, 1, 0.01)),
    "jump27": lambda: jump27(16),
}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("np_", [2, 3, 4])
def test_partition_plan_invariants(case, np_):
    A = CASES[case]()
    P = Plan(A, np_, max_coarse_size=40)
    assert P.code == 0
    ho = O.OracleHierarchy(A, max_coarse_size=40)
    assert ho.nlevels == P.nl
    for l in range(P.nl):
        # owned blocks partition [0, n_l)
        infos = [P.info(g, l) for g in range(np_)]
        assert infos[0]["own_begin"] == 0 and infos[-1]["own_end"] == ho.level_n(l)
        for a, b in zip(infos, infos[1:]):
            assert a["own_end"] == b["own_begin"]
        if l > 0:  # coarse owner = owner of the aggregate's minimum member (R18)
            agg = ho.agg(l - 1)
            first = np.full(ho.level_n(l), -1)
            for i in range(len(agg) - 1, -1, -1):
                first[agg[i]] = i
            prev = [P.info(g, l - 1) for g in range(np_)]
            for g in range(np_):
                for G in (infos[g]["own_begin"], infos[g]["own_end"] - 1):
                    if infos[g]["own_begin"] < infos[g]["own_end"]:
                        assert prev[g]["own_begin"] <= first[G] < prev[g]["own_end"]
        Ag = ho.A(l).to_scipy()
        Pg = ho.P(l).to_scipy() if l + 1 < P.nl else None
        for g in range(np_):
            I, ops = P.local_ops(g, l)
            wb, we = I["win_begin"], I["win_end"]
            # local A = global rows, columns in the window frame
            rp, ci, v = ops["A"]
            loc = _csr(rp, ci + wb, v, ho.level_n(l))
            assert (loc != Ag[I["comp_begin"]:I["comp_end"]]).nnz == 0
            referenced = set((ci + wb).tolist())
            if Pg is not None:
                I1 = P.info(g, l + 1)
                rp, ci, v = ops["P"]
                assert (_csr(rp, ci + I1["win_begin"], v, ho.level_n(l + 1)) != Pg[I["comp_begin"]:I["comp_end"]]).nnz == 0
                rp, ci, v = ops["R"]
                Rg = Pg.T.tocsr()
                assert (_csr(rp, ci + wb, v, ho.level_n(l)) != Rg[I["rst_begin"]:I["rst_end"]]).nnz == 0
                referenced |= set((ci + wb).tolist())
            if l > 0 and not I["replicated"]:
                Ip = P.info(g, l - 1)
                _, opsp = P.local_ops(g, l - 1)
                rp, ci, v = opsp["P"]
                referenced |= set((ci + wb).tolist())
            assert min(referenced) >= wb and max(referenced) < we
            own = set(range(I["own_begin"], I["own_end"]))
            if not I["replicated"]:
                assert set(ops["recv_ids"].tolist()) == referenced - own
            # send lists mirror the peers' receive lists
            for q in range(np_):
                Iq, opsq = P.local_ops(q, l)
                mine = ops["send_ids"][ops["send_off"][q]:ops["send_off"][q + 1]]
                theirs = opsq["recv_ids"][opsq["recv_off"][g]:opsq["recv_off"][g + 1]]
                assert np.array_equal(mine, theirs)
                assert all(I["own_begin"] <= x < I["own_end"] for x in mine)
            assert np.array_equal(ops["m"], ho.m(l)[wb:we])


def test_partition_rejects_bad_blocks():
    A = poisson7(8, 8, 8)
    assert Plan(A, 2, bounds=[0, 300, 200]).code != 0
    assert Plan(A, 2, bounds=[0, 100, 500]).code != 0


# ------------------------------------------------------------ gloo V-cycle
def _dist_vcycle(rank, world, port, q):
    """Distributed V-cycle (s1 = s2 = 1) with gloo halo exchanges, numpy local ops."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = poisson7(16, 16, 24)
        P = Plan(A, world, max_coarse_size=30, rep_bytes=0)
        nl = P.nl
        lv = [P.local_ops(rank, l) for l in range(nl)]
        Ls = []
        for l, (I, ops) in enumerate(lv):
            d = dict(I=I, ops=ops, win=I["win_end"] - I["win_begin"])
            if "A" in ops:
                d["A"] = _csr(*ops["A"], d["win"])
            if l + 1 < nl:
                d["P"] = _csr(*ops["P"], lv[l + 1][0]["win_end"] - lv[l + 1][0]["win_begin"])
                d["R"] = _csr(*ops["R"], d["win"])
            Ls.append(d)

        def exch(l, vec):
            d = Ls[l]
            I, ops = d["I"], d["ops"]
            wb = I["win_begin"]
            reqs = []
            for peer in range(world):
                if peer == rank:
                    continue
                s0, s1 = ops["send_off"][peer], ops["send_off"][peer + 1]
                r0, r1 = ops["recv_off"][peer], ops["recv_off"][peer + 1]
                if s1 > s0:
                    buf = torch.tensor(vec[ops["send_ids"][s0:s1] - wb])
                    reqs.append(dist.isend(buf, peer))
                if r1 > r0:
                    rb = torch.zeros(r1 - r0, dtype=torch.float64)
                    reqs.append((dist.irecv(rb, peer), rb, r0, r1))
            for rq in reqs:
                if isinstance(rq, tuple):
                    rq[0].wait()
                    vec[ops["recv_ids"][rq[2]:rq[3]] - wb] = rq[1].numpy()
                else:
                    rq.wait()

        n0 = A.n_global
        rglob = uniform_pm1(77, n0)
        # level-0 input in its window (owned part), everything else filled by halos
        vec = {}
        for l, d in enumerate(Ls):
            d["b"] = np.zeros(d["win"])
            d["x"] = np.zeros(d["win"])
        I0 = Ls[0]["I"]
        Ls[0]["b"][I0["own_begin"] - I0["win_begin"]:I0["own_end"] - I0["win_begin"]] = \
            rglob[I0["own_begin"]:I0["own_end"]]
        for l in range(nl - 1):
            d = Ls[l]
            I = d["I"]
            e0 = I["comp_begin"] - I["win_begin"]
            ne = I["comp_end"] - I["comp_begin"]
            m = d["ops"]["m"]
            if not I["replicated"]:
                exch(l, d["b"])
            mb = m * d["b"]
            r = np.zeros(d["win"])
            r[e0:e0 + ne] = d["b"][e0:e0 + ne] - d["A"] @ mb
            if not I["replicated"]:
                exch(l, r)
            C_ = Ls[l + 1]
            IC = C_["I"]
            ro = I["rst_begin"] - IC["win_begin"]
            C_["b"][ro:ro + (I["rst_end"] - I["rst_begin"])] = d["R"] @ r
            if IC["replicated"] and not I["replicated"]:
                exch(l + 1, C_["b"])
            d["r"] = r
        # coarsest: dense solve of the replicated level
        Lc = Ls[nl - 1]
        Ac = _csr(*Lc["ops"]["A"], Lc["win"]).toarray()
        Lc["x"][:] = np.linalg.solve(Ac, Lc["b"])
        for l in range(nl - 2, -1, -1):
            d = Ls[l]
            I = d["I"]
            e0 = I["comp_begin"] - I["win_begin"]
            ne = I["comp_end"] - I["comp_begin"]
            C_ = Ls[l + 1]
            if not C_["I"]["replicated"]:
                exch(l + 1, C_["x"])
            m = d["ops"]["m"]
            x = np.zeros(d["win"])
            x[e0:e0 + ne] = (m * d["b"])[e0:e0 + ne] + d["P"] @ C_["x"]
            if not I["replicated"]:
                exch(l, x)
            x2 = np.zeros(d["win"])
            x2[e0:e0 + ne] = x[e0:e0 + ne] + m[e0:e0 + ne] * (d["b"][e0:e0 + ne] - d["A"] @ x)
            d["x"] = x2
        own = Ls[0]["x"][I0["own_begin"] - I0["win_begin"]:I0["own_end"] - I0["win_begin"]]
        q.put((rank, I0["own_begin"], own.copy(), [L["I"]["replicated"] for L in Ls]))
    finally:
        dist.destroy_process_group()


@pytest.mark.slow
def test_gloo_world2_distributed_vcycle_matches_oracle():
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_vcycle, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = poisson7(16, 16, 24)
    ho = O.OracleHierarchy(A, max_coarse_size=30)
    zo = ho.vcycle(uniform_pm1(77, A.n_global))
    z = np.zeros(A.n_global)
    for rank, ob, own, rep in res:
        z[ob:ob + len(own)] = own
        assert rep[0] == 0 and rep[-1] == 1  # level 0 distributed, coarsest replicated
    assert np.linalg.norm(z - zo) <= 1e-12 * np.linalg.norm(zo)
