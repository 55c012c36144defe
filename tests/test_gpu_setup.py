"""GPU-resident hierarchy setup (setup_gpu.cu) — bit-identical to
the host setup and to the oracle.

The GPU build uses its own algorithms (suitor matching with 64-bit atomicMax on packed
key ranks; expand-sort-compress SpGEMM with a stable radix sort and sequential run sums)
under the canonical arithmetic contract C1-C5, so every aggregate map, every coarse
operator A_l and every smoothed prolongator P-bar_l must equal the host build's bit for
bit, and the aggregate maps must equal the oracle's.
"""
import os
import time

import numpy as np
import pytest

import oracle as O
from inputs import config_problem, jump27, poisson7, random_spd, uniform01
from test_abi_cpu import HostH

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def amg():
    import paper_2006_16147_b200 as amg
    torch.cuda.init()
    return amg


def _case(name):
    if name == "c1":
        return config_problem(1)[0], None, {}
    if name == "c2_128":
        return config_problem(2)[0], None, {}
    if name == "aniso_48_2x2":
        return config_problem(3, grid=(48, 48, 48))[0], None, dict(pre_sweeps=2, post_sweeps=2)
    if name == "jump27_32":
        return jump27(32), None, {}
    if name == "ragged_17x13x11":
        return poisson7(17, 13, 11), None, {}
    if name == "unsmoothed_40":
        return poisson7(40, 40, 40), None, dict(smooth_prolongator=0)
    if name == "four_sweeps_48":
        return poisson7(48, 48, 48), None, dict(sweeps_per_level=4)
    if name == "random_w_24":
        A = poisson7(24, 24, 24)
        return A, 0.5 + uniform01(77, A.n_global), {}
    if name == "omega_text_32":
        return poisson7(32, 32, 32), None, dict(prol_omega_scale=1.0)
    if name == "maxsize_2400_64":
        return poisson7(64, 64, 64), None, dict(max_coarse_size=2400)
    # row-chunked expand-sort-compress SpGEMM (AMG_SPGEMM_CHUNK products per chunk):
    # hundreds of chunks at the level-0 Galerkin step, single rows over the budget
    if name == "c2_128_chunked":
        return config_problem(2)[0], None, {}
    if name == "jump27_48_chunked":
        return jump27(48), None, {}
    if name == "irregular_200k_chunked":
        return random_spd(200000, hubs=8), None, {}
    raise KeyError(name)


CHUNK = {"c2_128_chunked": 200000, "jump27_48_chunked": 100000, "irregular_200k_chunked": 150}

CASES = ["c1", "c2_128", "aniso_48_2x2", "jump27_32", "ragged_17x13x11", "unsmoothed_40", "four_sweeps_48",
         "random_w_24", "omega_text_32", "maxsize_2400_64", "c2_128_chunked", "jump27_48_chunked",
         "irregular_200k_chunked"]


def _same(a, b):
    return a.shape == b.shape and np.array_equal(a.view(np.int64), b.view(np.int64))


@pytest.mark.parametrize("name", CASES)
def test_gpu_setup_bit_identical_to_host_setup(amg, name):
    A, w, kw = _case(name)
    hh = HostH(amg, A, w=w, setup_device=0, **kw)
    if name in CHUNK:
        os.environ["AMG_SPGEMM_CHUNK"] = str(CHUNK[name])
    try:
        hg = HostH(amg, A, w=w, setup_device=1, **kw)
    finally:
        os.environ.pop("AMG_SPGEMM_CHUNK", None)
    assert hh.code == 0 and hg.code == 0, amg.amg_last_error()
    assert hg.nlevels == hh.nlevels
    for l in range(hh.nlevels):
        assert hg.sizes(l) == hh.sizes(l), l  # n, nnz(A_l), nnz(P-bar_l), omega (bitwise via ==)
        for which in ((0, 1) if l + 1 < hh.nlevels else (0,)):
            g, h = hg.matrix(l, which), hh.matrix(l, which)
            assert np.array_equal(g[0], h[0]) and np.array_equal(g[1], h[1]), (l, which)
            assert _same(g[2], h[2]), f"level {l} {'A' if which == 0 else 'P-bar'} values differ bitwise"
        if l + 1 < hh.nlevels:
            assert np.array_equal(hg.agg(l), hh.agg(l))
    if name in ("c1", "jump27_32", "random_w_24"):
        ho = O.OracleHierarchy(A, w=w, **kw)
        assert ho.nlevels == hg.nlevels
        for l in range(ho.nlevels - 1):
            assert np.array_equal(hg.agg(l), ho.agg(l))


def test_gpu_setup_solve_parity_and_speed(amg):
    """A GPU-built hierarchy solves exactly like the host-built one (bitwise equal x).  The
    build times are printed (not asserted: wall-clock comparisons on a shared box are noise)."""
    A, b, _ = config_problem(2)
    ctx = amg.Context(device=0)
    t0 = time.perf_counter()
    hh = amg.Hierarchy(ctx, A, cfg=amg.make_config(setup_device=0))
    th = time.perf_counter() - t0
    t0 = time.perf_counter()
    hg = amg.Hierarchy(ctx, A, cfg=amg.make_config(setup_device=1))
    tg = time.perf_counter() - t0
    bt = torch.tensor(b, device="cuda:0")
    xh, rh = hh.solve(bt, rtol=1e-6)
    xg, rg = hg.solve(bt, rtol=1e-6)
    assert rh["iterations"] == rg["iterations"] and torch.equal(xh, xg)
    print(f"setup c2: host {th:.2f} s, gpu {tg:.2f} s")
