"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star):
  * aggregate maps bit-exact at every level;
  * one preconditioner application on a seeded vector <= 1e-12 relative 2-norm;
  * PCG iterations equal or +-1;
  * x within 1e-8 relative, compared at EQUAL iteration counts (fixed-count mode,
    rtol = 0, maxit = min of the two natural counts; SURVEY.md §4 protocol).
"""
import os

import numpy as np
import pytest

import oracle as O
from inputs import config_problem, diagonal_spd, islands, jump27, poisson7, random_spd, uniform01, uniform_pm1

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

VCYCLE_TOL = 1e-12
X_TOL = 1e-8


def _amg():
    import paper_2006_16147_b200 as amg
    return amg


@pytest.fixture(scope="module")
def ctx():
    amg = _amg()
    c = amg.Context(device=0)
    yield c
    c.close()


def _cfg(**kw):
    return _amg().make_config(**kw) if kw else None


# name -> (A builder, b builder, oracle kwargs, library config kwargs)
def _case(name):
    if name == "c1":
        A, b, _ = config_problem(1)
        return A, b, {}, {}
    if name == "c2":
        A, b, _ = config_problem(2)
        return A, b, {}, {}
    if name == "c3_64":  # config-3 analogue: anisotropic, 2/2 sweeps
        A, b, _ = config_problem(3, grid=(64, 64, 64))
        kw = dict(pre_sweeps=2, post_sweeps=2)
        return A, b, kw, kw
    if name == "c4_64x64x128":  # config-4 analogue, 2-slab weak-scaling shape, maxsize 200*2
        A, b, _ = config_problem(4, grid=(64, 64, 128))
        kw = dict(max_coarse_size=400)
        return A, b, kw, kw
    if name == "c5_32":  # config-5 analogue: 27-point jump coefficients
        A = jump27(32)
        b = uniform01(5, A.n_global)
        return A, b, {}, {}
    if name == "ragged_17x13x11":
        A = poisson7(17, 13, 11)
        b = uniform_pm1(7, A.n_global)
        return A, b, {}, {}
    if name == "unsmoothed_24":
        A = poisson7(24, 24, 24)
        b = np.ones(A.n_global)
        kw = dict(smooth_prolongator=0)
        return A, b, kw, kw
    if name == "omega_text_32":  # reading R3 alternative: omega = 1/||D^-1 A||
        A = poisson7(32, 32, 32)
        b = np.ones(A.n_global)
        kw = dict(prol_omega_scale=1.0)
        return A, b, kw, kw
    if name == "single_level":
        A = poisson7(5, 4, 3)
        b = uniform01(3, A.n_global)
        return A, b, {}, {}
    if name == "irregular_hubs":  # ragged rows (3..312 entries), CSR-vector at every level
        A = random_spd(20000, hubs=4)
        return A, uniform_pm1(21, A.n_global), {}, {}
    if name == "irregular_narrow":
        A = random_spd(3000, deg=3, window=5)
        return A, uniform01(22, A.n_global), {}, {}
    if name == "line_1d_100k":  # 1-D chain; level 0 in SDIA (offsets -1, 0, 1)
        A = poisson7(100000, 1, 1)
        return A, uniform01(23, A.n_global), {}, {}
    if name == "plane_2d_300":  # 2-D 5-point; level 0 in SDIA
        A = poisson7(300, 300, 1)
        return A, uniform_pm1(24, A.n_global), {}, {}
    if name == "diagonal":  # no couplings: single level, dense coarsest
        A = diagonal_spd(1000)
        return A, uniform01(25, A.n_global), {}, {}
    if name == "c5_72":  # ragged P-bar_0 (irregular aggregates, 8.5 entries/row) -> SELL-32-sigma
        A = jump27(72)
        return A, uniform01(26, A.n_global), {}, {}
    if name == "irregular_400k":  # ragged short rows, n >= 148 x 2048 -> SELL-32-sigma at level 0
        A = random_spd(400000, deg=4, window=32)
        return A, uniform_pm1(27, A.n_global), {}, {}
    if name == "n1":
        A = diagonal_spd(1)
        return A, np.array([3.0]), {}, {}
    if name == "va4_48":  # VA4: 4 matching sweeps per level (aggregates <= 16), smoothed P
        A = poisson7(48, 48, 48)
        kw = dict(sweeps_per_level=4)
        return A, uniform01(28, A.n_global), kw, kw
    if name == "islands":  # disconnected components + isolated rows, interleaved; coarsening stalls
        A = islands()
        kw = dict(max_coarse_size=20)
        return A, uniform01(29, A.n_global), kw, kw
    if name == "pair_mcs1":  # 2 rows, max_coarse_size 1: a 1-row coarsest level
        A = poisson7(2, 1, 1)
        kw = dict(max_coarse_size=1)
        return A, np.array([1.0, -3.0]), kw, kw
    raise KeyError(name)


CASES = ["c1", "c2", "c3_64", "c4_64x64x128", "c5_32", "ragged_17x13x11", "unsmoothed_24",
         "omega_text_32", "single_level", "irregular_hubs", "irregular_narrow", "line_1d_100k",
         "plane_2d_300", "diagonal", "n1", "c5_72", "irregular_400k", "va4_48", "islands", "pair_mcs1"]
_cache = {}


def _built(ctx, name):
    if name not in _cache:
        A, b, okw, lkw = _case(name)
        ho = O.OracleHierarchy(A, **okw)
        h = _amg().Hierarchy(ctx, A, cfg=_cfg(**lkw))
        _cache.clear()
        _cache[name] = (A, b, ho, h)
    return _cache[name]


@pytest.mark.parametrize("name", CASES)
def test_hierarchy_and_aggregates_bit_exact(ctx, name):
    A, b, ho, h = _built(ctx, name)
    if name == "irregular_400k":  # the ragged level-0 operator takes the row-sorted SELL layout
        assert h.level_info(0)["format"] == "sell32_sigma"
    assert h.sizes() == ho.sizes()
    for l in range(h.nlevels):
        info = h.level_info(l)
        assert info["nnzA"] == ho.nnz(l)
    for l in range(h.nlevels - 1):
        assert np.array_equal(h.level_aggregates(l), ho.agg(l)), f"level {l}"
    rep = h.report()
    assert rep["opc"] == pytest.approx(ho.opc, rel=1e-15)


@pytest.mark.parametrize("name", CASES)
def test_vcycle_parity(ctx, name):
    A, b, ho, h = _built(ctx, name)
    r = uniform_pm1(1000 + len(name), A.n_global)  # seeded parity vector (R17)
    z = h.precond_apply(torch.tensor(r, device="cuda:0")).cpu().numpy()
    zo = ho.vcycle(r)
    rel = np.linalg.norm(z - zo) / np.linalg.norm(zo)
    assert rel <= VCYCLE_TOL, rel


@pytest.mark.parametrize("name", CASES)
def test_pcg_parity(ctx, name):
    A, b, ho, h = _built(ctx, name)
    bt = torch.tensor(b, device="cuda:0")
    x, rep = h.solve(bt, rtol=1e-6, maxit=500)
    xo, info = ho.pcg(b, rtol=1e-6, maxit=500)
    assert rep["converged"] == 1 and info["status"] == O.OR_OK
    assert abs(rep["iterations"] - info["iterations"]) <= 1, (rep["iterations"], info["iterations"])
    assert rep["final_relres"] <= 1e-6
    k = min(rep["iterations"], info["iterations"])
    x, rep2 = h.solve(bt, rtol=0.0, maxit=k)
    assert rep2["iterations"] == k
    xo, _ = ho.pcg(b, rtol=0.0, maxit=k)
    rel = np.linalg.norm(x.cpu().numpy() - xo) / np.linalg.norm(xo)
    assert rel <= X_TOL, rel


def test_pcg_edge_cases(ctx):
    amg = _amg()
    A = poisson7(12, 10, 9)
    h = amg.Hierarchy(ctx, A)
    n = A.n_global
    # b = 0 -> x = 0 after 0 iterations
    x, rep = h.solve(torch.zeros(n, dtype=torch.float64, device="cuda:0"))
    assert rep["iterations"] == 0 and rep["converged"] == 1 and not x.any()
    b = torch.tensor(uniform01(11, n), device="cuda:0")
    # maxit = 0 -> not converged, x = 0
    x, rep = h.solve(b, rtol=1e-6, maxit=0)
    assert rep["iterations"] == 0 and rep["converged"] == 0 and not x.any()
    # rtol = 0 runs exactly maxit iterations
    x, rep = h.solve(b, rtol=0.0, maxit=7)
    assert rep["iterations"] == 7 and rep["converged"] == 0
    # determinism: bitwise identical repeats
    x1, _ = h.solve(b, rtol=1e-8)
    x2, _ = h.solve(b, rtol=1e-8)
    assert torch.equal(x1, x2)
    # host-buffer entry point == device entry point
    xh, reph = h.solve_host(b.cpu().numpy(), rtol=1e-8)
    assert np.array_equal(xh, x1.cpu().numpy())


def test_eager_launches_equal_graph(ctx):
    amg = _amg()
    A = poisson7(20, 18, 16)
    b = torch.tensor(uniform01(12, A.n_global), device="cuda:0")
    hg = amg.Hierarchy(ctx, A)
    he = amg.Hierarchy(ctx, A, cfg=amg.make_config(use_graphs=0))
    xg, rg = hg.solve(b)
    xe, re_ = he.solve(b)
    assert rg["iterations"] == re_["iterations"]
    assert torch.equal(xg, xe)
    assert torch.equal(hg.precond_apply(b), he.precond_apply(b))


def test_build_errors(ctx):
    amg = _amg()
    A = poisson7(4, 4, 4)
    A.values = A.values.copy()
    A.values[1] = -2.0  # breaks symmetry
    with pytest.raises(amg.AmgError) as e:
        amg.Hierarchy(ctx, A)
    assert e.value.code == 1
    A = poisson7(4, 4, 4)
    A.values = -A.values  # negative diagonal
    with pytest.raises(amg.AmgError) as e:
        amg.Hierarchy(ctx, A)
    assert e.value.code == 2


def test_vcycle_properties_full_c4(ctx):
    """BASELINE config 4 at its full per-GPU size (256^3), in the configuration
    bench.py times: level-0 aggregates equal the closed-form 2x2x2 cubes (pin P4),
    the device V-cycle is linear and symmetric, and PCG converges with a true
    residual at the requested tolerance."""
    amg = _amg()
    A, b, meta = config_problem(4)
    h = amg.Hierarchy(ctx, A)
    nx = 256
    i = np.arange(A.n_global)
    x, y, z = i % nx, (i // nx) % nx, i // (nx * nx)
    cube = x // 2 + (nx // 2) * (y // 2 + (nx // 2) * (z // 2))
    assert np.array_equal(h.level_aggregates(0), cube)
    g = torch.Generator(device="cpu").manual_seed(5)
    r = torch.rand(A.n_global, generator=g, dtype=torch.float64).cuda()
    s = torch.rand(A.n_global, generator=g, dtype=torch.float64).cuda()
    Br, Bs = h.precond_apply(r).clone(), h.precond_apply(s).clone()
    lin = h.precond_apply(2.0 * r - 3.0 * s)
    assert (torch.linalg.norm(lin - (2.0 * Br - 3.0 * Bs)) / torch.linalg.norm(lin)).item() <= 1e-12
    sym = abs(torch.dot(Br, s) - torch.dot(r, Bs)).item()
    assert sym <= 1e-12 * torch.linalg.norm(r).item() * torch.linalg.norm(s).item()
    assert torch.dot(r, Br).item() > 0
    bt = torch.tensor(b, device="cuda:0")
    xs, rep = h.solve(bt, rtol=1e-6)
    assert rep["converged"] == 1
    Asp = torch.sparse_csr_tensor(torch.tensor(A.rowptr), torch.tensor(A.colind), torch.tensor(A.values),
                                  size=(A.n_global, A.n_global)).cuda()
    res = bt - (Asp @ xs.unsqueeze(1)).squeeze(1)
    assert (torch.linalg.norm(res) / torch.linalg.norm(bt)).item() <= 1.5e-6


def test_full_c3_anisotropic_properties(ctx):
    """BASELINE config 3 at full size (256^3, (1,1,1e-2), 2/2 sweeps) as bench.py
    --config 3 runs it: level-0 aggregates are the closed-form 4x2x1 bricks (pin P16),
    the device V-cycle is linear and symmetric, PCG converges with the true residual
    at the requested tolerance."""
    amg = _amg()
    A, b, meta = config_problem(3)
    h = amg.Hierarchy(ctx, A, cfg=amg.make_config(pre_sweeps=2, post_sweeps=2))
    nx = 256
    i = np.arange(A.n_global)
    x, y, z = i % nx, (i // nx) % nx, i // (nx * nx)
    brick = x // 4 + (nx // 4) * (y // 2 + (nx // 2) * z)
    assert np.array_equal(h.level_aggregates(0), brick)
    g = torch.Generator(device="cpu").manual_seed(6)
    r = torch.rand(A.n_global, generator=g, dtype=torch.float64).cuda()
    s = torch.rand(A.n_global, generator=g, dtype=torch.float64).cuda()
    Br, Bs = h.precond_apply(r).clone(), h.precond_apply(s).clone()
    lin = h.precond_apply(0.5 * r + 2.0 * s)
    assert (torch.linalg.norm(lin - (0.5 * Br + 2.0 * Bs)) / torch.linalg.norm(lin)).item() <= 1e-12
    sym = abs(torch.dot(Br, s) - torch.dot(r, Bs)).item()
    assert sym <= 1e-12 * torch.linalg.norm(r).item() * torch.linalg.norm(s).item()
    bt = torch.tensor(b, device="cuda:0")
    xs, rep = h.solve(bt, rtol=1e-6)
    assert rep["converged"] == 1
    Asp = torch.sparse_csr_tensor(torch.tensor(A.rowptr), torch.tensor(A.colind), torch.tensor(A.values),
                                  size=(A.n_global, A.n_global)).cuda()
    res = bt - (Asp @ xs.unsqueeze(1)).squeeze(1)
    assert (torch.linalg.norm(res) / torch.linalg.norm(bt)).item() <= 1.5e-6


def _full_size_parity(h, ho, A, b, seed, threads=1):
    """V-cycle <= 1e-12; PCG iterations +-1; x <= 1e-8 at equal counts.  threads > 1 runs the
    oracle's solve with its OpenMP row loops (only the dot summation order differs)."""
    r = uniform_pm1(seed, A.n_global)
    z = h.precond_apply(torch.tensor(r, device="cuda:0")).cpu().numpy()
    zo = ho.vcycle(r)
    rel = np.linalg.norm(z - zo) / np.linalg.norm(zo)
    assert rel <= VCYCLE_TOL, rel
    bt = torch.tensor(b, device="cuda:0")
    x, rep = h.solve(bt, rtol=1e-6)
    O.OracleHierarchy.set_threads(threads)
    try:
        xo, info = ho.pcg(b, rtol=1e-6)
        assert rep["converged"] == 1 and info["status"] == O.OR_OK
        assert abs(rep["iterations"] - info["iterations"]) <= 1, (rep["iterations"], info["iterations"])
        k = min(rep["iterations"], info["iterations"])
        x, _ = h.solve(bt, rtol=0.0, maxit=k)
        if k != info["iterations"]:
            xo, _ = ho.pcg(b, rtol=0.0, maxit=k)
    finally:
        O.OracleHierarchy.set_threads(1)
    relx = np.linalg.norm(x.cpu().numpy() - xo) / np.linalg.norm(xo)
    assert relx <= X_TOL, relx


def test_full_c4_hierarchy_vcycle_and_pcg_vs_oracle(ctx):
    """BASELINE config 4 at full size (256^3) exactly as bench.py builds and solves it (GPU
    setup, default config): every level's aggregate map equals the oracle's bit for bit, one
    V-cycle agrees to 1e-12, the PCG iteration counts agree +-1 and x agrees to 1e-8 at equal
    iteration counts (the oracle runs single-threaded: the sequential parity reference)."""
    amg = _amg()
    A, b, meta = config_problem(4)
    h = amg.Hierarchy(ctx, A)
    ho = O.OracleHierarchy(A)
    assert h.sizes() == ho.sizes()
    for l in range(h.nlevels - 1):
        assert np.array_equal(h.level_aggregates(l), ho.agg(l)), f"level {l}"
    _full_size_parity(h, ho, A, b, 1004)


def test_full_c3_hierarchy_vcycle_and_pcg_vs_oracle(ctx):
    """BASELINE config 3 at full size (256^3 anisotropic, 2/2 sweeps) as bench.py --config 3
    runs it: aggregates bit-exact, V-cycle <= 1e-12, iterations +-1, x <= 1e-8 at equal counts.
    The oracle's solve uses its OpenMP row loops here to bound the test's time."""
    amg = _amg()
    A, b, meta = config_problem(3)
    kw = dict(pre_sweeps=2, post_sweeps=2)
    h = amg.Hierarchy(ctx, A, cfg=amg.make_config(**kw))
    ho = O.OracleHierarchy(A, **kw)
    assert h.sizes() == ho.sizes()
    for l in range(h.nlevels - 1):
        assert np.array_equal(h.level_aggregates(l), ho.agg(l)), f"level {l}"
    _full_size_parity(h, ho, A, b, 1003, threads=os.cpu_count() or 1)


def test_breakdown_on_an_indefinite_matrix(ctx):
    """O11 / SPEC.md:468: p^T A p <= 0 stops PCG with AMG_ERR_BREAKDOWN (x = the last
    iterate).  tridiag(1.5, 2, 1.5) has a positive diagonal (the build accepts it; its
    Galerkin coarse operators are s.p.d.) but eigenvalues 2 + 3 cos(k pi/(n+1)) of both signs;
    the oracle breaks down at the same iteration."""
    import ctypes as C
    import scipy.sparse as sp
    from inputs.problems import CSR
    amg = _amg()
    n = 1000
    M = sp.diags([1.5 * np.ones(n - 1), 2.0 * np.ones(n), 1.5 * np.ones(n - 1)], [-1, 0, 1]).tocsr()
    A = CSR(n_global=n, row_begin=0, row_end=n, rowptr=M.indptr.astype(np.int64),
            colind=M.indices.astype(np.int64), values=M.data.astype(np.float64))
    b = np.ones(n)
    ho = O.OracleHierarchy(A, max_coarse_size=10)
    xo, info = ho.pcg(b, rtol=1e-8, maxit=100)
    assert info["status"] == O.OR_BREAKDOWN
    for graphs in (1, 0):
        h = amg.Hierarchy(ctx, A, cfg=amg.make_config(max_coarse_size=10, use_graphs=graphs))
        bt = torch.tensor(b, device="cuda:0")
        x = torch.empty_like(bt)
        rep = amg.amg_report_t()
        code = amg.lib.amg_solve(h.h, C.c_void_p(bt.data_ptr()), C.c_void_p(x.data_ptr()), 1e-8, 100,
                                 C.byref(rep))
        assert code == amg.AMG_ERR_BREAKDOWN and rep.status == amg.AMG_ERR_BREAKDOWN
        assert rep.iterations == info["iterations"] and rep.converged == 0
        assert np.linalg.norm(x.cpu().numpy() - xo) <= 1e-10 * np.linalg.norm(xo)
        with pytest.raises(amg.AmgError) as e:
            h.solve(bt, rtol=1e-8, maxit=100)
        assert e.value.code == amg.AMG_ERR_BREAKDOWN


def test_compact_and_collapsed_levels_are_taken(ctx):
    """c2's deep levels run in the compact form (S2(b) on the second stream, Rc restriction,
    Pc prolongation+post) and the level above the coarsest as one dense GEMV; the parity cases
    above check their numbers against the oracle, this checks the paths are actually used."""
    amg = _amg()
    A, b, _ = config_problem(2)
    ho2 = O.OracleHierarchy(A)
    r2 = uniform_pm1(4243, A.n_global)
    zo2 = ho2.vcycle(r2)
    # forced second collapse: the compact 4147-row level above the collapsed 522-row level becomes
    # one dense GEMV for the whole cycle below level 2 (by default c2 keeps it compact: the dense
    # operator would move 3x the bytes)
    os.environ["AMG_FORCE_COLLAPSE2"] = "1"
    try:
        h = amg.Hierarchy(ctx, A)
    finally:
        os.environ.pop("AMG_FORCE_COLLAPSE2", None)
    names = [k["name"] for k in h.profile_vcycle(1)]
    assert names.count("collapsed") == 1 and "coarse_gemv" not in names and "restrict_c" not in names, names
    z = h.precond_apply(torch.tensor(r2, device="cuda:0")).cpu().numpy()
    assert np.linalg.norm(z - zo2) / np.linalg.norm(zo2) <= VCYCLE_TOL
    # default (byte rule): the compact level runs its three kernels
    h = amg.Hierarchy(ctx, A)
    names = [k["name"] for k in h.profile_vcycle(1)]
    assert "collapsed" in names and "restrict_c" in names and "sweep0_c" in names
    assert names.count("collapsed") == 1 and "coarse_gemv" not in names
    z = h.precond_apply(torch.tensor(r2, device="cuda:0")).cpu().numpy()
    assert np.linalg.norm(z - zo2) / np.linalg.norm(zo2) <= VCYCLE_TOL
    # and 2/2 sweeps collapse too (general dense level operator)
    A3 = poisson7(32, 32, 32, (1.0, 1.0, 0.01))
    h3 = amg.Hierarchy(ctx, A3, cfg=amg.make_config(pre_sweeps=2, post_sweeps=2))
    ho = O.OracleHierarchy(A3, pre_sweeps=2, post_sweeps=2)
    assert "collapsed" in [k["name"] for k in h3.profile_vcycle(1)]
    r = uniform_pm1(4242, A3.n_global)
    z = h3.precond_apply(torch.tensor(r, device="cuda:0")).cpu().numpy()
    zo = ho.vcycle(r)
    assert np.linalg.norm(z - zo) / np.linalg.norm(zo) <= VCYCLE_TOL


@pytest.mark.parametrize("name", ["c2", "c5_72", "islands"])
def test_16bit_columns_bitwise_equal_to_32bit(ctx, name):
    """Operators whose rows span < 2^16 columns store 16-bit column offsets from a per-row (per
    SELL slot) base instead of int32 columns: the same entries in the same order, so the V-cycle
    and the PCG iterates are bitwise equal to the 32-bit form (AMG_NO_C16=1), with fewer bytes."""
    amg = _amg()
    A, b, _, lkw = _case(name)
    h16 = amg.Hierarchy(ctx, A, cfg=_cfg(**lkw))
    os.environ["AMG_NO_C16"] = "1"
    try:
        h32 = amg.Hierarchy(ctx, A, cfg=_cfg(**lkw))
    finally:
        os.environ.pop("AMG_NO_C16", None)
    p16, p32 = h16.profile_vcycle(1), h32.profile_vcycle(1)
    assert [k["name"] for k in p16] == [k["name"] for k in p32]
    s16, s32 = sum(k["stored_bytes"] for k in p16), sum(k["stored_bytes"] for k in p32)
    assert s16 < s32, (s16, s32)
    r = torch.tensor(uniform_pm1(77, A.n_global), device="cuda:0")
    assert torch.equal(h16.precond_apply(r), h32.precond_apply(r))
    bt = torch.tensor(b, device="cuda:0")
    x16, r16 = h16.solve(bt, rtol=1e-8)
    x32, r32 = h32.solve(bt, rtol=1e-8)
    assert r16["iterations"] == r32["iterations"] and torch.equal(x16, x32)


def test_solve_host_batch_equals_single_solves(ctx):
    """amg_solve_host_batch (copies pipelined with the solves over two device buffer pairs)
    returns exactly the solutions and reports of one amg_solve_host per right-hand side."""
    amg = _amg()
    A, _, _ = config_problem(2)
    h = amg.Hierarchy(ctx, A)
    n = A.n_global
    B = np.stack([uniform01(300 + k, n) for k in range(5)])
    B[3] = 0.0  # a zero right-hand side inside the batch
    Bp = torch.tensor(B).pin_memory().numpy()
    Xp = torch.empty(B.shape, dtype=torch.float64).pin_memory().numpy()
    X, reps = h.solve_host_batch(Bp, Xp, rtol=1e-6)
    for k in range(B.shape[0]):
        xk, rk = h.solve_host(B[k].copy(), rtol=1e-6)
        assert np.array_equal(X[k], xk), k
        assert reps[k]["iterations"] == rk["iterations"] and reps[k]["converged"] == rk["converged"]
    assert reps[3]["iterations"] == 0 and not X[3].any()
    # pageable buffers: same results
    X2, _ = h.solve_host_batch(B.copy(), rtol=1e-6)
    assert np.array_equal(X2, X)


def test_repeated_builds_are_bitwise_identical(ctx):
    """Builds of the same matrix in one process give the same solve bit for bit (round 2 found a
    build-to-build race: device buffers zeroed by a synchronous-API memset on the legacy default
    stream were written by the next kernel on the context's non-blocking stream; ~1 build in 10 of
    the c5 256^3 analogue then had a corrupt SELL-32-sigma slot map, profiles/r02_race_legacy_stream_fix.txt).
    The 27-point jump operator at 96^3 takes the SELL-32-sigma path on level 1."""
    import hashlib
    import paper_2006_16147_b200 as amg
    A = jump27(96)
    b = uniform01(5, A.n_global)
    bt = torch.tensor(b, device="cuda:0")
    ref = None
    for _ in range(4):
        h = amg.Hierarchy(ctx, A)
        x, rep = h.solve(bt)
        got = (rep["iterations"], hashlib.sha1(x.cpu().numpy().tobytes()).hexdigest())
        ref = ref or got
        assert got == ref
        h.close()
