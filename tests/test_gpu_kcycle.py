"""GPU parity of the K-cycle.

The coarse correction of every level whose coarse level is not the coarsest is two
FCG(1) iterations preconditioned by the cycle rooted there.  The CUDA path
(recursive graph of level kernels, inner FCG scalars kept on the device and every
dot fused into the kernel producing its operand) is compared with the oracle's
kcycle_fcg2 (oracle/oracle.c), itself pinned in tests/test_oracle_pins.py.

Bars: aggregates bit-exact; one K-cycle application within KC_TOL; FCG iterations
equal or +-1 and x within 1e-8 at equal iteration counts.
"""
import numpy as np
import pytest

import oracle as O
from inputs import config_problem, jump27, poisson7, uniform01, uniform_pm1

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

# The K-cycle is smooth in its input (no stop decisions besides p^T q > 0), so the
# only difference from the oracle is the summation order of fp64 dots and SpMV rows
# (~1e-16 relative per operation) propagated through 2^(nl-2) nested FCG steps.
KC_TOL = 1e-12
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


def _case(name):
    """name -> (A, b, hierarchy kwargs shared by oracle and library, library-only kwargs, coarse CG)"""
    K = dict(cycle=1, krylov=1)
    if name == "ka1_c1":  # KA1: 3 sweeps unsmoothed, K-cycle (PAPER.md:277-312 labels)
        A, b, _ = config_problem(1)
        return A, b, dict(smooth_prolongator=0), K, False
    if name == "ka1_48":
        A = poisson7(48, 48, 48)
        return A, uniform01(2, A.n_global), dict(smooth_prolongator=0), K, False
    if name == "ka2_64":  # KA2: 4 sweeps (aggregates of 16) unsmoothed
        A = poisson7(64, 64, 64)
        return A, np.ones(A.n_global), dict(smooth_prolongator=0, sweeps_per_level=4), K, False
    if name == "k_smoothed_32":
        A = poisson7(32, 32, 32)
        return A, uniform_pm1(6, A.n_global), {}, K, False
    if name == "k_aniso_coarse_cg":
        A, b, _ = config_problem(3, grid=(40, 40, 40))
        return A, b, dict(smooth_prolongator=0, pre_sweeps=2, post_sweeps=2), dict(K, coarse_solver=1), True
    if name == "k_jump27_24":
        A = jump27(24)
        return A, uniform01(5, A.n_global), dict(smooth_prolongator=0), K, False
    # several ranks (loopback): the inner FCG exchanges p halos, finishes its dots in rank order
    if name == "ka1_48_loop2":
        A = poisson7(48, 48, 48)
        return A, uniform01(2, A.n_global), dict(smooth_prolongator=0), dict(K, emulate_ranks=2), False
    if name == "ka1_64_loop4_dist":  # replicate nothing but the coarsest: inner FCG on distributed levels
        A = poisson7(64, 64, 64)
        return (A, np.ones(A.n_global), dict(smooth_prolongator=0),
                dict(K, emulate_ranks=4, replicate_below_bytes=0), False)
    if name == "k_aniso22_loop3":
        A, b, _ = config_problem(3, grid=(36, 36, 36))
        return (A, b, dict(smooth_prolongator=0, pre_sweeps=2, post_sweeps=2),
                dict(K, emulate_ranks=3, replicate_below_bytes=1 << 18), False)
    raise KeyError(name)


CASES = ["ka1_c1", "ka1_48", "ka2_64", "k_smoothed_32", "k_aniso_coarse_cg", "k_jump27_24", "ka1_48_loop2",
         "ka1_64_loop4_dist", "k_aniso22_loop3"]
_cache = {}


def _built(ctx, name):
    if name not in _cache:
        A, b, hkw, lkw, ccg = _case(name)
        ho = O.OracleHierarchy(A, **hkw)
        ho.set_cycle("K")
        if ccg:
            ho.set_coarse_cg(True, 1e-4, 30)
        h = _amg().Hierarchy(ctx, A, cfg=_amg().make_config(**hkw, **lkw))
        _cache.clear()
        _cache[name] = (A, b, ho, h)
    return _cache[name]


@pytest.mark.parametrize("name", CASES)
def test_kcycle_hierarchy_bit_exact(ctx, name):
    A, b, ho, h = _built(ctx, name)
    assert h.sizes() == ho.sizes()
    assert h.nlevels >= 3
    for l in range(h.nlevels - 1):
        assert np.array_equal(h.level_aggregates(l), ho.agg(l)), f"level {l}"


@pytest.mark.parametrize("name", CASES)
def test_kcycle_application_parity(ctx, name):
    A, b, ho, h = _built(ctx, name)
    for seed in (1200, 1201):
        r = uniform_pm1(seed, A.n_global)
        z = h.precond_apply(torch.tensor(r, device="cuda:0")).cpu().numpy()
        zo = ho.vcycle(r)
        rel = np.linalg.norm(z - zo) / np.linalg.norm(zo)
        assert rel <= KC_TOL, (seed, rel)


@pytest.mark.parametrize("name", CASES)
def test_kcycle_fcg_parity(ctx, name):
    A, b, ho, h = _built(ctx, name)
    bt = torch.tensor(b, device="cuda:0")
    x, rep = h.solve(bt, rtol=1e-6, maxit=500)
    xo, info = ho.fcg(b, rtol=1e-6, maxit=500)
    assert rep["converged"] == 1 and info["status"] == O.OR_OK, (rep, info)
    assert abs(rep["iterations"] - info["iterations"]) <= 1, (rep["iterations"], info["iterations"])
    k = min(rep["iterations"], info["iterations"])
    x, rep2 = h.solve(bt, rtol=0.0, maxit=k)
    xo, _ = ho.fcg(b, rtol=0.0, maxit=k)
    rel = np.linalg.norm(x.cpu().numpy() - xo) / np.linalg.norm(xo)
    assert rel <= X_TOL, rel


def test_kcycle_eager_equals_graph_and_is_deterministic(ctx):
    amg = _amg()
    A = poisson7(40, 40, 40)
    cfg = dict(smooth_prolongator=0, cycle=1, krylov=1)
    hg = amg.Hierarchy(ctx, A, cfg=amg.make_config(**cfg))
    he = amg.Hierarchy(ctx, A, cfg=amg.make_config(**cfg, use_graphs=0))
    r = torch.tensor(uniform_pm1(88, A.n_global), device="cuda:0")
    zg = hg.precond_apply(r)
    assert torch.equal(zg, he.precond_apply(r))
    assert torch.equal(zg, hg.precond_apply(r))
    b = torch.tensor(uniform01(89, A.n_global), device="cuda:0")
    x1, r1 = hg.solve(b, rtol=1e-8)
    x2, r2 = he.solve(b, rtol=1e-8)
    assert r1["iterations"] == r2["iterations"] and torch.equal(x1, x2)


def test_kcycle_multirank_graph_equals_eager_and_single_rank(ctx):
    """Loopback K-cycle: the WHILE-graph solve equals the eager one bitwise, and both agree with
    the single-rank K-cycle to rounding (same iterations)."""
    amg = _amg()
    A = poisson7(40, 40, 40)
    cfg = dict(smooth_prolongator=0, cycle=1, krylov=1)
    h1 = amg.Hierarchy(ctx, A, cfg=amg.make_config(**cfg))
    hg = amg.Hierarchy(ctx, A, cfg=amg.make_config(**cfg, emulate_ranks=2, replicate_below_bytes=0))
    he = amg.Hierarchy(ctx, A, cfg=amg.make_config(**cfg, emulate_ranks=2, replicate_below_bytes=0,
                                                      use_graphs=0))
    b = torch.tensor(uniform01(90, A.n_global), device="cuda:0")
    x1, r1 = h1.solve(b, rtol=1e-8)
    xg, rg = hg.solve(b, rtol=1e-8)
    xe, re_ = he.solve(b, rtol=1e-8)
    assert rg["iterations"] == re_["iterations"] and torch.equal(xg, xe)
    assert rg["iterations"] == r1["iterations"]
    assert (torch.linalg.norm(xg - x1) / torch.linalg.norm(x1)).item() <= 1e-10
