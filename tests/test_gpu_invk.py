"""GPU parity of the INVK smoother.

Each smoothing step is x += Z (Wd (b - A x)) with Wd = D^{-1} W, Z = W^T, W the IC(0)
factor's inverse truncated to `invk_fill` levels of positional fill.  The library builds
the factors with its own host code (setup.cpp invk_factors) and applies them with the
generic SpMV kernels; the oracle (oracle.c ic0 / invk_inverse) is pinned in
tests/test_oracle_pins.py.  Bars as for the other smoothers: cycle <= 1e-12, iterations
+-1, x <= 1e-8 at equal counts.
"""
import numpy as np
import pytest

import oracle as O
from inputs import config_problem, jump27, poisson7, uniform01, uniform_pm1

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _amg():
    import paper_2006_16147_b200 as amg
    return amg


@pytest.fixture(scope="module")
def ctx():
    c = _amg().Context(device=0)
    yield c
    c.close()


def _case(name):
    """-> (A, b, shared hierarchy kwargs, library kwargs, oracle fill, krylov 'pcg'|'fcg', K-cycle?)"""
    if name == "c1_fill1":
        A, b, _ = config_problem(1)
        return A, b, {}, dict(smoother=1, invk_fill=1), 1, "pcg", False
    if name == "p32_fill1":
        A = poisson7(32, 32, 32)
        return A, uniform01(2, A.n_global), {}, dict(smoother=1, invk_fill=1), 1, "pcg", False
    if name == "p24_fill0":
        A = poisson7(24, 24, 24)
        return A, uniform_pm1(3, A.n_global), {}, dict(smoother=1, invk_fill=0), 0, "pcg", False
    if name == "p24_fill2_2x2":
        A = poisson7(24, 24, 24)
        kw = dict(pre_sweeps=2, post_sweeps=2)
        return A, uniform01(4, A.n_global), kw, dict(smoother=1, invk_fill=2), 2, "pcg", False
    if name == "aniso40_fill1":
        A, b, _ = config_problem(3, grid=(40, 40, 40))
        return A, b, {}, dict(smoother=1, invk_fill=1), 1, "pcg", False
    if name == "jump27_24_fill1":
        A = jump27(24)
        return A, uniform01(5, A.n_global), {}, dict(smoother=1, invk_fill=1), 1, "pcg", False
    if name == "kcycle_fcg_fill1":
        A = poisson7(40, 40, 40)
        kw = dict(smooth_prolongator=0)
        return A, np.ones(A.n_global), kw, dict(smoother=1, invk_fill=1, cycle=1, krylov=1), 1, "fcg", True
    raise KeyError(name)


CASES = ["c1_fill1", "p32_fill1", "p24_fill0", "p24_fill2_2x2", "aniso40_fill1", "jump27_24_fill1",
         "kcycle_fcg_fill1"]
_cache = {}


def _built(ctx, name):
    if name not in _cache:
        A, b, hkw, lkw, fill, kr, kc = _case(name)
        ho = O.OracleHierarchy(A, **hkw)
        ho.set_smoother("invk", fill=fill)
        if kc:
            ho.set_cycle("K")
        h = _amg().Hierarchy(ctx, A, cfg=_amg().make_config(**hkw, **lkw))
        _cache.clear()
        _cache[name] = (A, b, ho, h, kr)
    return _cache[name]


@pytest.mark.parametrize("name", CASES)
def test_invk_cycle_parity(ctx, name):
    A, b, ho, h, _ = _built(ctx, name)
    for seed in (1400, 1401):
        r = uniform_pm1(seed, A.n_global)
        z = h.precond_apply(torch.tensor(r, device="cuda:0")).cpu().numpy()
        zo = ho.vcycle(r)
        rel = np.linalg.norm(z - zo) / np.linalg.norm(zo)
        assert rel <= 1e-12, (seed, rel)


@pytest.mark.parametrize("name", CASES)
def test_invk_solver_parity(ctx, name):
    A, b, ho, h, kr = _built(ctx, name)
    solve_o = ho.fcg if kr == "fcg" else ho.pcg
    bt = torch.tensor(b, device="cuda:0")
    x, rep = h.solve(bt, rtol=1e-6)
    xo, info = solve_o(b, rtol=1e-6)
    assert rep["converged"] == 1 and info["status"] == O.OR_OK
    assert abs(rep["iterations"] - info["iterations"]) <= 1, (rep["iterations"], info["iterations"])
    k = min(rep["iterations"], info["iterations"])
    x, _ = h.solve(bt, rtol=0.0, maxit=k)
    xo, _ = solve_o(b, rtol=0.0, maxit=k)
    rel = np.linalg.norm(x.cpu().numpy() - xo) / np.linalg.norm(xo)
    assert rel <= 1e-8, rel


def test_invk_fewer_iterations_than_l1_jacobi(ctx):
    """Table 1 / PAPER.md:420-421: INVK is the stronger smoother — fewer PCG iterations than
    one l1-Jacobi sweep on the same hierarchy."""
    amg = _amg()
    A = poisson7(64, 64, 64)
    b = torch.ones(A.n_global, dtype=torch.float64, device="cuda:0")
    _, rj = amg.Hierarchy(ctx, A).solve(b, rtol=1e-6)
    _, ri = amg.Hierarchy(ctx, A, cfg=amg.make_config(smoother=1)).solve(b, rtol=1e-6)
    assert ri["iterations"] < rj["iterations"], (ri, rj)


def test_invk_rejects_multirank(ctx):
    amg = _amg()
    with pytest.raises(amg.AmgError):
        amg.Hierarchy(ctx, poisson7(16, 16, 16), cfg=amg.make_config(smoother=1, emulate_ranks=2))
