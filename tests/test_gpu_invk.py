"""GPU parity of the INVK smoother.

Each smoothing step is x += Z (Wd (b - A x)) with Wd = D^{-1} W, Z = W^T, W the IC(0)
factor's inverse truncated to `invk_fill` levels of positional fill.  The library builds
the factors with its own host code (setup.cpp invk_factors) and applies them with the
generic SpMV kernels; the oracle (oracle.c ic0 / invk_inverse) is pinned in
tests/test_oracle_pins.py.  Bars as for the other smoothers: cycle <= 1e-12, iterations
+-1, x <= 1e-8 at equal counts.  Cases cover the literal fill definition on every level,
the block-Jacobi forms HINVK / l1-INVK (k blocks on one GPU and one block per loopback
rank), VA3S3CS1 (FCG, one HINVK sweep, coarse CG preconditioned by HINVK)
and the non-paper invk_dense_cut knob against the oracle's per-level fill.
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


def _eq_bounds(n, k):
    return [n * g // k for g in range(k + 1)]


def _case(name):
    """-> (A, b, shared hierarchy kwargs, library kwargs, oracle smoother kwargs, krylov 'pcg'|'fcg',
    K-cycle?, oracle coarse CG (rtol, maxit) or None)"""
    if name == "c1_fill1":
        A, b, _ = config_problem(1)
        return A, b, {}, dict(smoother=1, invk_fill=1), dict(fill=1), "pcg", False, None
    if name == "p32_fill1":
        A = poisson7(32, 32, 32)
        return A, uniform01(2, A.n_global), {}, dict(smoother=1, invk_fill=1), dict(fill=1), "pcg", False, None
    if name == "p24_fill0":
        A = poisson7(24, 24, 24)
        return A, uniform_pm1(3, A.n_global), {}, dict(smoother=1, invk_fill=0), dict(fill=0), "pcg", False, None
    if name == "p24_fill2_2x2":
        A = poisson7(24, 24, 24)
        kw = dict(pre_sweeps=2, post_sweeps=2)
        return A, uniform01(4, A.n_global), kw, dict(smoother=1, invk_fill=2), dict(fill=2), "pcg", False, None
    if name == "aniso40_fill1":
        A, b, _ = config_problem(3, grid=(40, 40, 40))
        return A, b, {}, dict(smoother=1, invk_fill=1), dict(fill=1), "pcg", False, None
    if name == "jump27_24_fill1":
        A = jump27(24)
        return A, uniform01(5, A.n_global), {}, dict(smoother=1, invk_fill=1), dict(fill=1), "pcg", False, None
    if name == "kcycle_fcg_fill1":
        A = poisson7(40, 40, 40)
        kw = dict(smooth_prolongator=0)
        return (A, np.ones(A.n_global), kw, dict(smoother=1, invk_fill=1, cycle=1, krylov=1), dict(fill=1), "fcg",
                True, None)
    # --- the paper's block-Jacobi forms: k diagonal blocks on one GPU
    if name == "hinvk4_p24":
        A = poisson7(24, 24, 24)
        return (A, uniform01(6, A.n_global), {}, dict(smoother=1, invk_blocks=4),
                dict(fill=1, blocks=_eq_bounds(A.n_global, 4)), "pcg", False, None)
    if name == "l1invk4_p24":
        A = poisson7(24, 24, 24)
        return (A, uniform01(7, A.n_global), {}, dict(smoother=1, invk_blocks=4, invk_l1=1),
                dict(fill=1, blocks=_eq_bounds(A.n_global, 4), l1=True), "pcg", False, None)
    if name == "kcycle_hinvk8":
        A = poisson7(40, 40, 40)
        kw = dict(smooth_prolongator=0)
        return (A, np.ones(A.n_global), kw, dict(smoother=1, invk_blocks=8, cycle=1, krylov=1),
                dict(fill=1, blocks=_eq_bounds(A.n_global, 8)), "fcg", True, None)
    # --- several ranks (loopback): the blocks are the ranks' rows
    if name == "loop2_hinvk_p32":
        A = poisson7(32, 32, 32)
        return (A, uniform01(8, A.n_global), {}, dict(smoother=1, emulate_ranks=2),
                dict(fill=1, blocks=_eq_bounds(A.n_global, 2)), "pcg", False, None)
    if name == "loop3_l1invk_jump27":
        A = jump27(24)
        return (A, uniform01(9, A.n_global), {}, dict(smoother=1, emulate_ranks=3, invk_l1=1,
                                                       replicate_below_bytes=1 << 16),
                dict(fill=1, blocks=_eq_bounds(A.n_global, 3), l1=True), "pcg", False, None)
    # --- VA3S3CS1: one HINVK sweep, FCG, coarse CG preconditioned by HINVK
    if name == "va3s3cs1_p32":
        A = poisson7(32, 32, 32)
        kw = dict(max_coarse_size=2400)
        lk = dict(smoother=1, krylov=1, coarse_solver=1, coarse_prec=1, coarse_rtol=1e-4, coarse_maxit=30)
        return A, np.ones(A.n_global), kw, lk, dict(fill=1), "fcg", False, (1e-4, 30)
    if name == "va3s3cs1_loop2_jump27":
        A = jump27(24)
        kw = dict(max_coarse_size=2400)
        lk = dict(smoother=1, krylov=1, coarse_solver=1, coarse_prec=1, coarse_rtol=1e-4, coarse_maxit=30,
                  emulate_ranks=2)
        return (A, uniform01(10, A.n_global), kw, lk, dict(fill=1, blocks=_eq_bounds(A.n_global, 2)), "fcg",
                False, (1e-4, 30))
    # --- the non-paper setup-cost knob: fill 0 on levels with > 27 entries per row
    if name == "densecut27_p32":
        A = poisson7(32, 32, 32)
        ho = O.OracleHierarchy(A)
        fills = [0 if ho.nnz(l) > 27 * ho.level_n(l) else 1 for l in range(ho.nlevels)]
        assert 0 in fills and 1 in fills
        return (A, uniform01(11, A.n_global), {}, dict(smoother=1, invk_dense_cut=27),
                dict(fill=1, fill_per_level=fills), "pcg", False, None)
    raise KeyError(name)


CASES = ["c1_fill1", "p32_fill1", "p24_fill0", "p24_fill2_2x2", "aniso40_fill1", "jump27_24_fill1",
         "kcycle_fcg_fill1", "hinvk4_p24", "l1invk4_p24", "kcycle_hinvk8", "loop2_hinvk_p32",
         "loop3_l1invk_jump27", "va3s3cs1_p32", "va3s3cs1_loop2_jump27", "densecut27_p32"]
_cache = {}


def _built(ctx, name):
    if name not in _cache:
        A, b, hkw, lkw, okw, kr, kc, ccg = _case(name)
        ho = O.OracleHierarchy(A, **hkw)
        if ccg is not None:
            ho.set_coarse_cg(True, rtol=ccg[0], maxit=ccg[1])
            ho.set_coarse_prec("invk")
        ho.set_smoother("invk", **okw)
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


def test_invk_block_options_rejected_when_inconsistent(ctx):
    """With several ranks the INVK blocks are the ranks' row blocks (invk_blocks 0 or np)."""
    amg = _amg()
    with pytest.raises(amg.AmgError):
        amg.Hierarchy(ctx, poisson7(16, 16, 16), cfg=amg.make_config(smoother=1, emulate_ranks=2, invk_blocks=3))
    with pytest.raises(amg.AmgError):
        amg.Hierarchy(ctx, poisson7(16, 16, 16), cfg=amg.make_config(smoother=1, invk_l1=2))


def test_hinvk_more_blocks_weaker_smoother(ctx):
    """Table 1 trend: K of HINVK grows with the number of blocks, so the
    solver needs at least as many iterations with 64 blocks as with one."""
    amg = _amg()
    A = poisson7(48, 48, 48)
    b = torch.ones(A.n_global, dtype=torch.float64, device="cuda:0")
    _, r1 = amg.Hierarchy(ctx, A, cfg=amg.make_config(smoother=1)).solve(b, rtol=1e-6)
    _, r64 = amg.Hierarchy(ctx, A, cfg=amg.make_config(smoother=1, invk_blocks=64)).solve(b, rtol=1e-6)
    assert r64["iterations"] >= r1["iterations"], (r64, r1)
