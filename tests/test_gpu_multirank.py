"""Multi-rank CUDA path on one GPU ("loopback", cfg.emulate_ranks = np).

The hierarchy is partitioned into np row blocks exactly as across np GPUs; every
rank's kernels run on its own window of each level, halos are packed, copied
device-to-device (instead of NCCL send/recv) and unpacked, dot products are
reduced per rank, all-gathered and summed in rank order, and the deep levels are
replicated after a gather.  Every operator that gathers a distributed vector runs
its interior rows (no halo columns) while the halo exchange is in flight on a second
stream, then its boundary rows (north_star (4)).  Same parity bars as the single-rank
path against the CPU oracle.  (Ranks that wait on each other are never launched as concurrent
kernels on one GPU: the loopback transport is stream-ordered copies.)
"""
import numpy as np
import pytest

import oracle as O
from inputs import config_problem, islands, jump27, poisson7, random_spd, uniform01, uniform_pm1

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2006_16147_b200 as amg
    c = amg.Context(device=0)
    yield c
    c.close()


def _case(name):
    if name == "c4_slabs":
        A, b, _ = config_problem(4, grid=(32, 32, 64))
        return A, b, {}
    if name == "aniso22":
        A, b, _ = config_problem(3, grid=(32, 32, 32))
        return A, b, dict(pre_sweeps=2, post_sweeps=2)
    if name == "jump27":
        A = jump27(16)
        return A, uniform01(5, A.n_global), {}
    if name == "irregular_hubs":  # not slab-shaped: hub rows couple every rank with every rank
        A = random_spd(6000, hubs=3)
        return A, uniform_pm1(6, A.n_global), {}
    if name == "islands":  # disconnected components + isolated rows interleaved over the ranks
        A = islands()
        return A, uniform01(29, A.n_global), dict(max_coarse_size=20)
    raise KeyError(name)


@pytest.mark.parametrize("rep_bytes", [0, 1 << 22])
@pytest.mark.parametrize("np_", [2, 3, 4])
@pytest.mark.parametrize("name", ["c4_slabs", "aniso22", "jump27", "irregular_hubs", "islands"])
def test_loopback_multirank_parity(ctx, name, np_, rep_bytes):
    import paper_2006_16147_b200 as amg
    A, b, kw = _case(name)
    ho = O.OracleHierarchy(A, **kw)
    h = amg.Hierarchy(ctx, A, cfg=amg.make_config(emulate_ranks=np_, replicate_below_bytes=rep_bytes, **kw))
    assert h.sizes() == ho.sizes()
    for l in range(h.nlevels - 1):
        assert np.array_equal(h.level_aggregates(l), ho.agg(l))
    r = uniform_pm1(2024, A.n_global)
    z = h.precond_apply(torch.tensor(r, device="cuda:0")).cpu().numpy()
    zo = ho.vcycle(r)
    assert np.linalg.norm(z - zo) / np.linalg.norm(zo) <= 1e-12
    bt = torch.tensor(b, device="cuda:0")
    x, rep = h.solve(bt)
    xo, info = ho.pcg(b)
    assert rep["converged"] == 1
    assert abs(rep["iterations"] - info["iterations"]) <= 1
    k = min(rep["iterations"], info["iterations"])
    x, _ = h.solve(bt, rtol=0.0, maxit=k)
    xo, _ = ho.pcg(b, rtol=0.0, maxit=k)
    assert np.linalg.norm(x.cpu().numpy() - xo) / np.linalg.norm(xo) <= 1e-8


def test_loopback_matches_single_rank_and_is_deterministic(ctx):
    import paper_2006_16147_b200 as amg
    A, b, _ = config_problem(4, grid=(32, 32, 96))
    bt = torch.tensor(b, device="cuda:0")
    h1 = amg.Hierarchy(ctx, A)
    h3 = amg.Hierarchy(ctx, A, cfg=amg.make_config(emulate_ranks=3, replicate_below_bytes=0))
    x1, r1 = h1.solve(bt)
    x3, r3 = h3.solve(bt)
    assert r1["iterations"] == r3["iterations"]
    assert (torch.linalg.norm(x1 - x3) / torch.linalg.norm(x1)).item() <= 1e-10
    x3b, _ = h3.solve(bt)
    assert torch.equal(x3, x3b)
    xh, _ = h3.solve_host(b)
    assert np.array_equal(xh, x3.cpu().numpy())


def test_too_small_for_ranks_is_an_error(ctx):
    import paper_2006_16147_b200 as amg
    A = poisson7(5, 4, 3)  # single-level hierarchy
    with pytest.raises(amg.AmgError):
        amg.Hierarchy(ctx, A, cfg=amg.make_config(emulate_ranks=2))


def test_loopback_overlap_splits_operators_into_interior_and_boundary(ctx):
    """With a z-slab partition every distributed operator launch is split: the interior
    part (while the halo is exchanged) and the head/tail boundary parts after it, so the
    level-0 residual appears as more than one launch per rank in a profiled V-cycle."""
    import paper_2006_16147_b200 as amg
    A, b, _ = config_problem(4, grid=(64, 64, 128))
    h = amg.Hierarchy(ctx, A, cfg=amg.make_config(emulate_ranks=2, replicate_below_bytes=0))
    prof = h.profile_vcycle(1)
    n_resid0 = sum(1 for k in prof if k["name"] == "resid0")
    n_post = sum(1 for k in prof if k["name"].startswith("postsweep"))
    # one launch per rank would give exactly 2 per level; the split gives interior + boundary
    assert n_resid0 > 2 * (h.nlevels - 1) and n_post > 2 * (h.nlevels - 1), (n_resid0, n_post)
    # and the split application equals the single-rank one to rounding
    r = uniform_pm1(1500, A.n_global)
    z = h.precond_apply(torch.tensor(r, device="cuda:0")).cpu().numpy()
    zs = amg.Hierarchy(ctx, A).precond_apply(torch.tensor(r, device="cuda:0")).cpu().numpy()
    assert np.linalg.norm(z - zs) <= 1e-12 * np.linalg.norm(zs)


def test_loopback_profile_vcycle_and_report(ctx):
    """The instrumented V-cycle (per-kernel events, bench.py's roofline source) and the
    report work on the multi-rank path too (what bench.py calls under torchrun)."""
    import paper_2006_16147_b200 as amg
    A, b, _ = config_problem(4, grid=(32, 32, 64))
    h = amg.Hierarchy(ctx, A, cfg=amg.make_config(emulate_ranks=2, replicate_below_bytes=0))
    prof = h.profile_vcycle(2)
    assert prof and all(k["ms"] > 0 and k["bytes"] > 0 for k in prof)
    names = {k["name"] for k in prof}
    assert {"resid0", "restrict", "prolong", "postsweep"} <= names
    rep = h.report()
    assert rep["vcycle_bytes_model"] > 0 and rep["nlevels"] == h.nlevels


@pytest.mark.parametrize("np_", [2, 4])
def test_loopback_graph_equals_eager_and_oracle(ctx, np_):
    """The multi-rank PCG is ONE graph per solve (a device-side WHILE node over the iteration,
    halo copies / exchanges and the rank-ordered dot finishers inside it): bitwise the same x
    and iteration count as the eager host loop, and the oracle's iterations +-1."""
    import paper_2006_16147_b200 as amg
    A, b, _ = config_problem(4, grid=(48, 48, 96))
    bt = torch.tensor(b, device="cuda:0")
    hg = amg.Hierarchy(ctx, A, cfg=amg.make_config(emulate_ranks=np_))
    he = amg.Hierarchy(ctx, A, cfg=amg.make_config(emulate_ranks=np_, use_graphs=0))
    xg, rg = hg.solve(bt)
    xe, re_ = he.solve(bt)
    assert rg["iterations"] == re_["iterations"]
    assert torch.equal(xg, xe)
    _, info = O.OracleHierarchy(A).pcg(b)
    assert abs(rg["iterations"] - info["iterations"]) <= 1
    zg = hg.precond_apply(bt)
    ze = he.precond_apply(bt)
    assert torch.equal(zg, ze)


def test_loopback_replicated_levels_run_the_single_rank_fused_forms(ctx):
    """Replicated levels compute every row on every rank, so they use the same compact /
    collapsed level forms as one rank (W5); level 0 uses the fused direction update with the
    z-halo unpack forming p_new at the halo (no separate p-update kernel)."""
    import paper_2006_16147_b200 as amg
    import os
    A, b, _ = config_problem(4, grid=(96, 96, 96))  # levels ... -> 1.7k (compact) -> 220 (collapsed) -> 28
    os.environ["AMG_NO_COLLAPSE2"] = "1"  # keep the compact level visible (else it collapses as well)
    try:
        h = amg.Hierarchy(ctx, A, cfg=amg.make_config(emulate_ranks=4))
    finally:
        os.environ.pop("AMG_NO_COLLAPSE2", None)
    names = [k["name"] for k in h.profile_vcycle(1)]
    assert "collapsed" in names and "prolong_post_c" in names, names
    os.environ["AMG_FORCE_COLLAPSE2"] = "1"  # second collapse on the replicated levels
    try:
        h2 = amg.Hierarchy(ctx, A, cfg=amg.make_config(emulate_ranks=4))
    finally:
        os.environ.pop("AMG_FORCE_COLLAPSE2", None)
    n2 = [k["name"] for k in h2.profile_vcycle(1)]
    assert n2.count("collapsed") == 4 and "prolong_post_c" not in n2, n2  # one per loopback rank
    it = [k["name"] for k in h.profile_iteration(torch.tensor(b, device="cuda:0"), 2)]
    assert "spmv_dot_pupd" in it and "pupdate" not in it, it
    ho = O.OracleHierarchy(A)
    r = uniform_pm1(77, A.n_global)
    z = h.precond_apply(torch.tensor(r, device="cuda:0")).cpu().numpy()
    zo = ho.vcycle(r)
    assert np.linalg.norm(z - zo) <= 1e-12 * np.linalg.norm(zo)
    bt = torch.tensor(b, device="cuda:0")
    x, rep = h.solve(bt)
    xo, info = ho.pcg(b)
    assert abs(rep["iterations"] - info["iterations"]) <= 1
    k = min(rep["iterations"], info["iterations"])
    x, _ = h.solve(bt, rtol=0.0, maxit=k)
    xo, _ = ho.pcg(b, rtol=0.0, maxit=k)
    assert np.linalg.norm(x.cpu().numpy() - xo) <= 1e-8 * np.linalg.norm(xo)
    z2 = h2.precond_apply(torch.tensor(r, device="cuda:0")).cpu().numpy()
    assert np.linalg.norm(z2 - zo) <= 1e-12 * np.linalg.norm(zo)


@pytest.mark.parametrize("np_,extra", [(2, {}), (4, dict(replicate_below_bytes=0)), (3, dict(smoother=1)),
                                       (2, dict(smooth_prolongator=0, cycle=1, krylov=1)),
                                       (2, dict(smoother=1, invk_l1=1, krylov=1, coarse_solver=1, coarse_prec=1,
                                                max_coarse_size=2400))])
def test_distributed_setup_solves_exactly_like_the_gathered_setup(ctx, np_, extra):
    """setup_distributed = 1 (NEXT-1): every rank builds only its rows and its own plan (loopback:
    np threads of this process with an in-process transport).  The plans are bit-identical to
    the gathered build's (tests/test_dist_setup_cpu.py), so the solves are bitwise equal; the
    aggregate maps equal the oracle's.  Covers HINVK / l1-INVK factors built per rank and the
    K-cycle on the distributed hierarchy."""
    import paper_2006_16147_b200 as amg
    A, b, _ = config_problem(4, grid=(32, 32, 96))
    bt = torch.tensor(b, device="cuda:0")
    kw = dict(emulate_ranks=np_, **extra)
    hg = amg.Hierarchy(ctx, A, cfg=amg.make_config(setup_distributed=0, **kw))
    hd = amg.Hierarchy(ctx, A, cfg=amg.make_config(setup_distributed=1, **kw))
    assert hd.sizes() == hg.sizes()
    okw = {k: v for k, v in extra.items() if k in ("smooth_prolongator", "max_coarse_size")}
    ho = O.OracleHierarchy(A, **okw)
    for l in range(hd.nlevels - 1):
        assert np.array_equal(hd.level_aggregates(l), ho.agg(l)), l
    assert hd.report()["opc"] == hg.report()["opc"]
    xg, rg = hg.solve(bt)
    xd, rd = hd.solve(bt)
    assert rg["iterations"] == rd["iterations"] and torch.equal(xg, xd)
    r = torch.tensor(uniform_pm1(31, A.n_global), device="cuda:0")
    assert torch.equal(hg.precond_apply(r), hd.precond_apply(r))


def test_loopback_host_batch_equals_single_solves(ctx):
    """amg_solve_host_batch pipelines the copies with the (WHILE-graph) solves on a loopback
    multi-rank hierarchy too: bitwise the solutions and reports of one amg_solve_host each."""
    import paper_2006_16147_b200 as amg
    A, _, _ = config_problem(4, grid=(32, 32, 64))
    h = amg.Hierarchy(ctx, A, cfg=amg.make_config(emulate_ranks=2))
    n = A.n_global
    B = np.stack([uniform01(400 + k, n) for k in range(4)])
    B[2] = 0.0
    X, reps = h.solve_host_batch(B.copy(), rtol=1e-6)
    for k in range(B.shape[0]):
        xk, rk = h.solve_host(B[k].copy(), rtol=1e-6)
        assert np.array_equal(X[k], xk), k
        assert reps[k]["iterations"] == rk["iterations"]
    assert reps[2]["iterations"] == 0 and not X[2].any()
