"""The persistent deep-level tail (cfg.tail_rows): the cycle rooted at the first level
with n_l <= tail_rows runs as one cooperative kernel executing a compiled program of
row reductions / dots / vector updates with grid barriers in between.

It is experimental and OFF by default (measured slower than the launched graph on B200,
see DESIGN.md).  It performs the same operations in the same order as the launched path;
only the lane split of the CSR row sums differs, so results agree to rounding: the
V-cycle / K-cycle application and the PCG / FCG iterates are compared with the
launched path (tail_rows = 0) and with the oracle.
"""
import numpy as np
import pytest

import oracle as O
from inputs import config_problem, poisson7, uniform01, uniform_pm1

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2006_16147_b200 as amg
    c = amg.Context(device=0)
    yield c
    c.close()


TAIL = 40000
MODES = {"grid": dict(tail_rows=TAIL), "cluster": dict(tail_bytes=8 << 20)}


def _pair(ctx, A, mode, **kw):
    import paper_2006_16147_b200 as amg
    return (amg.Hierarchy(ctx, A, cfg=amg.make_config(**MODES[mode], **kw)),
            amg.Hierarchy(ctx, A, cfg=amg.make_config(tail_rows=0, **kw)))


CASES = {
    "v_c2": (lambda: config_problem(2)[0], {}, {}),
    "v_aniso_2x2": (lambda: config_problem(3, grid=(48, 48, 48))[0], dict(pre_sweeps=2, post_sweeps=2), {}),
    "k_ka1_48": (lambda: poisson7(48, 48, 48), dict(smooth_prolongator=0, cycle=1, krylov=1), {"cycle": "K"}),
    "v_fcg_4x4": (lambda: poisson7(40, 40, 40), dict(pre_sweeps=4, post_sweeps=4, krylov=1), {}),
}


@pytest.mark.parametrize("mode", sorted(MODES))
@pytest.mark.parametrize("name", sorted(CASES))
def test_tail_matches_launched_path_and_oracle(ctx, name, mode):
    build, kw, okw = CASES[name]
    A = build()
    ht, hl = _pair(ctx, A, mode, **kw)
    ho = O.OracleHierarchy(A, **{k: v for k, v in kw.items() if k not in ("cycle", "krylov")})
    if okw.get("cycle") == "K":
        ho.set_cycle("K")
    r = uniform_pm1(1300, A.n_global)
    rt = torch.tensor(r, device="cuda:0")
    zt = ht.precond_apply(rt).cpu().numpy()
    zl = hl.precond_apply(rt).cpu().numpy()
    zo = ho.vcycle(r)
    assert np.linalg.norm(zt - zl) <= 1e-13 * np.linalg.norm(zl)
    assert np.linalg.norm(zt - zo) <= 1e-12 * np.linalg.norm(zo)
    b = torch.tensor(uniform01(1301, A.n_global), device="cuda:0")
    xt, rept = ht.solve(b, rtol=1e-6)
    xl, repl = hl.solve(b, rtol=1e-6)
    assert abs(rept["iterations"] - repl["iterations"]) <= 1
    k = min(rept["iterations"], repl["iterations"])
    xt, _ = ht.solve(b, rtol=0.0, maxit=k)
    xl, _ = hl.solve(b, rtol=0.0, maxit=k)
    assert (torch.linalg.norm(xt - xl) / torch.linalg.norm(xl)).item() <= 1e-10


@pytest.mark.parametrize("mode", sorted(MODES))
def test_tail_eager_equals_graph_and_is_deterministic(ctx, mode):
    import paper_2006_16147_b200 as amg
    A = poisson7(64, 64, 64)
    hg = amg.Hierarchy(ctx, A, cfg=amg.make_config(**MODES[mode]))
    he = amg.Hierarchy(ctx, A, cfg=amg.make_config(**MODES[mode], use_graphs=0))
    r = torch.tensor(uniform_pm1(1302, A.n_global), device="cuda:0")
    zg = hg.precond_apply(r)
    assert torch.equal(zg, he.precond_apply(r))
    assert torch.equal(zg, hg.precond_apply(r))
    prof = hg.profile_vcycle(2)
    assert any(k["name"] == "tail" for k in prof)
