"""The NCCL transport of the multi-rank path, exercised on ONE GPU.

A single-rank context given an ncclUniqueId holds a one-rank NCCL communicator; loopback
hierarchies (cfg.emulate_ranks = np) built on it move every halo and every rank's dot slots
by grouped NCCL self send/recv instead of device copies, and take the real ranks' code path
around them: the collectives are captured into the solve's WHILE-graph body (or, if NCCL
refuses that capture, the collective fallback to one graph per iteration, then to eager
launches), the all-reduced capture decision, eager precond_apply and one-after-another host
batches.  The arithmetic is the same as the device-copy loopback, so x, z and the iteration
counts must be BITWISE equal to it (and that path is oracle-checked in test_gpu_multirank.py).
No kernel waits on another rank: a self send/recv is one NCCL kernel on one stream.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
from inputs import config_problem, jump27, uniform01

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ctxs():
    import paper_2006_16147_b200 as amg
    plain = amg.Context(device=0)
    nccl = amg.Context(device=0, nranks=1, nccl_uid=amg.nccl_unique_id())
    yield plain, nccl
    nccl.close()
    plain.close()


def _case(name):
    if name == "c4_slabs":
        A, b, _ = config_problem(4, grid=(48, 48, 96))
        return A, b, {}
    if name == "jump27":
        A = jump27(24)
        return A, uniform01(5, A.n_global), {}
    if name == "kcycle":  # inner FCG: p halos + K-state dot finishers (dot_finish_k)
        A, b, _ = config_problem(4, grid=(48, 48, 96))
        return A, b, dict(cycle=1, krylov=1, smooth_prolongator=0)
    if name == "hinvk_va3s3cs1":  # block-Jacobi INVK smoother + HINVK coarse CG
        A, b, _ = config_problem(2, grid=(32, 32, 64))
        return A, b, dict(smoother=1, krylov=1, coarse_solver=1, coarse_prec=1, max_coarse_size=400)
    raise KeyError(name)


@pytest.mark.parametrize("np_", [2, 3])
@pytest.mark.parametrize("name", ["c4_slabs", "jump27", "kcycle", "hinvk_va3s3cs1"])
def test_nccl_loopback_bitwise_equals_copy_loopback(ctxs, name, np_):
    import paper_2006_16147_b200 as amg
    plain, nccl = ctxs
    A, b, kw = _case(name)
    cfg = dict(emulate_ranks=np_, replicate_below_bytes=0, **kw)
    hc = amg.Hierarchy(plain, A, cfg=amg.make_config(**cfg))
    hn = amg.Hierarchy(nccl, A, cfg=amg.make_config(**cfg))
    bt = torch.tensor(b, device="cuda:0")
    xc, rc = hc.solve(bt)
    xn, rn = hn.solve(bt)
    mode = hn.graph_mode()
    print(f"{name} np={np_}: NCCL loopback solve graph mode = {mode}, its {rn['iterations']}")
    assert mode in ("while", "iter")
    assert rn["converged"] == 1 and rn["iterations"] == rc["iterations"]
    assert torch.equal(xn, xc)
    xn2, _ = hn.solve(bt)  # the cached graph (or the fallback) again
    assert torch.equal(xn2, xc)
    zc = hc.precond_apply(bt)
    zn = hn.precond_apply(bt)  # eager on NCCL transports, as on real ranks
    assert torch.equal(zn, zc)


def test_nccl_loopback_vs_oracle_and_host_batch(ctxs):
    import paper_2006_16147_b200 as amg
    _, nccl = ctxs
    A, b, _ = config_problem(4, grid=(32, 32, 64))
    h = amg.Hierarchy(nccl, A, cfg=amg.make_config(emulate_ranks=2))
    ho = O.OracleHierarchy(A)
    bt = torch.tensor(b, device="cuda:0")
    x, rep = h.solve(bt)
    _, info = ho.pcg(b)
    assert abs(rep["iterations"] - info["iterations"]) <= 1
    k = min(rep["iterations"], info["iterations"])
    x, _ = h.solve(bt, rtol=0.0, maxit=k)
    xo, _ = ho.pcg(b, rtol=0.0, maxit=k)
    assert np.linalg.norm(x.cpu().numpy() - xo) / np.linalg.norm(xo) <= 1e-8
    B = np.stack([b, uniform01(77, A.n_global)])
    X, reps = h.solve_host_batch(B)
    for j in range(2):
        xj, _ = h.solve_host(B[j])
        assert np.array_equal(X[j], xj)


_FORCED = r"""
import sys, torch
sys.path.insert(0, {root!r})
import paper_2006_16147_b200 as amg
from inputs import config_problem
A, b, _ = config_problem(4, grid=(32, 32, 64))
plain = amg.Context(device=0)
nccl = amg.Context(device=0, nranks=1, nccl_uid=amg.nccl_unique_id())
bt = torch.tensor(b, device="cuda:0")
xc, rc = amg.Hierarchy(plain, A, cfg=amg.make_config(emulate_ranks=2)).solve(bt)
h = amg.Hierarchy(nccl, A, cfg=amg.make_config(emulate_ranks=2, use_graphs={ug}))
xn, rn = h.solve(bt)
assert rn["iterations"] == rc["iterations"] and torch.equal(xn, xc), (rn, rc)
print("MODE", h.graph_mode())
"""


@pytest.mark.parametrize("forced,ug,expect", [("iter", 1, "iter"), ("", 0, "eager")])
def test_nccl_loopback_fallback_shapes(forced, ug, expect):
    """The fallback shapes a real NCCL job may take (one graph per iteration, eager launches),
    run with NCCL collectives, give the same x bitwise."""
    env = dict(os.environ)
    if forced:
        env["AMG_MULTI_GRAPH"] = forced
    out = subprocess.run([sys.executable, "-c", _FORCED.format(root=ROOT, ug=ug)], env=env, cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    assert f"MODE {expect}" in out.stdout, out.stdout


_ORPHAN = r"""
import sys, torch
sys.path.insert(0, {root!r})
import paper_2006_16147_b200 as amg
from inputs import config_problem
A, b, _ = config_problem(4, grid=(32, 32, 64))
nccl = amg.Context(device=0, nranks=1, nccl_uid=amg.nccl_unique_id())
h = amg.Hierarchy(nccl, A, cfg=amg.make_config(emulate_ranks=2))
x, rep = h.solve(torch.tensor(b, device="cuda:0"))
nccl.close()   # the hierarchy (and its graphs of captured NCCL work) is still alive
del h
print("CLOSED", rep["iterations"])
"""


def test_ctx_destroy_with_live_hierarchy_does_not_hang():
    """A graph that captured NCCL collectives holds the communicator: amg_ctx_destroy must release
    the graphs of hierarchies still alive before ncclCommDestroy, or it waits forever (what a
    garbage-collection order at interpreter exit produces under torchrun)."""
    out = subprocess.run([sys.executable, "-c", _ORPHAN.format(root=ROOT)], cwd=ROOT, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "CLOSED" in out.stdout
