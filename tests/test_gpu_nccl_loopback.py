"""The NCCL transports of the multi-rank path, exercised on ONE GPU.

Two transports run on NCCL contexts: peer memory over an NCCL symmetric window ("lsa", the
default: push kernels store halo values and dot slots straight into the receivers' window
segments, then a flag barrier) and NCCL send/recv (AMG_TRANSPORT=nccl, the fallback).

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


@pytest.mark.parametrize("transport", ["lsa", "nccl"])
@pytest.mark.parametrize("np_", [2, 3])
@pytest.mark.parametrize("name", ["c4_slabs", "jump27", "kcycle", "hinvk_va3s3cs1"])
def test_nccl_loopback_bitwise_equals_copy_loopback(ctxs, name, np_, transport, monkeypatch):
    import paper_2006_16147_b200 as amg
    plain, nccl = ctxs
    A, b, kw = _case(name)
    cfg = dict(emulate_ranks=np_, replicate_below_bytes=0, **kw)
    hc = amg.Hierarchy(plain, A, cfg=amg.make_config(**cfg))
    monkeypatch.setenv("AMG_TRANSPORT", transport)
    hn = amg.Hierarchy(nccl, A, cfg=amg.make_config(**cfg))
    assert hc.transport() == "copies" and hn.transport() == transport
    bt = torch.tensor(b, device="cuda:0")
    xc, rc = hc.solve(bt)
    xn, rn = hn.solve(bt)
    mode = hn.graph_mode()
    print(f"{name} np={np_} {transport}: solve graph mode = {mode}, its {rn['iterations']}")
    # peer memory keeps NCCL out of the solve: one WHILE graph; NCCL send/recv cannot sit in the
    # WHILE body (wait-event nodes) and falls back to one graph per iteration
    assert mode == ("while" if transport == "lsa" else "iter")
    assert rn["converged"] == 1 and rn["iterations"] == rc["iterations"]
    assert torch.equal(xn, xc)
    xn2, _ = hn.solve(bt)  # the cached graph (or the fallback) again
    assert torch.equal(xn2, xc)
    zc = hc.precond_apply(bt)
    zn = hn.precond_apply(bt)  # eager on NCCL transports, as on real ranks
    assert torch.equal(zn, zc)


@pytest.mark.parametrize("transport", ["lsa", "nccl"])
def test_nccl_loopback_vs_oracle_and_host_batch(ctxs, transport, monkeypatch):
    import paper_2006_16147_b200 as amg
    _, nccl = ctxs
    A, b, _ = config_problem(4, grid=(32, 32, 64))
    monkeypatch.setenv("AMG_TRANSPORT", transport)
    h = amg.Hierarchy(nccl, A, cfg=amg.make_config(emulate_ranks=2))
    assert h.transport() == transport
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


@pytest.mark.parametrize("transport", ["lsa", "nccl"])
@pytest.mark.parametrize("forced,ug,expect", [("iter", 1, "iter"), ("", 0, "eager")])
def test_nccl_loopback_fallback_shapes(forced, ug, expect, transport):
    """The other shapes a real NCCL job may take (one graph per iteration, eager launches), on
    either transport, give the same x bitwise."""
    env = dict(os.environ)
    env["AMG_TRANSPORT"] = transport
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


@pytest.mark.parametrize("transport", ["lsa", "nccl"])
def test_ctx_destroy_with_live_hierarchy_does_not_hang(transport):
    """A graph that captured NCCL collectives holds the communicator: amg_ctx_destroy must release
    the graphs of hierarchies still alive before ncclCommDestroy, or it waits forever (what a
    garbage-collection order at interpreter exit produces under torchrun)."""
    env = dict(os.environ, AMG_TRANSPORT=transport)
    out = subprocess.run([sys.executable, "-c", _ORPHAN.format(root=ROOT)], cwd=ROOT, capture_output=True,
                         text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "CLOSED" in out.stdout


def test_lsa_profiled_kernels_and_overlap(ctxs, monkeypatch):
    """On the peer-memory transport an exchange is a push (+ arrive) kernel and an unpack kernel that
    waits for the barrier itself (a rank with nothing to receive launches a bare wait); no pack
    into a send buffer."""
    import paper_2006_16147_b200 as amg
    _, nccl = ctxs
    A, b, _ = config_problem(4, grid=(64, 64, 128))
    monkeypatch.setenv("AMG_TRANSPORT", "lsa")
    h = amg.Hierarchy(nccl, A, cfg=amg.make_config(emulate_ranks=2, replicate_below_bytes=0))
    assert h.transport() == "lsa"
    names = [k["name"] for k in h.profile_vcycle(1)]
    assert "halo_push" in names and "halo_unpack" in names
    assert "halo_pack" not in names
