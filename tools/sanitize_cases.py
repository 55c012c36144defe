"""Small solves through every kernel family on one B200 (a kernel-family smoke run;
meant for compute-sanitizer memcheck, which this pool does not allow):
    python tools/sanitize_cases.py [v sigma j27 invk kcycle fcg multi eager]
Cases: default V-cycle (SDIA/SELL/CSR/block-CSR), SELL-32-sigma (ragged rows),
27-point, INVK, K-cycle, FCG + cluster coarse CG, loopback multi-rank (pack/unpack,
interior/boundary split), eager and graph launches."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_16147_b200 as amg  # noqa: E402
from inputs import jump27, poisson7, random_spd, uniform01  # noqa: E402


def run(name, A, **cfg):
    ctx = amg.Context(device=0)
    h = amg.Hierarchy(ctx, A, cfg=amg.make_config(**cfg) if cfg else None)
    b = torch.tensor(uniform01(3, A.n_global), device="cuda:0")
    x, rep = h.solve(b, rtol=1e-6, maxit=100)
    z = h.precond_apply(b)
    torch.cuda.synchronize()
    fmts = [h.level_info(l)["format"] for l in range(h.nlevels)]
    print(f"{name}: its {rep['iterations']} conv {rep['converged']} |z| {float(z.norm()):.3e} formats {fmts}",
          flush=True)
    h.close()
    ctx.close()


which = sys.argv[1:] or ["v", "sigma", "j27", "invk", "kcycle", "fcg", "multi", "eager"]
if "v" in which:
    run("v 24^3", poisson7(24, 24, 24))
if "sigma" in which:
    run("sell-sigma 320k irregular", random_spd(320000, deg=4, window=32))
if "j27" in which:
    run("jump27 24^3", jump27(24))
if "invk" in which:
    run("invk 20^3", poisson7(20, 20, 20), smoother=1)
if "kcycle" in which:
    run("kcycle 24^3", poisson7(24, 24, 24), cycle=1, krylov=1, smooth_prolongator=0)
if "fcg" in which:
    run("fcg+coarse cg 24^3", poisson7(24, 24, 24), krylov=1, coarse_solver=1, pre_sweeps=4, post_sweeps=4,
        max_coarse_size=2400)
if "multi" in which:
    run("loopback np=3", poisson7(16, 16, 24), emulate_ranks=3, replicate_below_bytes=0)
if "eager" in which:
    run("eager 20^3", poisson7(20, 20, 20), use_graphs=0)
print("sanitize cases done")
