"""Reproduces bench.py's call sequence on the c5 analogue step by step (debugging aid)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_16147_b200 as amg  # noqa: E402
from inputs import config_problem  # noqa: E402

g = int(sys.argv[1])
A, b, _ = config_problem(5, grid=(g, g, g))
ctx = amg.Context(device=0)
h = amg.Hierarchy(ctx, A)
bt = torch.tensor(b, device="cuda:0")
steps = [("solve", lambda: h.solve(bt)), ("solve2", lambda: h.solve(bt)),
         ("profile_iteration", lambda: h.profile_iteration(bt, 3, cap=4096)),
         ("profile_vcycle", lambda: h.profile_vcycle(3)),
         ("batch", lambda: h.solve_host_batch(np.stack([b, b]))),
         ("solve3", lambda: h.solve(bt))]
for name, f in steps:
    try:
        f()
        print(name, "ok", flush=True)
    except Exception as e:
        print(name, "FAIL", e, flush=True)
