"""Determinism probe for the c5 256^3 analogue: build the hierarchy several times (fresh
hierarchies in one process), hash every level's aggregate map, solve several times, print
iteration counts and a hash of x.  (Investigates one A/B run that took 36 iterations instead of 19.)"""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_16147_b200 as amg  # noqa: E402
from inputs import config_problem  # noqa: E402

grid = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "256x256x256").split("x"))
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 3
A, b, meta = config_problem(5, grid=grid)
ctx = amg.Context(device=0)
bt = torch.tensor(b, device="cuda:0")
for k in range(nb):
    h = amg.Hierarchy(ctx, A)
    hs = hashlib.sha1()
    for l in range(h.nlevels - 1):
        hs.update(h.level_aggregates(l).tobytes())
    its = []
    xh = None
    for _ in range(4):
        x, rep = h.solve(bt)
        its.append(rep["iterations"])
        xh = hashlib.sha1(x.cpu().numpy().tobytes()).hexdigest()[:12]
    z = h.precond_apply(bt)
    zh = hashlib.sha1(z.cpu().numpy().tobytes()).hexdigest()[:12]
    print(f"build {k}: sizes {h.sizes()} agg {hs.hexdigest()[:12]} its {its} x {xh} z {zh}", flush=True)
    h.close()
