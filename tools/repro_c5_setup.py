"""Determinism probe, setup side: build the c5 hierarchy several times with the GPU setup
(amg_host_hierarchy_build, setup_device = 1) and hash every level's A_l, P-bar_l and omega."""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2006_16147_b200 as amg  # noqa: E402
from inputs import config_problem  # noqa: E402
from test_abi_cpu import HostH  # noqa: E402

grid = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "256x256x256").split("x"))
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = int(sys.argv[3]) if len(sys.argv) > 3 else 1
A, b, meta = config_problem(5, grid=grid)
ref = None
for k in range(nb):
    h = HostH(amg, A, setup_device=dev)
    assert h.code == 0
    per = []
    for l in range(h.nlevels):
        n, na, npp, om = h.sizes(l)
        hs = hashlib.sha1()
        for which in ([0, 1] if l + 1 < h.nlevels else [0]):
            rp, ci, v = h.matrix(l, which)
            hs.update(rp.tobytes()); hs.update(ci.tobytes()); hs.update(v.tobytes())
        per.append((n, na, npp, om, hs.hexdigest()[:10]))
    print(f"build {k} (setup_device={dev}):", [p[4] for p in per], "omega", [p[3] for p in per], flush=True)
    if ref is None:
        ref = per
    else:
        for l, (a, c) in enumerate(zip(ref, per)):
            if a != c:
                print(f"   level {l} differs: {a} vs {c}", flush=True)
    del h
