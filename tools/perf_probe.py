"""Perf probe (not a test): per-kernel V-cycle timing of the c4 hierarchy."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_16147_b200 as amg
from inputs import config_problem
cfg = int(os.environ.get("PROBE_CONFIG", "4"))
A, b, meta = config_problem(cfg)
ctx = amg.Context(0)
h = amg.Hierarchy(ctx, A, cfg=amg.make_config(pre_sweeps=meta["sweeps"][0], post_sweeps=meta["sweeps"][1]))
prof = h.profile_vcycle(20)
bt = torch.tensor(b, device="cuda")
z = torch.empty_like(bt)
h.precond_apply(bt, z)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(20): h.precond_apply(bt, z)
e1.record(); torch.cuda.synchronize()
tag = os.environ.get("PROBE_TAG", "")
print(json.dumps({"tag": tag, "vcycle_ms_approx": e0.elapsed_time(e1) / 20,
                  "levels": [h.level_info(l)["format"] for l in range(h.nlevels)],
                  "kernels": [(k["name"], round(k["ms"] * 1e3, 1), round(k["bytes"] / k["ms"] / 1e6, 0)) for k in prof]}))
