import os, sys, torch
sys.path.insert(0, ".")
import paper_2006_16147_b200 as amg
from inputs import config_problem
A, b, _ = config_problem(4, grid=(128, 128, 256))
tr = sys.argv[1]
os.environ["AMG_TRANSPORT"] = "nccl" if tr == "nccl" else "lsa"
ctx = amg.Context(device=0, nranks=1, nccl_uid=amg.nccl_unique_id()) if tr != "copies" else amg.Context(device=0)
h = amg.Hierarchy(ctx, A, cfg=amg.make_config(emulate_ranks=2))
bt = torch.tensor(b, device="cuda:0")
for _ in range(2):
    h.solve(bt)
print(tr, h.transport(), h.graph_mode())
