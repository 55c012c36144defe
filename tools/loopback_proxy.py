"""Loopback overhead proxy for the weak-scaling efficiency.

With one GPU per gpurun call, the multi-rank path can only run in loopback mode: all np
ranks' windows live on ONE GPU, halos move by device copies inside the same CUDA graph, and
every rank's kernels run one after another.  The same total problem (c4 at 256^3 by default)
is solved (a) by one rank and (b) by np loopback ranks; t_loop(np) / t(1) is then the cost of
the multi-rank machinery itself -- split interior/boundary launches, pack/unpack, the halo
copies, per-rank dot slots and rank-ordered finishers -- with the transport at device-copy
speed.  It is a measured stand-in for E_iter until an N-GPU run exists: on N GPUs each rank's
work is 1/N of this and the NVLink transfers replace the copies.

    python tools/loopback_proxy.py [--grid 256x256x256] [--nps 1,2,4,8] [--steps 10]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2006_16147_b200 as amg
    from inputs import config_problem

    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", default="256x256x256")
    ap.add_argument("--nps", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--eager", action="store_true", help="also time use_graphs=0 (host loop)")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: np ranks hold np x the grid (z extent x np), as on np GPUs; "
                         "reports t_loop(np) / (np t(1)), the per-rank share of the serialised loopback time")
    ap.add_argument("--rep", type=int, default=None, help="replicate_below_bytes (default: the library's)")
    ap.add_argument("--nccl", action="store_true",
                    help="build on a one-rank NCCL communicator: the real ranks' transport on one GPU "
                         "(--transport lsa: peer memory through the symmetric window, one WHILE graph; "
                         "nccl: self send/recv, one graph per iteration)")
    ap.add_argument("--transport", default="lsa", choices=["lsa", "nccl"])
    args = ap.parse_args()
    os.environ["AMG_TRANSPORT"] = args.transport
    grid0 = tuple(int(v) for v in args.grid.split("x"))
    ctx = amg.Context(device=0, nranks=1, nccl_uid=amg.nccl_unique_id()) if args.nccl else amg.Context(device=0)
    out = {"grid": list(grid0), "weak": args.weak, "what": __doc__.strip().splitlines()[0], "runs": []}
    base = None
    cache = {}
    for np_ in [int(v) for v in args.nps.split(",")]:
        grid = (grid0[0], grid0[1], grid0[2] * (np_ if args.weak else 1))
        if grid not in cache:
            cache.clear()
            A, b, meta = config_problem(4, grid=grid)
            cache[grid] = (A, torch.tensor(b, device="cuda:0"))
        A, bt = cache[grid]
        for graphs in ([1, 0] if args.eager else [1]):
            extra = {} if args.rep is None else {"replicate_below_bytes": args.rep}
            cfg = amg.make_config(max_coarse_size=200 * np_, emulate_ranks=np_, use_graphs=graphs, **extra)
            h = amg.Hierarchy(ctx, A, cfg=cfg)
            for _ in range(3):
                h.solve(bt)
            ts, its = [], None
            for _ in range(args.steps):
                _, rep = h.solve(bt)
                ts.append(rep["solve_s"])
                its = rep["iterations"]
            t = sorted(ts)[len(ts) // 2]
            prof = h.profile_iteration(bt, 3, cap=4096)
            rec = {"np": np_, "graphs": graphs, "graph_mode": h.graph_mode(), "transport":
                   h.transport(), "grid": list(grid), "solve_ms": t * 1e3, "iterations": its,
                   "ms_per_iter": t * 1e3 / its, "launches_per_iter": len(prof), "levels": h.sizes()}
            if np_ == 1 and graphs == 1:
                base = rec
            if base:
                share = np_ if args.weak else 1
                rec["t_over_t1"] = rec["ms_per_iter"] / (share * base["ms_per_iter"])
            out["runs"].append(rec)
            print(json.dumps(rec), flush=True)
            h.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
