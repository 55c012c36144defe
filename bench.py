"""bench.py — AMG-PCG solve benchmark (BASELINE.json metric) on 1..N B200s.

Default workload: BASELINE config 4 (weak scaling), 3D Poisson 7-point with
256^3 unknowns per GPU (z-slabs), b = 1, x0 = 0, PCG rtol 1e-6, one V-cycle per
iteration over the matching-aggregation hierarchy (3 sweeps, smoothed P,
l1-Jacobi 1/1, direct coarsest solve).  A "step" is one full PCG solve.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

Prints ONE JSON line on rank 0.  `value` = unknowns solved per second over all
ranks (n_global / device time per solve, max over ranks).  The hierarchy and
inputs are resident in HBM before the timed region; the hierarchy (GBs) is far
larger than the 126 MB L2, so no L2 flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AMG-PCG solve s & ms/iter at rtol 1e-6; V-cycle HBM GB/s; weak-scaling eff 1/2/4/8"
UNIT = "dof/s (unknowns solved to rtol 1e-6 per second)"
NOMINAL_HBM_GBS = 8000.0
CPU_SAMPLE_GRID = (96, 96, 96)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def workload_name(cfg, grid):
    return {1: "c1_poisson7_16^3", 2: "c2_poisson7_128^3_u01", 3: "c3_aniso7_256^3_2x2sweeps",
            4: "c4_poisson7_256^3_per_gpu_weak", 5: "c5_jump27_512^3"}[cfg] + f"_grid{grid[0]}x{grid[1]}x{grid[2]}"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        under = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(under) if under else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ dist
def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "gloo" if args.impl == "reference" else "nccl"
        dist.init_process_group(backend=backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allmax(world, v):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ oracle
def oracle_sample(rtol, nsolves=1):
    """The CPU oracle, as it stands, on a bounded sample of the workload family:
    the same 7-point generator and settings on a 96^3 grid (b = 1)."""
    import oracle as O
    from inputs import poisson7
    A = poisson7(*CPU_SAMPLE_GRID)
    t0 = time.perf_counter()
    h = O.OracleHierarchy(A)
    setup = time.perf_counter() - t0
    b = np.ones(A.n_global)
    times, its = [], []
    for _ in range(nsolves):
        t0 = time.perf_counter()
        _, info = h.pcg(b, rtol=rtol, maxit=500)
        times.append(time.perf_counter() - t0)
        its.append(info["iterations"])
    return A.n_global, setup, times, its


def run_reference(args):
    world, rank, _ = dist_init(args)
    if rank != 0:
        return 0
    n, setup, times, its = oracle_sample(args.rtol, args.warmup + args.steps)
    timed = times[args.warmup:]
    sec = sum(timed) / len(timed)
    value = n / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config, (256, 256, 256 * args.gpus)),
                   "sample": f"oracle PCG solve of the {CPU_SAMPLE_GRID} grid of the same generator",
                   "rtol": args.rtol},
        "iterations": its[-1],
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"single-thread fp64 C oracle, full PCG solve on {CPU_SAMPLE_GRID} "
                                   f"(setup {setup:.1f} s untimed)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ ours
def method_settings(args, meta, world):
    """--method default: the north_star path (PCG, l1-Jacobi with the config's sweeps, direct
    coarsest, maxsize 200*np).  --method va3s5cs1: the paper's own GPU method:
    FCG(1), 4/4 l1-Jacobi sweeps, coarsest CG + l1-Jacobi to 1e-4 / 30 its,
    maxsize 12*200*np.  --method ka1: the paper's KA1 hierarchy with the K-cycle
    (PAPER.md:136, 277-312): unsmoothed 3-sweep matching, two inner FCG(1) iterations per
    intermediate level, FCG(1) outer solver, l1-Jacobi sweeps of the config."""
    if args.method == "va3s5cs1":
        return {"name": "va3s5cs1", "desc": "3 matching sweeps/level, smoothed P (omega=4/3/||D^-1A||), "
                                            "FCG(1), coarsest l1-Jacobi CG (1e-4, 30 its)",
                "cfg": dict(pre_sweeps=4, post_sweeps=4, max_coarse_size=12 * 200 * world, krylov=1,
                            coarse_solver=1, coarse_rtol=1e-4, coarse_maxit=30)}
    if args.method == "invk":
        return {"name": "invk", "desc": "3 matching sweeps/level, smoothed P (omega=4/3/||D^-1A||), INVK smoother "
                                        "(IC(0) + 1 level of fill in the inversion), PCG, direct coarsest",
                "cfg": dict(pre_sweeps=meta["sweeps"][0], post_sweeps=meta["sweeps"][1],
                            max_coarse_size=meta["max_coarse_size"], smoother=1, invk_fill=1)}
    if args.method == "ka1":
        return {"name": "ka1", "desc": "3 matching sweeps/level, unsmoothed P, K-cycle (2 inner FCG(1) "
                                       "iterations per intermediate level), FCG(1), direct coarsest",
                "cfg": dict(pre_sweeps=meta["sweeps"][0], post_sweeps=meta["sweeps"][1],
                            max_coarse_size=meta["max_coarse_size"], smooth_prolongator=0, cycle=1, krylov=1)}
    return {"name": "default", "desc": "3 matching sweeps/level, smoothed P (omega=4/3/||D^-1A||), PCG, "
                                       "direct coarsest",
            "cfg": dict(pre_sweeps=meta["sweeps"][0], post_sweeps=meta["sweeps"][1],
                        max_coarse_size=meta["max_coarse_size"])}


def run_ours(args):
    import torch

    world, rank, local = dist_init(args)
    if world != args.gpus:
        print(f"--gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    torch.cuda.set_device(local)
    import paper_2006_16147_b200 as amg
    from inputs import config_problem

    A, b, meta = config_problem(args.config, nranks=world, rank=rank, grid=args.grid)
    n_global = A.n_global
    stream = torch.cuda.Stream(device=local)
    uid = None
    if world > 1:
        import torch.distributed as dist
        obj = [amg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    ctx = amg.Context(device=local, rank=rank, nranks=world, nccl_uid=uid, stream=stream.cuda_stream)
    method = method_settings(args, meta, world)
    extra = {} if args.tail_rows is None else {"tail_rows": args.tail_rows}
    if args.tail_bytes is not None:
        extra["tail_bytes"] = args.tail_bytes
    cfg = amg.make_config(**method["cfg"], **extra)
    t0 = time.perf_counter()
    h = amg.Hierarchy(ctx, A, cfg=cfg)
    setup_s = time.perf_counter() - t0
    del A
    bt = torch.tensor(b, device=f"cuda:{local}")
    xt = torch.empty_like(bt)
    torch.cuda.synchronize()

    def solve():
        return h.solve_raw(bt.data_ptr(), xt.data_ptr(), rtol=args.rtol, maxit=args.maxit)

    for _ in range(args.warmup):
        rep = solve()
    clocks = ClockSampler(local)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    e0.record(stream)
    reps = []
    for _ in range(args.steps):
        reps.append(solve())
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ck = clocks.stop()
    ms_total = allmax(world, e0.elapsed_time(e1))
    ms_per_step = ms_total / args.steps
    iters = reps[-1]["iterations"]
    dev_solve_ms = allmax(world, 1e3 * statistics.mean(r["solve_s"] for r in reps))

    # V-cycle timing (graph-launched amg_precond_apply), SURVEY.md §8d
    napply = 20
    z = torch.empty_like(bt)
    h.precond_apply(bt, z)
    barrier(world)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(napply):
        amg.lib.amg_precond_apply(h.h, amg._abi.C.c_void_p(bt.data_ptr()), amg._abi.C.c_void_p(z.data_ptr()))
    e1.record(stream)
    torch.cuda.synchronize()
    t_v_ms = allmax(world, e0.elapsed_time(e1) / napply)
    hrep = h.report()
    bytes_v = hrep["vcycle_bytes_model"]
    bytes_it = hrep["iteration_bytes_model"]
    peak, peak_src = measured_peaks()

    # per-kernel timing (instrumented eager V-cycles on the same stream) -> dominant kernel
    prof = h.profile_vcycle(10)
    per_v = len(prof)
    dom = max(prof, key=lambda k: k["ms"])
    dom_gbs = dom["bytes"] / (dom["ms"] * 1e-3) / 1e9
    dom_stored_gbs = dom["stored_bytes"] / (dom["ms"] * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tr = json.load(f)
        traffic = tr.get(f"c{args.config}:{dom['name']}")

    # e2e through the public API with host buffers: every step copies its b host->device and
    # its x device->host; amg_solve_host_batch pipelines those copies with the solves
    bh = torch.tensor(b).pin_memory().numpy()
    Bh = torch.empty((args.steps, bh.shape[0]), dtype=torch.float64).pin_memory().numpy()
    Xh = torch.empty((args.steps, bh.shape[0]), dtype=torch.float64).pin_memory().numpy()
    Bh[:] = bh
    h.solve_host_batch(Bh[:min(2, args.steps)], Xh[:min(2, args.steps)], rtol=args.rtol, maxit=args.maxit)
    barrier(world)
    t0 = time.perf_counter()
    h.solve_host_batch(Bh, Xh, rtol=args.rtol, maxit=args.maxit)
    e2e_s = allmax(world, (time.perf_counter() - t0) / args.steps)

    # CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nS, setupS, timesS, itsS = oracle_sample(args.rtol, 1)
        cpu = {"value": nS / timesS[0], "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"single-thread fp64 C oracle, one full PCG solve ({itsS[0]} its) on the "
                         f"{CPU_SAMPLE_GRID} grid of the same generator, setup {setupS:.1f} s untimed"}

    if rank == 0:
        value = n_global / (ms_per_step * 1e-3)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(args.config, meta["grid"]), "n_global": n_global,
                       "grid": list(meta["grid"]), "partition": f"z-slabs x{world}",
                       "rtol": args.rtol, "method": method["name"],
                       "sweeps": f"{method['cfg']['pre_sweeps']}/{method['cfg']['post_sweeps']}",
                       "hierarchy": method["desc"],
                       "max_coarse_size": method["cfg"]["max_coarse_size"], "rhs": meta["rhs"],
                       "l2_policy": "inputs larger than L2 (hierarchy >> 126 MB), no flush",
                       "parallelism": f"rowblock{world}"},
            "solve_s": ms_per_step * 1e-3, "device_solve_s": dev_solve_ms * 1e-3, "iterations": iters,
            "ms_per_iter": ms_per_step / max(iters, 1), "setup_s": setup_s,
            "levels": h.sizes(), "opc": hrep["opc"],
            "vcycle": {"ms": t_v_ms, "bytes_model": bytes_v, "GBps": bytes_v / (t_v_ms * 1e-3) / 1e9,
                       "frac_of_8TBps": bytes_v / (t_v_ms * 1e-3) / 1e9 / NOMINAL_HBM_GBS,
                       "frac_of_measured": bytes_v / (t_v_ms * 1e-3) / 1e9 / peak},
            "iteration_bytes_model": bytes_it,
            "roofline": {"bound": "hbm", "kernel": dom["name"], "achieved": dom_gbs, "peak": peak,
                         "unit": "GB/s", "frac": dom_gbs / peak, "traffic": traffic,
                         "bytes_per_launch": dom["bytes"], "ms_per_launch": dom["ms"],
                         "stored_bytes_per_launch": dom["stored_bytes"],
                         "achieved_stored_GBps": dom_stored_gbs, "frac_stored": dom_stored_gbs / peak,
                         "note": "achieved uses SURVEY 8(d) algorithmic bytes (12 B/nnz); SDIA-32 stores no "
                                 "per-entry column index, so the compulsory (stored) bytes are smaller",
                         "share_of_vcycle": dom["ms"] / sum(k["ms"] for k in prof),
                         "peak_source": peak_src,
                         "timing": "CUDA events on the solve stream, instrumented V-cycles after the timed region"},
            "kernels_per_vcycle": [(k["name"], round(k["ms"], 4), round(k["bytes"] / (k["ms"] * 1e-3) / 1e9, 1),
                                    round(k["stored_bytes"] / (k["ms"] * 1e-3) / 1e9, 1)) for k in prof],
            "vcycle_stored_bytes": sum(k["stored_bytes"] for k in prof),
            "cpu_baseline": cpu,
            "e2e": {"value": n_global / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * bh.shape[0] * world,
                    "d2h_bytes_per_step": 8 * bh.shape[0] * world, "s_per_step": e2e_s,
                    "api": "amg_solve_host_batch (pinned host b/x per step, copies pipelined with the solves)"},
            # per solve: prologue + per iteration (cycle kernels + q = A p [+ p-update] + r-update)
            # + the deferred final x update; single-rank PCG fuses the p-update into q = A p
            "gpu_launches": args.steps * (2 + iters * (per_v + (2 if (method["cfg"].get("krylov", 0) == 0
                                                                    and world == 1) else 3))),
            "clocks": ck,
        }
        print(json.dumps(line), flush=True)
    h.close()
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--grid", type=lambda s: tuple(int(v) for v in s.split("x")), default=None)
    ap.add_argument("--rtol", type=float, default=1e-6)
    ap.add_argument("--maxit", type=int, default=500)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--method", choices=["default", "va3s5cs1", "ka1", "invk"], default="default")
    ap.add_argument("--tail-rows", type=int, default=None, help="override cfg.tail_rows (0 = no persistent tail)")
    ap.add_argument("--tail-bytes", type=int, default=None, help="override cfg.tail_bytes (0 = no cluster tail)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    sys.exit(run_reference(args) if args.impl == "reference" else run_ours(args))


if __name__ == "__main__":
    main()
