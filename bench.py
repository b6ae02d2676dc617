#!/usr/bin/env python3
"""Benchmark: Lorenz Taylor steps/sec at (N, K) and limb-MAC/s vs the INT roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload k500] [--impl b200|reference]

One bench step = one launch of the persistent kernel advancing every
trajectory by S Taylor steps (S = --taylor-steps, default 100 = one time unit
at tau = 0.01) over inputs already resident in HBM. The default workload is
BASELINE.json configs[1] (K = 500 digits, N = 200, tau = 0.01, one
trajectory per GPU). With N > 1 GPUs (torchrun) every rank integrates its own
trajectory (initial condition perturbed by rank * 1e-20: an ensemble, weak
scaling, no collective on the data path); final states are gathered with NCCL
after the timed region.

Outputs one JSON line (rank 0). See DESIGN.md §6 for every field.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from fractions import Fraction

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "Lorenz Taylor steps/sec at (N,K) and limb-MAC/s as fraction of INT roofline"
INIT = ("-15.8", "-17.48", "35.64")

# name -> (K digits, order N, tau, trajectories per GPU, default Taylor steps per bench step, label)
WORKLOADS = {
    "k50": (50, 40, "0.01", 1, 100, "configs[0]: K=50 N=40 tau=0.01, single trajectory"),
    "k500": (500, 200, "0.01", 1, 100, "configs[1]: K=500 N=200 tau=0.01, single trajectory"),
    "k2200": (2200, 1000, "0.01", 1, 5, "configs[2]: K=2200 N=1000 tau=0.01, single trajectory"),
    "k4200": (4200, 3500, "0.01", 1, 1, "configs[3]: K=4200 N=3500 tau=0.01, single trajectory"),
    "ens100": (100, 60, "0.01", 4096, 10, "configs[4]: ensemble M=4096 at (K,N)=(100,60)"),
    "ens200": (200, 120, "0.01", 4096, 5, "configs[4]: ensemble M=4096 at (K,N)=(200,120)"),
    "ens400": (400, 240, "0.01", 4096, 2, "configs[4]: ensemble M=4096 at (K,N)=(400,240)"),
    "ens800": (800, 480, "0.01", 4096, 1, "configs[4]: ensemble M=4096 at (K,N)=(800,480)"),
}


def bits_for_digits(d: int) -> int:
    from paper_1908_09301_b200.mp import bits_for_digits as b

    return b(d)


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ workload
def build_workload(name, rank, world):
    import numpy as np

    import paper_1908_09301_b200 as M
    from paper_1908_09301_b200.engine import SystemTables
    from paper_1908_09301_b200.fixed import FixedFormat

    K, N, tau_text, n_traj, S, label = WORKLOADS[name]
    P = bits_for_digits(K)
    ctx = M.PrecisionContext(P)
    system = M.builtin_system("lorenz", ctx)
    fmt = FixedFormat(P)
    tau = M.mp_from_decimal(tau_text, ctx)
    tables = SystemTables.build(system, fmt, N, tau.as_fraction())
    base = [M.mp_from_decimal(t, ctx).as_fraction() for t in INIT]
    if n_traj > 1:  # ensemble: strong scaling over a fixed total
        per = (n_traj + world - 1) // world
        lo, hi = rank * per, min(n_traj, (rank + 1) * per)
        import random

        rnd = random.Random(0)
        pert = [[Fraction(rnd.randint(-10**6, 10**6), 10**26) for _ in range(3)] for _ in range(n_traj)]
        ids = range(lo, hi)
    else:  # one trajectory per GPU: weak scaling
        pert = {rank: [Fraction(rank, 10**20)] * 3}
        ids = [rank]
    states = np.stack([fmt.to_digits([b + d for b, d in zip(base, pert[j])]) for j in ids])
    return dict(name=name, K=K, N=N, P=P, tau_text=tau_text, n_total=n_traj if n_traj > 1 else world,
                n_local=len(states), S=S, label=label, ctx=ctx, system=system, fmt=fmt, tables=tables,
                states=states, strong=n_traj > 1)


# --------------------------------------------------------------- cpu legs
def cpu_rate(w, seconds: float, threads: int, threshold: int = 256, max_steps: int = 10**6):
    """Reference-semantics oracle (C + MPFR, bit-identical to the reference) on
    the host: Taylor steps/s of one trajectory, bounded sample."""
    from oracle import ref as R

    P, N = w["P"], w["N"]
    system = R.lorenz(P)
    state = [R.from_decimal(t, P) for t in INIT]
    tau = R.from_decimal(w["tau_text"], P)
    n = 1
    while True:  # grow the sample until it takes >= seconds
        t0 = time.perf_counter()
        R.integrate(system, state, tau, N, n, P, stride=n, threads=threads, threshold=threshold)
        dt = time.perf_counter() - t0
        if dt >= seconds or n >= max_steps:
            return n / dt, n, dt
        n = min(max_steps, max(n * 2, int(n * seconds / max(dt, 1e-3) * 1.1)))


# ------------------------------------------------------------------ main legs
def run_reference(args, rank, world):
    if rank != 0:
        return None
    w = build_workload(args.workload, 0, 1)
    ncpu = os.cpu_count() or 1
    # the reference's parallel reduction engages from the serial threshold on
    # (default 256); for orders below it the plain serial loop runs. Warm-up
    # tries the default plan and an all-threads plan (threshold 32) and keeps
    # the faster one -- the reference arm is given its best configuration.
    candidates = [(1, 256)] + ([(ncpu, 256), (ncpu, 32)] if ncpu > 1 else [])
    best = None
    for _ in range(args.warmup):
        for threads, threshold in candidates:
            rate = cpu_rate(w, min(2.0, args.cpu_seconds / 4), threads, threshold)[0]
            if best is None or rate > best[0]:
                best = (rate, threads, threshold)
    _, threads, threshold = best
    samples = []
    for _ in range(args.steps):
        rate, n, dt = cpu_rate(w, args.cpu_seconds / max(1, args.steps), threads, threshold)
        samples.append((rate, n, dt))
    total_n = sum(s[1] for s in samples)
    total_t = sum(s[2] for s in samples)
    value = total_n / total_t
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "taylor_steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "mpfr (binary, RNDN)",
        "data": "synthetic: Lorenz initial condition (-15.8,-17.48,35.64)",
        "config": {"workload": w["label"], "K_digits": w["K"], "order": w["N"], "prec_bits": w["P"],
                   "tau": w["tau_text"]},
        "cpu_baseline": {"value": value, "unit": "taylor_steps/s", "cores": threads, "kind": "port",
                         "sample": f"{total_n} Taylor steps of one trajectory over {args.steps} samples; "
                                   f"oracle/mpfr_ref.c (C restatement of the reference on MPFR, "
                                   f"bit-identical to it), OpenMP {threads} threads, 64 chunks, "
                                   f"serial threshold {threshold}"},
        "e2e": {"value": value, "unit": "taylor_steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    return line


def run_b200(args, rank, world, local_rank):
    import numpy as np

    import paper_1908_09301_b200 as M
    from paper_1908_09301_b200 import _native
    from paper_1908_09301_b200.engine import DevicePlan

    lib = _native.load()
    device = local_rank
    w = build_workload(args.workload, rank, world)
    S = args.taylor_steps or w["S"]
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(device)
        dist.init_process_group("nccl")

    def barrier():
        if dist is not None:
            dist.barrier()

    # integer-pipe roofline probe (measured live)
    import ctypes

    peak = ctypes.c_double()
    pms = ctypes.c_float()
    _native.check(lib.mpt_imad_probe(device, ctypes.byref(peak), ctypes.byref(pms)))

    plan = DevicePlan(w["tables"], w["fmt"], w["N"], w["n_local"], device)
    kinfo = plan.info()
    plan.upload(w["states"])
    # warm-up; the last warm-up launch counts limb-MACs for the roofline
    for k in range(args.warmup):
        if k == args.warmup - 1:
            plan.count_macs(True)
        plan.run_device(S)
        plan.last_kernel_ms()
    useful, executed = plan.read_macs()
    plan.count_macs(False)
    flush = 256 << 20

    launch_ms = []
    barrier()
    with ClockSampler(device) as clocks:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            _native.check(lib.mpt_l2_flush(device, flush))  # outside the kernel's event bracket
            plan.run_device(S)
            launch_ms.append(plan.last_kernel_ms())
        wall = time.perf_counter() - t0
    barrier()
    dev_ms = sum(launch_ms)
    final = plan.download()
    if dist is not None:
        import torch

        t = torch.tensor([dev_ms, wall], dtype=torch.float64, device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms_max, wall_max = t.tolist()
        # gather the trajectories' final states (NCCL over NVLink)
        ft = torch.from_numpy(final.astype(np.int32)).to(f"cuda:{device}")
        sizes = [torch.zeros(1, dtype=torch.int64, device=f"cuda:{device}") for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([ft.numel()], device=f"cuda:{device}"))
        maxn = int(max(s.item() for s in sizes))
        pad = torch.zeros(maxn, dtype=torch.int32, device=f"cuda:{device}")
        pad[: ft.numel()] = ft.flatten()
        bufs = [torch.zeros_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad)
    else:
        dev_ms_max, wall_max = dev_ms, wall
    plan.close()

    total_steps = args.steps * S * (w["n_total"])
    value = total_steps / (dev_ms_max * 1e-3)
    avg_launch_s = dev_ms / args.steps * 1e-3
    achieved = useful / avg_launch_s
    line = None
    if rank == 0:
        # ---- e2e: the public drop-in API with host MPValues (plan setup, H2D, kernel, D2H)
        e2e = None
        if not args.no_e2e and w["strong"]:
            # ensemble: the public ensemble entry point with host decimal initial conditions
            # (parse -> digits -> H2D -> kernel -> D2H of the recorded states), this rank's shard
            from paper_1908_09301_b200 import ensemble as E

            lo, hi = E.shard_bounds(w["n_total"], world, rank)
            inits = E.perturbed_inits(w["n_total"], seed=0)[lo:hi]
            reps = max(1, min(args.steps, args.e2e_reps))
            E.run_members("lorenz", inits, w["P"], w["N"], w["tau_text"], S, S, device=device)  # warm
            t0 = time.perf_counter()
            for _ in range(reps):
                E.run_members("lorenz", inits, w["P"], w["N"], w["tau_text"], S, S, device=device)
            dt = (time.perf_counter() - t0) / reps
            RS, D, N, M = (w["fmt"].width + 3) // 4 * 4, 3, w["N"], hi - lo
            h2d = 4 * RS * (D + D * D + 2 + N) + 4 * RS * D * M
            d2h = 4 * w["fmt"].width * D * M * 2 + 4 * M  # records at steps 0 and S, status
            e2e = {"value": S * M * world / dt, "unit": "taylor_steps/s", "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h,
                   "how": f"paper_1908_09301_b200.ensemble.run_members(...) of {S} Taylor steps on {M} "
                          f"members (decimal inits, seed 0), wall clock incl. parsing and plan setup, mean "
                          f"of {reps}; x{world} ranks"}
        elif not args.no_e2e:
            ctx, system = w["ctx"], w["system"]
            st = tuple(M.MPValue.from_fraction(f, w["P"]) for f in w["fmt"].digits_to_fractions(w["states"][0]))
            cfg = M.StepConfig(w["tau_text"], w["N"])
            reps = max(1, min(args.steps, args.e2e_reps))
            M.integrate(system, st, cfg, S, ctx, record_stride=S)  # warm
            t0 = time.perf_counter()
            for _ in range(reps):
                traj = M.integrate(system, st, cfg, S, ctx, record_stride=S)
            dt = (time.perf_counter() - t0) / reps
            W, RS, D, N = w["fmt"].width, (w["fmt"].width + 3) // 4 * 4, 3, w["N"]
            h2d = 4 * W * D  # the state digits (integrate() caches its plan: constants uploaded once)
            d2h = 4 * RS * D * 1 + 4 * 1  # one record + status
            e2e = {"value": S / dt, "unit": "taylor_steps/s", "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h,
                   "how": f"paper_1908_09301_b200.integrate(...) of {S} Taylor steps on one trajectory, "
                          f"host MPValues in/out, wall clock incl. table build + plan-cache lookup, mean of {reps}"}
        cpu = None
        if not args.no_cpu_baseline:
            rate, n, dt = cpu_rate(w, args.cpu_seconds, 1)
            cpu = {"value": rate, "unit": "taylor_steps/s", "cores": 1, "kind": "port",
                   "sample": f"{n} Taylor steps of one trajectory in {dt:.1f}s: oracle/mpfr_ref.c "
                             f"(C restatement of the reference hot path on MPFR, bit-identical to the "
                             f"reference), 1 thread (reference default plan: N < serial threshold 256)"}
        prof = os.path.join(REPO, "profiles", f"traffic_{args.workload}.json")
        traffic = None
        if os.path.exists(prof):
            with open(prof) as fh:
                traffic = json.load(fh).get("dram_bytes_per_launch")
        line = {
            "metric": METRIC, "value": value, "unit": "taylor_steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong" if w["strong"] else "weak",
            "vs_baseline": None, "dtype": "int32 digits (radix 2^28) x int32 -> int64 accumulate",
            "data": "synthetic: Lorenz initial condition (-15.8,-17.48,35.64)"
                    + (" + seeded perturbations" if w["strong"] or world > 1 else ""),
            "config": {"workload": w["label"], "K_digits": w["K"], "order": w["N"], "prec_bits": w["P"],
                       "frac_bits": w["fmt"].frac_bits, "tau": w["tau_text"], "taylor_steps_per_bench_step": S,
                       "trajectories_total": w["n_total"], "trajectories_per_gpu": w["n_local"],
                       "l2": "flushed between timed launches (256 MiB memset, outside the kernel events)",
                       "kernel": kinfo["kernel"], "cluster_ctas": kinfo["cluster"],
                       "parallelism": (f"ensemble sharded over {world} GPUs" if w["strong"]
                                       else f"one trajectory per GPU ({world} replicas, weak)")},
            "roofline": {"bound": "int", "achieved": achieved, "peak": peak.value, "unit": "limb-MAC/s",
                         "frac": achieved / peak.value, "traffic": traffic,
                         "peak_source": "measured live: IMAD.WIDE (s64 += s32*s32) probe kernel, whole device",
                         "useful_limb_macs_per_launch": useful, "executed_limb_macs_per_launch": executed},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": args.steps, "clocks": clocks.summary(),
            "wall_ms_timed_region": wall_max * 1e3,
        }
    if dist is not None:
        dist.destroy_process_group()
    return line


def main():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="k500")
    ap.add_argument("--taylor-steps", type=int, default=0, dest="taylor_steps")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, dest="cpu_seconds")
    ap.add_argument("--e2e-reps", type=int, default=3, dest="e2e_reps")
    ap.add_argument("--no-e2e", action="store_true", dest="no_e2e")
    ap.add_argument("--no-cpu-baseline", action="store_true", dest="no_cpu_baseline")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and "RANK" in os.environ:
        print(f"warning: WORLD_SIZE={world} != --gpus {args.gpus}", file=sys.stderr)
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        line = run_b200(args, rank, world, local_rank)
    if line is not None and rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
