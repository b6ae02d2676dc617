#!/usr/bin/env python3
"""Benchmark: Lorenz Taylor steps/sec at (N, K) and limb-MAC/s vs the INT roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload k500] [--impl b200|reference]

One bench step = one launch of the persistent kernel advancing every
trajectory by S Taylor steps (S = --taylor-steps, default 100 = one time unit
at tau = 0.01) over inputs already resident in HBM. At N = 1 the default
workload is BASELINE.json configs[1] (K = 500 digits, N = 200, tau = 0.01, one
trajectory). At N > 1 the default is the configs[4] ensemble at (K, N) =
(100, 60): the M = 4096 seeded members are sharded over the ranks (strong
scaling, no collective on the data path), one bench step advances every
member's base run (K, N) AND its verify run (K+50, N+30) by S steps, and x, y,
z and t_c are gathered with NCCL after the timed region (ensemble.tc_sweep is
the e2e leg). `--workload ens100 --gpus 1` gives the 1-GPU point of that curve.

N > 1 ranks: under torchrun the RANK/WORLD_SIZE environment is used; started
plainly (`python bench.py --gpus N`) the script spawns its own N ranks on
127.0.0.1.

Outputs one JSON line (rank 0). See DESIGN.md §5 for every field.
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
# (ensemble launches are long enough to be past the start-up transient: the first steps from the canonical
# initial condition are 10-15 % cheaper than the sustained rate)
WORKLOADS = {
    "k50": (50, 40, "0.01", 1, 100, "configs[0]: K=50 N=40 tau=0.01, single trajectory"),
    "k500": (500, 200, "0.01", 1, 100, "configs[1]: K=500 N=200 tau=0.01, single trajectory"),
    "k2200": (2200, 1000, "0.01", 1, 5, "configs[2]: K=2200 N=1000 tau=0.01, single trajectory"),
    "k4200": (4200, 3500, "0.01", 1, 1, "configs[3]: K=4200 N=3500 tau=0.01, single trajectory"),
    "ens100": (100, 60, "0.01", 4096, 100, "configs[4]: ensemble M=4096 at (K,N)=(100,60)"),
    "ens200": (200, 120, "0.01", 4096, 50, "configs[4]: ensemble M=4096 at (K,N)=(200,120)"),
    "ens400": (400, 240, "0.01", 4096, 20, "configs[4]: ensemble M=4096 at (K,N)=(400,240)"),
    "ens800": (800, 480, "0.01", 4096, 2, "configs[4]: ensemble M=4096 at (K,N)=(800,480)"),
}


VERIFY_MARGIN = (50, 30)  # configs[4]: each member is checked against its own (K+50, N+30) run
# Taylor steps of the ensemble e2e call (ensemble.tc_sweep), sized for seconds of device time
E2E_STEPS = {"ens100": 1000, "ens200": 300, "ens400": 50, "ens800": 8}


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
    from paper_1908_09301_b200 import ensemble as E
    from paper_1908_09301_b200.engine import SystemTables
    from paper_1908_09301_b200.fixed import FixedFormat

    K, N, tau_text, n_traj, S, label = WORKLOADS[name]

    def leg(K, N, inits=None):
        P = bits_for_digits(K)
        ctx = M.PrecisionContext(P)
        system = M.builtin_system("lorenz", ctx)
        fmt = FixedFormat(P)
        tau = M.mp_from_decimal(tau_text, ctx)
        tables = SystemTables.build(system, fmt, N, tau.as_fraction())
        if inits is None:  # one trajectory per GPU (weak scaling): the canonical point + rank * 1e-20
            base = [M.mp_from_decimal(t, ctx).as_fraction() for t in INIT]
            states = np.stack([fmt.to_digits([b + Fraction(rank, 10**20) for b in base])])
        else:
            states = E.states_from_decimals(inits, P, fmt)
        return dict(K=K, N=N, P=P, ctx=ctx, system=system, fmt=fmt, tables=tables, states=states)

    if n_traj > 1:  # ensemble: strong scaling over a fixed total, the e2e leg's own members
        lo, hi = E.shard_bounds(n_traj, world, rank)
        inits = E.perturbed_inits(n_traj, seed=0)[lo:hi]
        legs = [leg(K, N, inits), leg(K + VERIFY_MARGIN[0], N + VERIFY_MARGIN[1], inits)]
    else:
        legs = [leg(K, N)]
    w = dict(legs[0])
    w.update(name=name, tau_text=tau_text, n_total=n_traj if n_traj > 1 else world, n_local=len(legs[0]["states"]),
             S=S, label=label, strong=n_traj > 1, legs=legs)
    return w


# --------------------------------------------------------------- cpu legs
def cpu_rate(w, seconds: float, threads: int, threshold: int = 256, max_steps: int = 10**6, tau_text=None):
    """Reference-semantics oracle (C + MPFR, bit-identical to the reference) on
    the host: Taylor steps/s of one trajectory, bounded sample."""
    from oracle import ref as R

    P, N = w["P"], w["N"]
    system = R.lorenz(P)
    state = [R.from_decimal(t, P) for t in INIT]
    tau = R.from_decimal(tau_text or w["tau_text"], P)
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
        "note": "the reference itself is Python on gmpy2 (not installed in this image); this arm is its C/MPFR "
                "restatement (pinned bit for bit to the unmodified reference, including this chunked plan) with "
                "OpenMP over the reference's chunks, so it is FASTER than the reference's own loop and the GPU/"
                "reference ratio against it is conservative",
    }
    return line


def run_b200(args, rank, world, local_rank):
    import ctypes

    import numpy as np

    import paper_1908_09301_b200 as M
    from paper_1908_09301_b200 import _native
    from paper_1908_09301_b200 import ensemble as E
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
    peak = ctypes.c_double()
    pms = ctypes.c_float()
    _native.check(lib.mpt_imad_probe(device, ctypes.byref(peak), ctypes.byref(pms)))

    # one device plan per leg: the trajectory (configs 0-3), or the shard's base and verify runs (configs[4])
    plans = []
    for lg in w["legs"]:
        if w["n_local"] == 0:
            break
        plan = DevicePlan(lg["tables"], lg["fmt"], lg["N"], w["n_local"], device)
        plan.upload(lg["states"])
        plans.append(plan)
    kinfo = plans[0].info() if plans else {"kernel": "none", "cluster": 0}
    # warm-up; the last warm-up launch counts limb-MACs for the roofline
    for k in range(args.warmup):
        for plan in plans:
            if k == args.warmup - 1:
                plan.count_macs(True)
            plan.run_device(S)
            plan.last_kernel_ms()
    useful = executed = 0
    for plan in plans:
        u, x = plan.read_macs()
        useful, executed = useful + u, executed + x
        plan.count_macs(False)
    flush = 256 << 20

    launch_ms = []
    barrier()
    with ClockSampler(device) as clocks:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ms = 0.0
            for plan in plans:
                _native.check(lib.mpt_l2_flush(device, flush))  # outside the kernel's event bracket
                plan.run_device(S)
                ms += plan.last_kernel_ms()
            launch_ms.append(ms)
        wall = time.perf_counter() - t0
    barrier()
    dev_ms = sum(launch_ms)
    finals = [plan.download() for plan in plans]
    n_comm = 1
    if dist is not None:
        import torch

        t = torch.tensor([dev_ms, wall], dtype=torch.float64, device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms_max, wall_max = t.tolist()
        n_comm = dist.get_world_size()
        # gather the trajectories' final states (NCCL over NVLink), after the timed region
        W0 = w["legs"][0]["fmt"].width
        local = finals[0].astype(np.int32) if finals else np.zeros((0, 3, W0), np.int32)
        if w["strong"]:
            gathered = E.gather_rows(local, w["n_total"], world, rank, f"cuda:{device}")
        else:
            gathered = E.gather_rows(local, world, world, rank, f"cuda:{device}")
        assert gathered.shape[0] == w["n_total"]
    else:
        dev_ms_max, wall_max = dev_ms, wall
    for plan in plans:
        plan.close()

    nlegs = len(w["legs"])
    total_steps = args.steps * S * w["n_total"] * nlegs
    value = total_steps / (dev_ms_max * 1e-3)
    avg_launch_s = dev_ms / args.steps * 1e-3 if dev_ms > 0 else float("inf")
    achieved = useful * (world if w["strong"] else 1) / avg_launch_s
    line = None
    e2e = None
    if not args.no_e2e and w["strong"]:
        # ensemble: the public sweep entry point on every rank -- decimal initial conditions of the
        # rank's shard (parse -> digits -> H2D), base + verify runs, D2H of the records, agreement
        # digits, t_c, and the gather of x, y, z, t_c over all ranks
        K, N = w["legs"][0]["K"], w["legs"][0]["N"]
        Se = args.e2e_steps or E2E_STEPS.get(w["name"], S)
        kw = dict(rank=rank, world=world, device=device, tau_text=w["tau_text"], stride=min(Se, 100),
                  gather_device=f"cuda:{device}" if dist is not None else None)
        E.tc_sweep(K, N, w["n_total"], Se, **kw)  # warm (plan cache, allocator)
        reps = max(1, min(args.steps, args.e2e_reps))
        barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            rep = E.tc_sweep(K, N, w["n_total"], Se, **kw)
        barrier()
        dt = (time.perf_counter() - t0) / reps
        Mloc = w["n_local"]
        h2d = sum(4 * ((lg["fmt"].width + 3) // 4 * 4) * 3 * Mloc for lg in w["legs"])
        nrec = Se // min(Se, 100) + 1
        d2h = sum(4 * lg["fmt"].width * 3 * Mloc * nrec + 4 * Mloc for lg in w["legs"])
        e2e = {"value": nlegs * Se * w["n_total"] / dt, "unit": "taylor_steps/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "bytes_are": "per tc_sweep call and rank",
               "how": f"paper_1908_09301_b200.ensemble.tc_sweep(K={K}, N={N}, M={w['n_total']}, {Se} Taylor steps): "
                      f"decimal inits (seed 0) -> base + verify runs -> agreement digits -> t_c -> gather; "
                      f"wall clock on {world} rank(s), mean of {reps}; mean t_c {rep.tc_mean():.2f}"}
    if rank == 0:
        # ---- e2e: the public drop-in API with host MPValues (plan lookup, H2D, kernel, D2H)
        if not args.no_e2e and not w["strong"]:
            ctx, system = w["ctx"], w["system"]
            st = tuple(M.MPValue.from_fraction(f, w["P"]) for f in w["fmt"].digits_to_fractions(w["states"][0]))
            cfg = M.StepConfig(w["tau_text"], w["N"])
            reps = max(1, min(args.steps, args.e2e_reps))
            M.integrate(system, st, cfg, S, ctx, record_stride=S)  # warm
            t0 = time.perf_counter()
            for _ in range(reps):
                M.integrate(system, st, cfg, S, ctx, record_stride=S)
            dt = (time.perf_counter() - t0) / reps
            W, RS, D = w["fmt"].width, (w["fmt"].width + 3) // 4 * 4, 3
            h2d = 4 * W * D  # the state digits (integrate() caches its plan: constants uploaded once)
            d2h = 4 * RS * D * 1 + 4 * 1  # one record + status
            e2e = {"value": S / dt, "unit": "taylor_steps/s", "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h, "bytes_are": f"per integrate() call of {S} Taylor steps",
                   "how": f"paper_1908_09301_b200.integrate(...) of {S} Taylor steps on one trajectory, "
                          f"host MPValues in/out, wall clock incl. table build + plan-cache lookup, mean of {reps}"}
        cpu = None
        if not args.no_cpu_baseline:
            rates = [cpu_rate(lg, args.cpu_seconds / nlegs, 1, tau_text=w["tau_text"]) for lg in w["legs"]]
            rate = nlegs / sum(1.0 / r[0] for r in rates)
            cpu = {"value": rate, "unit": "taylor_steps/s", "cores": 1, "kind": "port",
                   "sample": "; ".join(f"{n} Taylor steps of one trajectory at (K,N)=({lg['K']},{lg['N']}) in {dt:.1f}s"
                                       for lg, (_, n, dt) in zip(w["legs"], rates))
                             + ": oracle/mpfr_ref.c (C restatement of the reference hot path on MPFR, bit-identical "
                               "to the reference), 1 thread (reference default plan: N < serial threshold 256)"}
        prof = os.path.join(REPO, "profiles", f"traffic_{args.workload}.json")
        traffic = None
        if os.path.exists(prof):
            with open(prof) as fh:
                traffic = json.load(fh).get("dram_bytes_per_launch")
        cfgd = {"workload": w["label"], "K_digits": w["K"], "order": w["N"], "prec_bits": w["P"],
                "frac_bits": w["fmt"].frac_bits, "tau": w["tau_text"], "taylor_steps_per_bench_step": S,
                "trajectories_total": w["n_total"], "trajectories_per_gpu": w["n_local"],
                "l2": "flushed between timed launches (256 MiB memset, outside the kernel events)",
                "kernel": kinfo["kernel"], "cluster_ctas": kinfo["cluster"],
                "parallelism": (f"ensemble sharded over {world} GPUs, NCCL communicator of {n_comm} ranks "
                                f"(final gather only)" if w["strong"]
                                else f"one trajectory per GPU ({world} replicas, weak)")}
        if w["strong"]:
            v = w["legs"][1]
            cfgd["verify"] = {"K_digits": v["K"], "order": v["N"], "prec_bits": v["P"]}
            cfgd["counts"] = "Taylor steps of the base AND the verify run of every member"
        line = {
            "metric": METRIC, "value": value, "unit": "taylor_steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong" if w["strong"] else "weak",
            "vs_baseline": None, "dtype": "int32 digits (radix 2^28) x int32 -> int64 accumulate",
            "data": "synthetic: Lorenz initial condition (-15.8,-17.48,35.64)"
                    + (" + seeded perturbations" if w["strong"] or world > 1 else ""),
            "config": cfgd,
            "roofline": {"bound": "int", "achieved": achieved, "peak": peak.value * world, "unit": "limb-MAC/s",
                         "frac": achieved / (peak.value * world), "traffic": traffic,
                         "peak_source": "measured live: IMAD.WIDE (s64 += s32*s32) probe kernel, whole device"
                                        + (f" x {world} GPUs" if world > 1 else ""),
                         "useful_limb_macs_per_launch": useful, "executed_limb_macs_per_launch": executed},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": args.steps * len(plans), "clocks": clocks.summary(),
            "wall_ms_timed_region": wall_max * 1e3,
        }
    if dist is not None:
        dist.destroy_process_group()
    return line


def run_selftest_cpu(args, rank, world):
    """The multi-rank plumbing of this script on CPU (no GPU, gloo): spawn ->
    rendezvous on 127.0.0.1 -> ensemble.tc_sweep over the rank's shard with a
    synthetic run function -> gather -> one JSON line from rank 0."""
    import numpy as np
    import torch.distributed as dist

    from paper_1908_09301_b200 import ensemble as E
    from paper_1908_09301_b200.fixed import FixedFormat

    if world > 1:
        dist.init_process_group("gloo")

    def fake_run(inits, bits, order, tau_text, n_steps, stride):
        fmt = FixedFormat(bits)
        st = E.states_from_decimals(inits, bits, fmt)
        nrec = n_steps // stride + 1
        recs = np.repeat(st[None], nrec, axis=0).copy()
        drift = (np.arange(nrec) * (1 + order))[:, None, None]  # precision/order dependent low digits
        recs[..., fmt.width // 2] = (recs[..., fmt.width // 2] + drift * np.sign(recs[..., -1])) % (1 << 27) * np.sign(recs[..., -1])
        return E.EnsembleRun(bits, order, tau_text, fmt, np.arange(nrec, dtype=np.int32) * stride, recs,
                             np.zeros(len(inits), np.int32))

    M_total = 11
    t0 = time.perf_counter()
    rep = E.tc_sweep(40, 20, M_total, 400, rank=rank, world=world, stride=100, run_fn=fake_run)
    dt = time.perf_counter() - t0
    ok = rep.final_digits.shape[0] == M_total and rep.tc_step.shape == (M_total,)
    n_comm = dist.get_world_size() if world > 1 else 1
    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return None
    return {"metric": METRIC, "selftest_cpu": True, "ok": bool(ok), "n_gpus": world, "communicator_ranks": n_comm,
            "members_gathered": int(rep.final_digits.shape[0]), "seconds": dt, "value": None, "unit": "taylor_steps/s"}


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` without a launcher: start N ranks of this script
    (RANK/LOCAL_RANK/WORLD_SIZE/MASTER_ADDR/MASTER_PORT set), rank 0 owns stdout."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(args.gpus),
                   LOCAL_WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), *sys.argv[1:]], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    rc = 0
    for p in procs:
        rc = max(rc, abs(p.wait()))
    return rc


def main():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=None,
                    help="default: k500 (configs[1]) on one GPU, ens100 (configs[4]) on several")
    ap.add_argument("--taylor-steps", type=int, default=0, dest="taylor_steps")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, dest="cpu_seconds")
    ap.add_argument("--e2e-reps", type=int, default=3, dest="e2e_reps")
    ap.add_argument("--e2e-steps", type=int, default=0, dest="e2e_steps")
    ap.add_argument("--no-e2e", action="store_true", dest="no_e2e")
    ap.add_argument("--no-cpu-baseline", action="store_true", dest="no_cpu_baseline")
    ap.add_argument("--selftest-cpu", action="store_true", dest="selftest_cpu",
                    help="exercise the multi-rank plumbing on CPU (gloo, synthetic run function)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.gpus > 1 and "RANK" not in os.environ and args.impl != "reference":
        sys.exit(spawn_ranks(args))  # no launcher: this process only starts the ranks
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus))) if "RANK" in os.environ else 1
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and "RANK" in os.environ:
        print(f"warning: WORLD_SIZE={world} != --gpus {args.gpus}", file=sys.stderr)
    if args.workload is None:
        args.workload = "k500" if world == 1 or args.impl == "reference" else "ens100"
    if args.selftest_cpu:
        line = run_selftest_cpu(args, rank, world)
    elif args.impl == "reference":
        line = run_reference(args, rank, max(world, args.gpus))
    else:
        line = run_b200(args, rank, world, local_rank)
    if line is not None and rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
