#!/usr/bin/env python3
"""BASELINE configs[4] end to end on one GPU: M = 4096 seeded members at one
(K, N), 5000 steps (t = 50), each member's base run and its own (K+50, N+30)
verify run, agreement digits every 100 steps, divergence time t_c at d digits,
through the public entry point ensemble.tc_sweep. Writes one JSON summary.

    python tools/tc_sweep_full.py K N [n_steps] [M] [d] > out.json
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1908_09301_b200 import ensemble as E

K, N = int(sys.argv[1]), int(sys.argv[2])
n_steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5000
M = int(sys.argv[4]) if len(sys.argv) > 4 else 4096
d = int(sys.argv[5]) if len(sys.argv) > 5 else 10
t0 = time.perf_counter()
rep = E.tc_sweep(K, N, M, n_steps, d=d, stride=100)
wall = time.perf_counter() - t0
tc = np.array([float(t) for t in rep.t_c()])
last = rep.agreement[:, -1]
out = {
    "workload": f"configs[4]: M={M} members at (K,N)=({K},{N}), verify ({K + 50},{N + 30}), {n_steps} steps, stride 100, d={d}",
    "wall_seconds": wall, "kernel_ms": rep.kernel_ms,
    "taylor_steps_per_s_wall": 2 * M * n_steps / wall,
    "taylor_steps_per_s_device": 2 * M * n_steps / ((rep.kernel_ms["base"] + rep.kernel_ms["verify"]) * 1e-3),
    "t_c": {"min": float(tc.min()), "max": float(tc.max()), "mean": float(tc.mean()),
            "histogram": {str(v): int(c) for v, c in zip(*np.unique(tc, return_counts=True))}},
    "agreement_digits_at_t_end": {"min": int(last.min()), "max": int(last.max()), "median": float(np.median(last))},
    "agreement_digits_at_t0": {"min": int(rep.agreement[:, 0].min()), "max": int(rep.agreement[:, 0].max())},
    "final_x_range": [float(rep.final_xyz[:, 0].min()), float(rep.final_xyz[:, 0].max())],
    "members_with_distinct_final_state": int(len({tuple(r) for r in rep.final_digits.reshape(M, -1).tolist()})),
}
print(json.dumps(out, indent=1))
