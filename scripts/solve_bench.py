#!/usr/bin/env python
"""Full IPM solves: the reference (oracle/_ref/libref.so, CPU evaluation,
Backend::parallel on all cores) against the drop-in build
(integration/_out/libref_accel.so: the same reference Solver and LDL^T with
every evaluation and the KKT assembly on the B200). One JSON line per case.

usage: solve_bench.py [model:N[:max_iter] ...]
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from _oracle import RefModel  # noqa: E402
from paper_2510_03932_b200 import MODELS, Model, solve  # noqa: E402

cases = sys.argv[1:] or ["double_integrator:100000", "quadrotor:2000", "goddard:1000", "quadrotor:100000"]
cores = os.cpu_count() or 1
for case in cases:
    parts = case.split(":")
    name, N = parts[0], int(parts[1])
    max_iter = int(parts[2]) if len(parts) > 2 else 0
    row = {"model": name, "N": N, "cores": cores}
    for lib in ("ref", "accel"):
        t0 = time.perf_counter()
        rm = RefModel(MODELS[name], N, 1, lib=lib)
        t1 = time.perf_counter()
        r = rm.solve(parallel=True, workers=cores, max_iter=max_iter)
        t2 = time.perf_counter()
        r["wall_solve"] = t2 - t1
        r["wall_transcribe"] = t1 - t0
        row[lib] = r
        print(f"# {name} N={N} {lib}: status {r['status']} iters {r['iterations']:.0f} obj {r['objective']:.10f} "
              f"solve {r['wall_solve']:.2f}s (deriv {r['time_derivatives']:.2f}s factor {r['time_factorize']:.2f}s "
              f"solve {r['time_solve']:.2f}s)", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    m = Model(MODELS[name], N)
    t1 = time.perf_counter()
    d = solve(m, **({"max_iter": max_iter} if max_iter else {}))
    d["wall_solve"] = time.perf_counter() - t1
    d["wall_transcribe"] = t1 - t0
    row["device"] = d
    print(f"# {name} N={N} device: status {d['status']} iters {d['iterations']} obj {d['objective']:.10f} "
          f"solve {d['wall_solve']:.2f}s (deriv {d['time_derivatives']:.2f}s factor {d['time_factorize']:.2f}s "
          f"solve {d['time_solve']:.2f}s, {d['factorizations']} factorizations, bandwidth {d['bandwidth']})",
          file=sys.stderr, flush=True)
    row["device_iterations_match"] = d["iterations"] == row["ref"]["iterations"]
    row["device_speedup_solve"] = row["ref"]["wall_solve"] / d["wall_solve"]
    a, b = row["ref"], row["accel"]
    row["iterations_match"] = a["iterations"] == b["iterations"]
    row["objective_rel_diff"] = abs(a["objective"] - b["objective"]) / max(abs(a["objective"]), 1e-300)
    row["speedup_solve"] = a["wall_solve"] / b["wall_solve"] if b["wall_solve"] > 0 else None
    row["speedup_derivatives"] = a["time_derivatives"] / b["time_derivatives"] if b["time_derivatives"] > 0 else None
    print(json.dumps(row), flush=True)
