#!/usr/bin/env python
"""Goddard solves (BASELINE config 2): the device IPM (ocg_ipm_solve) against
the reference ipm::solve (oracle/_ref/libref.so, Backend::parallel on all
cores), each optionally capped at max_iter. Per-iteration times make the
capped runs comparable. One JSON line per case.

usage: goddard_solve.py N[:max_iter[:ref_max_iter]] ...   (ref_max_iter 0 = skip the reference)
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

model = os.environ.get("MODEL", "goddard")
cores = os.cpu_count() or 1
for case in sys.argv[1:]:
    p = [int(float(v)) for v in case.split(":")]
    N, max_iter = p[0], (p[1] if len(p) > 1 else 0)
    ref_iter = p[2] if len(p) > 2 else max_iter
    row = {"model": model, "N": N, "max_iter": max_iter}
    m = Model(MODELS[model], N)
    t0 = time.perf_counter()
    d = solve(m, **({"max_iter": max_iter} if max_iter else {}))
    d["wall_s"] = time.perf_counter() - t0
    d["s_per_iter"] = d["time_total"] / max(d["iterations"], 1)
    d["other_s"] = d["time_total"] - d["time_derivatives"] - d["time_factorize"] - d["time_solve"]
    row["device"] = d
    print(f"# {model} N={N} device: {d['status_name']} iters {d['iterations']} obj {d['objective']:.10f} "
          f"total {d['time_total']:.2f}s ({1e3 * d['s_per_iter']:.3f} ms/iter; factor {d['time_factorize']:.2f} "
          f"solve {d['time_solve']:.2f} deriv {d['time_derivatives']:.2f} other {d['other_s']:.2f}; "
          f"{d['factorizations']} factorizations) plans {d['time_plan_eval']:.2f}/{d['time_plan_kkt']:.2f}/"
          f"{d['time_plan_ldl']:.2f}", file=sys.stderr, flush=True)
    if ref_iter >= 0 and len(p) > 2 and ref_iter == 0:
        print(json.dumps(row), flush=True)
        continue
    rm = RefModel(MODELS[model], N)
    t0 = time.perf_counter()
    r = rm.solve(parallel=True, workers=cores, max_iter=ref_iter)
    r["wall_s"] = time.perf_counter() - t0
    r["s_per_iter"] = r["wall_s"] / max(r["iterations"], 1)
    r["cores"] = cores
    row["ref"] = r
    print(f"# {model} N={N} ref: status {r['status']:.0f} iters {r['iterations']:.0f} obj {r['objective']:.10f} "
          f"wall {r['wall_s']:.2f}s ({1e3 * r['s_per_iter']:.3f} ms/iter; factor {r['time_factorize']:.2f} "
          f"deriv {r['time_derivatives']:.2f}) {cores} cores", file=sys.stderr, flush=True)
    row["iterations_match"] = d["iterations"] == int(r["iterations"])
    row["objective_rel_diff"] = abs(d["objective"] - r["objective"]) / max(abs(r["objective"]), 1e-300)
    row["speedup_per_iter"] = r["s_per_iter"] / d["s_per_iter"]
    print(json.dumps(row), flush=True)
