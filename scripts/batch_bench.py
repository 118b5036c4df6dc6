#!/usr/bin/env python
"""BASELINE config 5: a batch of independent cart-pendulum OCP instances
(N=500, terminal target p(2) = 1 + b/4096).

--mode batch (default): one ocg_ipm_batch_solve over all instances — every
device step one launch over instance x node. --mode threads: independent
single-instance device solves from T host threads, one stream each. Against
the reference ipm::solve run one instance per host core. Multi-GPU: instances
shard by contiguous index range across ranks (replicas only, no collective) —
run under torchrun.

usage: batch_bench.py [--instances 4096] [--mode batch|threads] [--threads 16] [--N 500] [--ref-sample 64]
"""
import argparse
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from paper_2510_03932_b200 import Model, solve  # noqa: E402
from paper_2510_03932_b200.models import cart_pendulum_instance  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--instances", type=int, default=4096)
ap.add_argument("--mode", choices=["batch", "threads"], default="batch")
ap.add_argument("--batch", type=int, default=4096, help="b/batch in the terminal target")
ap.add_argument("--threads", type=int, default=16)
ap.add_argument("--N", type=int, default=500)
ap.add_argument("--ref-sample", type=int, default=64, help="instances solved by the reference (0 = skip)")
a = ap.parse_args()

rank = int(os.environ.get("RANK", "0"))
world = int(os.environ.get("WORLD_SIZE", "1"))
lo = a.instances * rank // world
hi = a.instances * (rank + 1) // world
dev = int(os.environ.get("LOCAL_RANK", "0"))


import threading  # noqa: E402

from paper_2510_03932_b200 import Solver, solve_batch  # noqa: E402

base = Model(cart_pendulum_instance(lo, a.batch), a.N)

if a.mode == "batch":
    # the instances' data (here: their terminal-target rows) prepared before
    # the timed region, like the reference arm's models below
    t0 = time.perf_counter()
    insts = [Model(cart_pendulum_instance(b, a.batch), a.N) for b in range(lo, hi)]
    arrs = [m.arrays() for m in insts]
    lcon = np.stack([r["lcon"] for r in arrs])
    ucon = np.stack([r["ucon"] for r in arrs])
    t_models = time.perf_counter() - t0
    solve_batch(base, insts[:2])  # warm the kernel cache
    t0 = time.perf_counter()
    res = solve_batch(base, lcon=lcon, ucon=ucon)
    wall = time.perf_counter() - t0
    results = [(b, r["status"], r["iterations"], r["objective"]) for b, r in zip(range(lo, hi), res)]
    extra = {"rounds": res[0]["rounds"], "launch_groups": res[0]["launch_groups"],
             "batch_time_total_s": res[0]["time_total"], "batch_setup_s": res[0]["time_setup"],
             "plan_s": res[0]["time_plan_eval"] + res[0]["time_plan_kkt"] + res[0]["time_plan_ldl"],
             "instance_data_s (untimed)": t_models}
else:
    tls = threading.local()

    def one(b):
        # one reusable solver context per host thread (plans built once), each
        # solve taking the instance's bounds and start point
        if not hasattr(tls, "solver"):
            tls.solver = Solver(base, device=dev)
        r = tls.solver.solve(Model(cart_pendulum_instance(b, a.batch), a.N))
        return b, r["status"], r["iterations"], r["objective"]

    one(lo)  # warm the kernel cache (identical generated source for every instance)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(a.threads) as ex:
        results = list(ex.map(one, range(lo, hi)))
    wall = time.perf_counter() - t0
    extra = {"threads": a.threads}
ok = sum(1 for _, st, _, _ in results if st == 0)
out = {"config": f"cart-pendulum N={a.N} batch, instances {lo}..{hi - 1} of {a.instances}", "rank": rank,
       "world": world, "instances": hi - lo, "optimal": ok, "wall_s": wall, "instances_per_s": (hi - lo) / wall,
       "mode": a.mode, "mean_iterations": sum(r[2] for r in results) / max(1, len(results)), **extra}
if a.ref_sample and rank == 0:
    from _oracle import RefModel
    cores = os.cpu_count() or 1
    sample = list(range(0, a.instances, max(1, a.instances // a.ref_sample)))[: a.ref_sample]

    ref_models = {b: RefModel(cart_pendulum_instance(b, a.batch), a.N) for b in sample}  # untimed, like ours

    def ref_one(b):
        r = ref_models[b].solve(parallel=False)
        return b, int(r["status"]), int(r["iterations"]), r["objective"]

    t0 = time.perf_counter()
    with ThreadPoolExecutor(cores) as ex:  # one solve per core (the C harness releases the GIL)
        refs = list(ex.map(ref_one, sample))
    rwall = time.perf_counter() - t0
    byb = {b: (st, it, obj) for b, st, it, obj in results}
    match = [abs(byb[b][2] - obj) <= 1e-8 * abs(obj) and byb[b][1] == it for b, _, it, obj in refs if b in byb]
    out["reference"] = {"sample": len(sample), "cores": cores, "wall_s": rwall, "instances_per_s": len(sample) / rwall,
                        "optimal": sum(1 for r in refs if r[1] == 0)}
    out["parity"] = {"compared": len(match), "iterations_and_objective_match": sum(match),
                     "mismatches": [{"b": b, "ref": [it, obj], "ours": list(byb[b][1:])}
                                    for (b, _, it, obj), ok_ in zip([r for r in refs if r[0] in byb], match) if not ok_]}
    out["speedup"] = out["instances_per_s"] / out["reference"]["instances_per_s"]
print(json.dumps(out), flush=True)
