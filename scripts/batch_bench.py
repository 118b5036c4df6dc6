#!/usr/bin/env python
"""BASELINE config 5: a batch of independent cart-pendulum OCP instances
(N=500, terminal target p(2) = 1 + b/4096), solved as independent device IPM
solves (ocg_ipm_solve) from T host threads, each with its own CUDA stream
(the C ABI releases the GIL), against the reference ipm::solve run one
instance per host core. Multi-GPU: instances shard by contiguous index range
across ranks (replicas only, no collective) — run under torchrun.

usage: batch_bench.py [--instances 256] [--threads 16] [--N 500] [--ref-sample 64]
"""
import argparse
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from paper_2510_03932_b200 import Model, solve  # noqa: E402
from paper_2510_03932_b200.models import cart_pendulum_instance  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--instances", type=int, default=256)
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

from paper_2510_03932_b200 import Solver  # noqa: E402

base = Model(cart_pendulum_instance(lo, a.batch), a.N)
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
ok = sum(1 for _, st, _, _ in results if st == 0)
out = {"config": f"cart-pendulum N={a.N} batch, instances {lo}..{hi - 1} of {a.instances}", "rank": rank,
       "world": world, "instances": hi - lo, "optimal": ok, "wall_s": wall, "instances_per_s": (hi - lo) / wall,
       "threads": a.threads, "mean_iterations": sum(r[2] for r in results) / max(1, len(results))}
if a.ref_sample and rank == 0:
    from _oracle import RefModel
    cores = os.cpu_count() or 1
    sample = list(range(0, a.instances, max(1, a.instances // a.ref_sample)))[: a.ref_sample]

    def ref_one(b):
        rm = RefModel(cart_pendulum_instance(b, a.batch), a.N)
        r = rm.solve(parallel=False)
        return b, int(r["status"]), int(r["iterations"]), r["objective"]

    t0 = time.perf_counter()
    with ThreadPoolExecutor(cores) as ex:  # one solve per core (the C harness releases the GIL)
        refs = list(ex.map(ref_one, sample))
    rwall = time.perf_counter() - t0
    byb = {b: (st, it, obj) for b, st, it, obj in results}
    match = [abs(byb[b][2] - obj) <= 1e-8 * abs(obj) and byb[b][1] == it for b, _, it, obj in refs if b in byb]
    out["reference"] = {"sample": len(sample), "cores": cores, "wall_s": rwall, "instances_per_s": len(sample) / rwall,
                        "optimal": sum(1 for r in refs if r[1] == 0)}
    out["parity"] = {"compared": len(match), "iterations_and_objective_match": sum(match)}
    out["speedup"] = out["instances_per_s"] / out["reference"]["instances_per_s"]
print(json.dumps(out), flush=True)
