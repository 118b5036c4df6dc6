#!/usr/bin/env python
"""Goddard solves with the reference-order device factorization against the
reference's ipm::solve (oracle/_ref/libref.so, Backend::parallel on every
host core) at larger N (BASELINE configs[0]/[1]; the reference's published
pins: Goddard@5000 = 2718 iterations with SuiteSparse AMD, 2717 with the
oracle's exact minimum degree, proj/test_output.txt:29 and SURVEY.md D5;
J(2500) = 1.0125663, J(10000) = 1.0125679, test_output.txt:30).
usage: goddard_parity.py N ... -> JSON lines"""
import json
import os
import sys
import time

ROOT = os.path.join(os.path.dirname(__file__), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from _oracle import RefModel  # noqa: E402
from paper_2510_03932_b200 import MODELS, Model, solve  # noqa: E402

for N in [int(a) for a in sys.argv[1:]] or [2500]:
    t0 = time.perf_counter()
    ref = RefModel(MODELS["goddard"], N).solve(parallel=True, workers=os.cpu_count() or 1, max_iter=30000)
    t_ref = time.perf_counter() - t0
    m = Model(MODELS["goddard"], N)
    t0 = time.perf_counter()
    got = solve(m, kkt_order="reference", max_iter=30000)
    t_dev = time.perf_counter() - t0
    row = {"model": "goddard", "N": N,
           "reference": {"iterations": int(ref["iterations"]), "factorizations": int(ref["factorizations"]),
                         "objective": ref["objective"], "status": int(ref["status"]), "wall_s": t_ref,
                         "cores": os.cpu_count()},
           "device_reference_order": {"iterations": got["iterations"], "factorizations": got["factorizations"],
                                      "objective": got["objective"], "status": got["status"], "wall_s": t_dev,
                                      "time_factorize_s": got["time_factorize"], "time_solve_s": got["time_solve"]},
           "iterations_match": int(ref["iterations"]) == got["iterations"],
           "factorizations_match": int(ref["factorizations"]) == got["factorizations"],
           "objective_rel_diff": abs(got["objective"] - ref["objective"]) / abs(ref["objective"])}
    print(json.dumps(row), flush=True)
