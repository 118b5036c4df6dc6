#!/usr/bin/env python
"""A/B of the J+H step: the fused ocg_cjh launch vs ocg_cjac and ocg_hess
launched concurrently on two streams (fork/join with events), and vs the two
back to back; CUDA events, L2 flushed (512 MiB read) before each rep, median
of reps. usage: split_ab.py model:N ... -> JSON lines"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2510_03932_b200 import MODELS, EvalContext, Model  # noqa: E402

flush = torch.ones(512 * 2**20 // 8, dtype=torch.float64, device="cuda")
sink = torch.zeros((), dtype=torch.float64, device="cuda")
main = torch.cuda.current_stream()
side = torch.cuda.Stream()


def timed(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.sum(flush, dim=0, out=sink)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        fn()
        b.record(main)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


for spec in sys.argv[1:] or ["goddard:100000", "quadrotor:100000", "hang_glider:100000"]:
    name, N = spec.split(":")
    m = Model(MODELS[name], int(N))
    ec = EvalContext(m)
    x, lam = m.synth_acceptance(20250808)
    xd, ld = torch.as_tensor(x, device="cuda"), torch.as_tensor(lam, device="cuda")
    c = torch.empty(m.m_con, dtype=torch.float64, device="cuda")

    def fused():
        ec.launch_jac_hess(xd, ld, c, main)

    def serial():
        ec.launch_constraints_jacobian(xd, c, main)
        ec.launch_hessian(xd, ld, main)

    def concurrent():
        e0 = torch.cuda.Event()
        e0.record(main)
        side.wait_event(e0)
        ec.launch_constraints_jacobian(xd, c, main)
        ec.launch_hessian(xd, ld, side)
        e1 = torch.cuda.Event()
        e1.record(side)
        main.wait_event(e1)

    row = {"model": name, "N": int(N), "fused_us": timed(fused), "serial_us": timed(serial),
           "concurrent_us": timed(concurrent)}
    print(json.dumps(row), flush=True)
