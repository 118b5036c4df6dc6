#!/usr/bin/env python
"""Per-call device time of the reference-order LDL^T (OCG_LDL_REFERENCE) and
the band LDL^T on the same assembled KKT matrix (acceptance-recipe x and
lambda, sigma ~ U(0.5, 2)), CUDA events on the launching stream, median of
reps. usage: refldl_bench.py model:N [...] -> JSON lines"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.join(os.path.dirname(__file__), "..")
sys.path.insert(0, ROOT)
from paper_2510_03932_b200 import MODELS, BandLdl, EvalContext, KktAssembler, Model  # noqa: E402


def timed(fn, reps=7):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for spec in sys.argv[1:] or ["goddard:1000", "goddard:5000", "goddard:100000", "double_integrator:20000"]:
    name, N = spec.split(":")
    N = int(N)
    m = Model(MODELS[name], N)
    ec = EvalContext(m)
    x, lam = m.synth_acceptance(20250808)
    c = torch.empty(m.m_con, dtype=torch.float64, device=ec.device)
    ec.eval_constraints_jacobian(x, c)
    ec.eval_hessian(x, lam)
    k = KktAssembler(m, ec)
    k.assemble(np.random.default_rng(5).uniform(0.5, 2.0, k.ntot))
    b = torch.randn(k.dim, dtype=torch.float64, device=ec.device)
    out = {"model": name, "N": N, "dim": k.dim}
    for order in ("reference", "band"):
        ldl = BandLdl(k, order=order)
        inertia = ldl.factor(1e-4, 1e-8)
        tf = timed(lambda: ldl.factor(1e-4, 1e-8))
        ts = timed(lambda: ldl.solve(b))
        xs = ldl.solve(b)
        res = (k.matvec(xs) + torch.cat([1e-4 * xs[:k.ntot], -1e-8 * xs[k.ntot:]]) - b).abs().max().item()
        out[order] = {"factor_ms": tf, "solve_ms": ts, "inertia": inertia, "residual": res, **ldl.info()}
    print(json.dumps(out), flush=True)
