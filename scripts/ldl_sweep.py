#!/usr/bin/env python
"""Time the device band LDL^T (factor + solve) of one assembled KKT matrix
for several time-partition counts. usage: ldl_sweep.py model:N [segments,...]"""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_03932_b200 import MODELS, BandLdl, EvalContext, KktAssembler, Model  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "quadrotor:100000"
segs = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "1,37,74,148,296,592").split(",")]
name, N = spec.split(":")
m = Model(MODELS[name], int(N))
x, lam = m.synth_acceptance(20250808)
ec = EvalContext(m)
c = torch.empty(m.m_con, dtype=torch.float64, device=ec.device)
assert ec.eval_jac_hess(x, lam, c)
k = KktAssembler(m, ec)
k.assemble(np.random.default_rng(1).uniform(0.5, 2.0, k.ntot))
b = torch.as_tensor(np.random.default_rng(2).standard_normal(k.dim), device=ec.device)
for P in segs:
    os.environ["OCG_LDL_SEGMENTS"] = str(P)
    ldl = BandLdl(k)
    info = ldl.info()
    ldl.factor(1e-4, 1e-8)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        inertia = ldl.factor(1e-4, 1e-8)
    torch.cuda.synchronize()
    tf = (time.perf_counter() - t0) / 3
    t0 = time.perf_counter()
    for _ in range(3):
        xs = ldl.solve(b)
    torch.cuda.synchronize()
    ts = (time.perf_counter() - t0) / 3
    r = k.matvec(xs) + 1e-4 * torch.cat([xs[: k.ntot], torch.zeros_like(xs[k.ntot:])]) \
        - 1e-8 * torch.cat([torch.zeros_like(xs[: k.ntot]), xs[k.ntot:]]) - b
    print(f"{name} N={N} segments={info['segments']} bandwidth={info['bandwidth']} factor {tf*1e3:.2f} ms "
          f"solve {ts*1e3:.2f} ms inertia {inertia} residual {float(r.abs().max()):.2e}", flush=True)
    del ldl
