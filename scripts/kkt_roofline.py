#!/usr/bin/env python
"""Roofline of the per-iteration KKT gathers:
device time (CUDA events, median of reps, L2 flushed before each rep) and
algorithmic bytes of
  kkt_assemble  8 (nnz_H + nnz_J + ntot + nnz_K)   sources read once, K.val written
  jt_lambda     8 (nnz_J + m + ntot)               jac_val, lambda read, out written
  sym_matvec    8 (2 nnz_K + 2 dim)                K.val read for both triangles, x, y
against MEASURED_PEAKS.json hbm_gbs. usage: kkt_roofline.py model:N ... -> JSON lines"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2510_03932_b200 import MODELS, EvalContext, KktAssembler, Model  # noqa: E402
from paper_2510_03932_b200.evaluation import LIB, _ptr, _stream  # noqa: E402

peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6553.9
flush = torch.ones(512 * 2**20 // 8, dtype=torch.float64, device="cuda")
sink = torch.zeros((), dtype=torch.float64, device="cuda")


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.sum(flush, dim=0, out=sink)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts))


for case in sys.argv[1:] or ["goddard:100000", "quadrotor:100000"]:
    name, N = case.split(":")
    N = int(N)
    m = Model(MODELS[name], N)
    ec = EvalContext(m)
    x, lam = m.synth_acceptance(20250808)
    c = torch.empty(m.m_con, dtype=torch.float64, device=ec.device)
    assert ec.eval_constraints_jacobian(x, c) and ec.eval_hessian(x, lam)
    k = KktAssembler(m, ec)
    sigma = torch.tensor(np.random.default_rng(5).uniform(0.5, 2.0, k.ntot), device=ec.device)
    xv = torch.tensor(np.random.default_rng(6).standard_normal(k.dim), device=ec.device)
    yv = torch.empty_like(xv)
    lv = torch.tensor(np.random.default_rng(7).standard_normal(k.m), device=ec.device)
    jv = torch.empty(k.ntot, dtype=torch.float64, device=ec.device)
    ops = {
        "kkt_assemble": (lambda: LIB.ocg_kkt_assemble(k._h, _ptr(sigma), _stream()),
                         8 * (ec.hess_nnz + ec.jac_nnz + k.ntot + k.nnz)),
        "jt_lambda": (lambda: LIB.ocg_kkt_jt_lambda(k._h, _ptr(lv), _ptr(jv), _stream()),
                      8 * (ec.jac_nnz + k.m + k.ntot)),
        "sym_matvec": (lambda: LIB.ocg_kkt_matvec(k._h, _ptr(xv), _ptr(yv), _stream()),
                       8 * (2 * k.nnz + 2 * k.dim)),
    }
    row = {"model": name, "N": N, "dim": k.dim, "nnz_K": k.nnz, "peak_gbs": peak}
    for op, (fn, nbytes) in ops.items():
        t = timed(fn)
        row[op] = {"us": t * 1e6, "algorithmic_bytes": nbytes, "gbs": nbytes / t / 1e9, "frac": nbytes / t / 1e9 / peak}
    print(json.dumps(row), flush=True)
