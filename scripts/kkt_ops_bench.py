#!/usr/bin/env python
"""Per-call device times of the KKT operations the IPM issues every iteration
(CUDA events on the launching stream, median of reps): assembly, J^T lambda,
matvec, norm, band LDL^T factor and solve. usage: kkt_ops_bench.py model:N ..."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from _oracle import RefModel  # noqa: E402
from paper_2510_03932_b200 import MODELS, BandLdl, EvalContext, KktAssembler, Model  # noqa: E402
from paper_2510_03932_b200.evaluation import LIB, _ptr, _stream  # noqa: E402


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for case in sys.argv[1:]:
    name, N = case.split(":")
    N = int(N)
    m, r = Model(MODELS[name], N), RefModel(MODELS[name], N)
    ec = EvalContext(m)
    x, lam = r.synth_acceptance(20250808)
    c = torch.empty(m.m_con, dtype=torch.float64, device=ec.device)
    assert ec.eval_constraints_jacobian(x, c) and ec.eval_hessian(x, lam)
    k = KktAssembler(m, ec)
    sigma = torch.tensor(np.random.default_rng(5).uniform(0.5, 2.0, k.ntot), device=ec.device)
    xv = torch.tensor(np.random.default_rng(6).standard_normal(k.dim), device=ec.device)
    yv = torch.empty_like(xv)
    lv = torch.tensor(np.random.default_rng(7).standard_normal(m.m_con), device=ec.device)
    jv = torch.empty(k.ntot, dtype=torch.float64, device=ec.device)
    sc = torch.empty(1, dtype=torch.float64, device=ec.device)
    row = {"model": name, "N": N, "dim": k.dim, "nnz": k.nnz}
    row["assemble_ms"] = timed(lambda: LIB.ocg_kkt_assemble(k._h, _ptr(sigma), _stream()))
    row["jt_lambda_ms"] = timed(lambda: LIB.ocg_kkt_jt_lambda(k._h, _ptr(lv), _ptr(jv), _stream()))
    row["matvec_ms"] = timed(lambda: LIB.ocg_kkt_matvec(k._h, _ptr(xv), _ptr(yv), _stream()))
    row["norm_inf_ms"] = timed(lambda: LIB.ocg_kkt_norm_inf(k._h, _ptr(sc), _stream()))
    ldl = BandLdl(k)
    row["ldl"] = ldl.info()
    row["factor_ms"] = timed(lambda: ldl.factor(1.0, 1e-8), reps=10)
    row["solve_ms"] = timed(lambda: ldl.solve(xv), reps=10)
    print(json.dumps(row), flush=True)
