#!/usr/bin/env python
"""A/B of the generated kernels' FMA contraction (EvalContext fma=): fused J+H
time at Goddard/quadrotor and the max relative deviation from the no-FMA
(glibc-bit-exact) values. usage: fma_ab.py model:N ..."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2510_03932_b200 import MODELS, EvalContext, Model  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.ones(bench.L2_FLUSH_BYTES // 8, dtype=torch.float64, device=dev)
sink = torch.zeros((), dtype=torch.float64, device=dev)
for case in sys.argv[1:]:
    name, N = case.split(":")
    m = Model(MODELS[name], int(N))
    x, lam = m.synth_acceptance(20250808)
    xd, ld = torch.as_tensor(x, device=dev), torch.as_tensor(lam, device=dev)
    out = {}
    vals = {}
    for fma in (False, True):
        ec = EvalContext(m, fma=fma)
        c = torch.zeros(m.m_con, dtype=torch.float64, device=dev)
        ts = []
        for it in range(25):
            torch.sum(flush, dim=0, out=sink)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ec.launch_jac_hess(xd, ld, c, torch.cuda.current_stream())
            b.record()
            torch.cuda.synchronize()
            if it >= 5:
                ts.append(a.elapsed_time(b) * 1e3)
        out["us_fma" if fma else "us_nofma"] = float(np.median(ts))
        vals[fma] = torch.cat([c, ec.jac_val, ec.hess_val]).cpu().numpy()
    ref = vals[False]
    scale = np.maximum(np.abs(ref), 1e-4 * np.abs(ref).max())
    out["max_rel_dev"] = float(np.max(np.abs(vals[True] - ref) / scale))
    print(json.dumps({"model": name, "N": int(N), **out}), flush=True)
