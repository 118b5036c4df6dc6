#!/usr/bin/env python
"""Sweep the fused J+H kernel over models and register budgets (min_blocks);
one JSON line per point. usage: sweep_eval.py [model:N ...] [--minb 1,2,4]"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_03932_b200 import MODELS, EvalContext, Model  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cases", nargs="*", default=["goddard:100000", "quadrotor:1000000", "quadrotor:100000",
                                             "hang_glider:100000", "shuttle:100000"])
ap.add_argument("--minb", default="0")
ap.add_argument("--split", default="-1")
ap.add_argument("--block", type=int, default=128)
ap.add_argument("--staging", default="-1", help="input_staging values, comma separated")
ap.add_argument("--steps", type=int, default=30)
a = ap.parse_args()
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream()
flush = torch.ones(bench.L2_FLUSH_BYTES // 8, dtype=torch.float64, device=dev)
sink = torch.zeros((), dtype=torch.float64, device=dev)
peak, _ = bench.peaks()
for case in a.cases:
    name, N = case.split(":")
    N = int(N)
    m = Model(MODELS[name], N)
    st = m.structure()
    x, lam = m.synth_acceptance(20250808)
    xd, ld = torch.as_tensor(x, device=dev), torch.as_tensor(lam, device=dev)
    c = torch.zeros(m.m_con, dtype=torch.float64, device=dev)
    nb = bench.algorithmic_bytes(st, *bench.main_space(st), True)
    for mb, sp, stg in [(int(v), int(w), int(z)) for v in a.minb.split(",") for w in a.split.split(",")
                        for z in a.staging.split(",")]:
        ec = EvalContext(m, block=a.block, min_blocks=mb, split_kinds=sp, input_staging=stg)
        ok = ec.eval_jac_hess(xd, ld, c)
        ts, _ = bench.time_eval_config(ec, xd, ld, c, flush, sink, stream, a.steps, 3)
        t = float(np.median(ts))
        # separate c+J and H launches too
        sep = []
        for _ in range(a.steps):
            torch.sum(flush, dim=0, out=sink)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            ec.launch_constraints_jacobian(xd, c, stream)
            ec.launch_hessian(xd, ld, stream)
            e.record(stream)
            e.synchronize()
            sep.append(s.elapsed_time(e) * 1e-3)
        ts2 = float(np.median(sep))
        print(json.dumps({"model": name, "N": N, "minb": mb, "split": sp, "staging": stg, "block": a.block, "ok": ok, "us_fused": t * 1e6, "us_sep": ts2 * 1e6,
                          "ns_per_node": t * 1e9 / N, "frac_fused": nb / t / 1e9 / peak,
                          "frac_sep": nb / ts2 / 1e9 / peak}), flush=True)
        del ec
