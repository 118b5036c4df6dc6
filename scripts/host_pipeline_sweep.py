#!/usr/bin/env python
"""Chunk-count sweep of ocg_eval_jac_hess_host (page-locked host buffers in and
out, pipelined over node-range chunks): median step time over 20 steps after
3 warm-up, CUDA events on the caller's stream; chunks=0 is the unpipelined
sequence (x, lambda up; one fused launch; c, jac, hess down on one stream)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/", 2)[0])
from paper_2510_03932_b200 import MODELS, EvalContext, Model  # noqa: E402

for spec in (sys.argv[1:] or ["goddard:100000", "quadrotor:100000", "quadrotor:1000000"]):
    name, N = spec.split(":")
    m = Model(MODELS[name], int(N))
    x, lam = m.synth_acceptance(20250808)
    ec = EvalContext(m, device=0)
    xh, lh = torch.as_tensor(x).pin_memory(), torch.as_tensor(lam).pin_memory()
    ch = torch.empty(m.m_con, dtype=torch.float64).pin_memory()
    jh = torch.empty(ec.jac_nnz, dtype=torch.float64).pin_memory()
    hh = torch.empty(ec.hess_nnz, dtype=torch.float64).pin_memory()
    xd, ld = torch.empty_like(xh, device="cuda"), torch.empty_like(lh, device="cuda")
    cd = torch.empty(m.m_con, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    nbytes = 8 * (m.nvar + 2 * m.m_con + ec.jac_nnz + ec.hess_nnz)
    for chunks in (0, 1, 2, 4, 8, 16, 32):
        def step():
            if chunks == 0:
                xd.copy_(xh, non_blocking=True)
                ld.copy_(lh, non_blocking=True)
                ec.launch_jac_hess(xd, ld, cd, s)
                ch.copy_(cd, non_blocking=True)
                jh.copy_(ec.jac_val, non_blocking=True)
                hh.copy_(ec.hess_val, non_blocking=True)
            else:
                ec.launch_jac_hess_host(xh, lh, ch, jh, hh, chunks=chunks, stream=s)
        for _ in range(3):
            step()
        s.synchronize()
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            step()
            b.record(s)
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        t = float(np.median(ts))
        print(json.dumps({"model": name, "N": int(N), "chunks": chunks, "median_ms": t * 1e3,
                          "ns_per_node": t * 1e9 / int(N), "gbs_pcie": nbytes / t / 1e9}), flush=True)
