"""Scratch timing of the J+H step (CUDA events), variants."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2510_03932_b200 import MODELS, EvalContext, Model
BW = 6534.5e9
cases = [("goddard", 100_000), ("quadrotor", 1_000_000), ("shuttle", 100_000), ("hang_glider", 100_000)]
if len(sys.argv) > 1: cases = [(a.split(":")[0], int(a.split(":")[1])) for a in sys.argv[1:]]
for name, N in cases:
    m = Model(MODELS[name], N)
    x, lam = m.synth_acceptance(20250808)
    for split in (True,):
      for block in (64, 128, 256):
        ec = EvalContext(m, block=block)
        xd = torch.tensor(x, device="cuda"); ld = torch.tensor(lam, device="cuda")
        c = torch.empty(m.m_con, dtype=torch.float64, device="cuda")
        flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")
        assert ec.eval_constraints_jacobian(xd, c) and ec.eval_hessian(xd, ld)
        res = {}
        for mode in ("sep", "fused", "jac", "hess"):
            ts = []
            for it in range(10):
                flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                if mode == "sep":
                    ec.launch_constraints_jacobian(xd, c); ec.launch_hessian(xd, ld)
                elif mode == "fused":
                    ec.launch_jac_hess(xd, ld, c)
                elif mode == "jac":
                    ec.launch_constraints_jacobian(xd, c)
                else:
                    ec.launch_hessian(xd, ld)
                e.record(); e.synchronize()
                ts.append(s.elapsed_time(e) * 1e-3)
            res[mode] = float(np.median(ts[2:]))
        nb = 8 * (ec.jac_nnz + ec.hess_nnz + 2 * m.m_con + m.nvar + m.m_con)
        print(f"{name:12s} N={N:8d} split={int(split)} B={block:3d} sep {res['sep']*1e6:8.1f}us fused {res['fused']*1e6:8.1f}us jac {res['jac']*1e6:7.1f} hess {res['hess']*1e6:7.1f} "
              f"ns/node fused {res['fused']/N*1e9:.3f} frac(fused) {nb/res['fused']/BW:.3f} frac(sep) {nb/res['sep']/BW:.3f}", flush=True)
        del ec
