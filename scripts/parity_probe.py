#!/usr/bin/env python
"""GPU probe (test infrastructure): per-entry relative error of the fused
J+H evaluation at the benchmarked configurations, launched exactly as
bench.py launches it (block 128, default options, persistent multi-tile
grid), against the reference EvalContext (oracle/_ref/libref.so) on the
acceptance recipe. Reports the worst entries with NO floor, so the entries
that need a cancellation floor can be identified.
usage: parity_probe.py [model:N ...]  -> JSON lines on stdout"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.join(os.path.dirname(__file__), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from _oracle import RefEval, RefModel  # noqa: E402
from paper_2510_03932_b200 import MODELS, EvalContext, Model  # noqa: E402

specs = sys.argv[1:] or ["goddard:100000", "hang_glider:100000", "shuttle:100000", "quadrotor:100000",
                         "quadrotor:1000000", "cart_pendulum:100000"]


def worst(got, ref, k=6):
    scale = np.max(np.abs(ref)) if ref.size else 1.0
    den = np.where(ref == 0, 1.0, np.abs(ref))
    err = np.abs(got - ref) / den
    idx = np.argsort(err)[::-1][:k]
    # smallest floor f with |got - ref| <= 1e-12 * max(|ref|, f * max|ref|) everywhere
    bad = np.abs(got - ref) > 1e-12 * np.abs(ref)
    need = float(np.max(np.abs(got - ref)[bad]) / (1e-12 * scale)) if bad.any() and scale > 0 else 0.0
    return {"max_rel_nofloor": float(err.max()) if err.size else 0.0, "floor_needed": need,
            "n_over_1e-12": int((err > 1e-12).sum()), "n": int(ref.size), "bit_exact_frac": float(np.mean(got == ref)),
            "worst": [{"i": int(i), "ref": float(ref[i]), "got": float(got[i]), "rel": float(err[i]),
                       "ref_over_max": float(abs(ref[i]) / scale)} for i in idx]}


for spec in specs:
    name, N = spec.split(":")
    N = int(N)
    src = MODELS[name]
    m, r = Model(src, N), RefModel(src, N)
    x, lam = r.synth_acceptance(20250808)
    ec, re = EvalContext(m, device=0, block=128), RefEval(r, parallel=True, workers=os.cpu_count() or 1)
    dev = ec.device
    c = torch.zeros(m.m_con, dtype=torch.float64, device=dev)
    ok = ec.eval_jac_hess(x, lam, c)
    ok1, c_r, j_r = re.constraints_jacobian(x)
    ok2, h_r = re.hessian(x, lam)
    out = {"model": name, "N": N, "ok": [ok, ok1, ok2]}
    out["c"] = worst(c.cpu().numpy(), c_r)
    out["jac"] = worst(ec.jac_val.cpu().numpy(), j_r)
    hg = ec.hess_val.cpu().numpy()
    out["hess"] = worst(hg, h_r)
    # which pattern entry / group the worst hess entries belong to
    st = m.structure()
    offs = []
    o = 0
    for g in st["con_groups"] + st["obj_groups"]:
        lo, hi, ends = g["range"]
        cnt = 2 if ends else hi - lo
        offs.append((o, len(g["hess"]), g.get("name", "")))
        o += cnt * len(g["hess"])
    for w in out["hess"]["worst"]:
        for gi, (o0, nh, nm) in enumerate(offs):
            if nh and o0 <= w["i"] < o0 + nh * 10**9 and (gi + 1 == len(offs) or w["i"] < offs[gi + 1][0]):
                w["group"] = gi
                w["entry"] = (w["i"] - o0) % nh
                break
    print(json.dumps(out), flush=True)
    del ec, re
