#!/usr/bin/env python
"""CPU probe (test infrastructure; reads the reference through oracle/_ref):
why Goddard's IPM trajectory depends on the elimination order. Dumps the
reference's first KKT matrix at Goddard N=1000 (REF_DUMP_KKT), prints its
extreme eigenvalues, then runs a dense right-looking LDL^T with the
reference's zero-pivot rule (|d| <= 1e-14 * max(|a_kk + delta|, largest single
update)) in (a) the device's node-major band order, (b) the reverse node order,
(c) reverse Cuthill-McKee. usage: goddard_pivot_probe.py [N]"""
import os
import sys
import tempfile
import warnings

import numpy as np
import scipy.io as sio
import scipy.sparse as sp
from scipy.sparse.csgraph import reverse_cuthill_mckee

warnings.filterwarnings("ignore")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from _oracle import RefEval, RefKkt, RefModel  # noqa: E402
from paper_2510_03932_b200 import MODELS  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
path = os.path.join(tempfile.mkdtemp(), "kkt.mtx")
os.environ["REF_DUMP_KKT"] = path
RefModel(MODELS["goddard"], N).solve(parallel=False, max_iter=1)
del os.environ["REF_DUMP_KKT"]
r = RefModel(MODELS["goddard"], N)
mp = RefKkt(RefEval(r)).maps()
A = sio.mmread(path).tocsc()
A = (sp.tril(A) + sp.tril(A, -1).T).tocsr()
n = A.shape[0]
pi, di = mp["prim_index"], mp["dual_index"]
nt = int((pi >= 0).sum())
ev = np.linalg.eigvalsh(A.toarray())
print(f"dim {n}, ntot {nt}: inertia ({(ev > 0).sum()}, {(ev < 0).sum()}), |ev| min {np.abs(ev).min():.3e} "
      f"max {np.abs(ev).max():.3e} (ratio {np.abs(ev).min() / np.abs(ev).max():.2e})")


def node_order(reverse):
    order = []
    nodes = range(N, -1, -1) if reverse else range(N + 1)
    for t in nodes:
        for slot in (1 + 3 * t, 2 + 3 * t, 3 + 3 * t, 3 * N + 4 + t):
            if pi[slot] >= 0:
                order.append(pi[slot])
        step = t if reverse else t - 1  # rows whose last (first) coupled node is t
        if 0 <= step < N:
            for g in range(3):
                if di[g * N + step] >= 0:
                    order.append(nt + di[g * N + step])
    return np.array(order + [pi[0]])


def ldl(order, dw, dc, label):
    B = A[order][:, order].toarray()
    B[np.arange(n), np.arange(n)] += np.where(order < nt, dw, -dc)
    r_, c_ = np.nonzero(B[: n - 1, : n - 1])
    bw = np.max(np.abs(r_ - c_))
    ps = np.abs(np.diag(B)).copy()
    zero, pos, neg, ratio = [], 0, 0, np.zeros(n)
    for k in range(n):
        d = B[k, k]
        ratio[k] = abs(d) / max(ps[k], 1e-30)
        if not np.isfinite(d) or abs(d) <= 1e-14 * max(ps[k], 1e-30):
            zero.append(k)
            dinv = 0.0
        else:
            dinv = 1.0 / d
            pos, neg = pos + (d > 0), neg + (d < 0)
        idx = list(range(k + 1, min(n - 1, k + bw) + 1)) + ([n - 1] if k + bw < n - 1 else [])
        col = B[idx, k]
        upd = np.outer(col * dinv, col)
        B[np.ix_(idx, idx)] -= upd
        ps[idx] = np.maximum(ps[idx], np.abs(np.diag(upd)))
    print(f"  {label:22s} dw {dw:g} dc {dc:g}: inertia ({pos}, {neg}, {len(zero)}), smallest |d|/scale "
          f"{np.sort(ratio)[len(zero)]:.2e}")


rest = np.arange(1, n)
rcm = np.concatenate([rest[reverse_cuthill_mckee(A[rest][:, rest].tocsr(), symmetric_mode=True)], [0]])
for label, order in (("node-major (device)", node_order(False)), ("reverse node-major", node_order(True)),
                     ("reverse Cuthill-McKee", rcm)):
    ldl(order, 1e-4, 0.0, label)
