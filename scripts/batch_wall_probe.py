#!/usr/bin/env python
"""Where the batch solve's wall goes beyond its device-side total: five
whole-batch solves of 4096 cart-pendulum instances (N=500), wall vs the
solver's own time_total, plus the Python-side conversion."""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/", 2)[0])
from paper_2510_03932_b200 import Model, solve_batch  # noqa: E402
from paper_2510_03932_b200.models import cart_pendulum_instance  # noqa: E402

B, N = 4096, 500
base = Model(cart_pendulum_instance(0, 4096), N)
insts = [Model(cart_pendulum_instance(b, 4096), N) for b in range(B)]
arrs = [m.arrays() for m in insts]
lcon = np.ascontiguousarray(np.stack([r["lcon"] for r in arrs]))
ucon = np.ascontiguousarray(np.stack([r["ucon"] for r in arrs]))
solve_batch(base, insts[:2])
import paper_2510_03932_b200.evaluation as ev  # noqa: E402
_orig = ev.LIB.ocg_ipm_batch_solve
_c = {}


def _timed(*a):
    t = time.perf_counter()
    r = _orig(*a)
    _c["c_abi"] = time.perf_counter() - t
    return r


ev.LIB.ocg_ipm_batch_solve = _timed
for i in range(5):
    t0 = time.perf_counter()
    res = solve_batch(base, lcon=lcon, ucon=ucon)
    w = time.perf_counter() - t0
    print(f"  c_abi call {_c.get('c_abi', float('nan')):.3f} s of wall {w:.3f} s", flush=True)
    print(f"solve {i}: wall {w:.3f} s, time_total {res[0]['time_total']:.3f} s, setup {res[0]['time_setup']:.3f} s, "
          f"plan {res[0]['time_plan_eval'] + res[0]['time_plan_kkt'] + res[0]['time_plan_ldl']:.3f} s", flush=True)
