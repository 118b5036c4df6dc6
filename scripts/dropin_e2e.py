#!/usr/bin/env python
"""Per-call timing of the drop-in's EvalContext J+H step (reference API,
integration/_out/libref_accel.so); set OCTRANS_ACCEL_TIMING=1 for the phase
breakdown on stderr. usage: dropin_e2e.py [model:N]"""
import os
import sys
import time

ROOT = os.path.join(os.path.dirname(__file__), "..")
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)
from _oracle import RefEval, RefModel  # noqa: E402
from paper_2510_03932_b200.models import MODELS  # noqa: E402

name, N = (sys.argv[1] if len(sys.argv) > 1 else "goddard:100000").split(":")
rm = RefModel(MODELS[name], int(N), lib="accel")
x, lam = rm.synth_acceptance(20250808)
re = RefEval(rm)
for _ in range(3):
    re.step_seconds(x, lam, 1)
ts = [re.step_seconds(x, lam, 1)[0] for _ in range(10)]
print(name, N, "J+H step ms", sorted(t * 1e3 for t in ts))
