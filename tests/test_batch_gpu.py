"""Batched device IPM (ocg_ipm_batch_solve, BASELINE config 5): every instance
of a batch must reach the reference ipm::solve's status, iteration count and
objective (1e-8 relative), and agree with the single-instance device solve of
the same instance — the batch shares launches, not decisions."""
from __future__ import annotations

import numpy as np
import pytest

from _oracle import RefModel
from paper_2510_03932_b200 import MODELS, Model, solve, solve_batch
from paper_2510_03932_b200.models import cart_pendulum_instance

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N", [60, 200])
def test_cart_pendulum_batch_matches_reference(N):
    bs = [0, 1, 517, 2048, 4095]
    insts = [Model(cart_pendulum_instance(b, 4096), N) for b in bs]
    got = solve_batch(insts[0], insts, return_x=True)
    assert len(got) == len(bs)
    for b, inst, g in zip(bs, insts, got):
        ref = RefModel(cart_pendulum_instance(b, 4096), N).solve(parallel=False)
        one = solve(inst)
        print(f"b={b} ref {ref['iterations']} {ref['objective']:.12g} batch {g['iterations']} {g['objective']:.12g} "
              f"single {one['iterations']} factorizations {g['factorizations']}/{one['factorizations']}")
        assert g["status"] == ref["status"] == one["status"] == 0
        assert g["iterations"] == ref["iterations"] == one["iterations"]
        assert abs(g["objective"] - ref["objective"]) <= 1e-8 * abs(ref["objective"])
        assert abs(g["objective"] - one["objective"]) <= 1e-9 * abs(one["objective"])
        assert np.all(np.isfinite(g["x"]))
    print("rounds", got[0]["rounds"], "launch groups", got[0]["launch_groups"])


@pytest.mark.parametrize("name,N", [("double_integrator", 1000), ("quadrotor", 300), ("goddard", 200)])
def test_batch_of_copies_matches_single_solve(name, N):
    """n copies of one model: identical instances must finish identically
    (determinism across launch positions) and like the single solve."""
    m = Model(MODELS[name], N)
    got = solve_batch(m, n=3, max_iter=3000)
    one = solve(m, max_iter=3000)
    for g in got:
        assert g["status"] == one["status"]
        assert g["iterations"] == got[0]["iterations"]
        assert g["objective"] == got[0]["objective"]
    if name != "goddard":  # Goddard's trajectory is rounding-sensitive (test_ipm_gpu.py)
        assert got[0]["iterations"] == one["iterations"]
    assert abs(got[0]["objective"] - one["objective"]) <= 1e-6 * abs(one["objective"])
