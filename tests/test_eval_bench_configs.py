"""GPU parity at the BENCHMARKED configurations, launched exactly as bench.py
launches them (block 32 and 128, default options: the persistent grid where blocks
loop over several tiles, shared-memory staging reused across tiles behind the
bulk-copy read waits, alignment shifts of the bulk copy-out), against the
reference EvalContext (oracle/_ref/libref.so, Backend::parallel) on:
  - the acceptance recipe (acceptance_main.cpp:179-193, mt19937(20250808));
  - the quadrotor eval recipe (ipm_test.cpp:394-423: x ~ U(-0.5, 0.5) with
    mt19937(11), lambda = 0.25).
Tolerance: tests/parity.py with the model's floor (none for Goddard and the
hang glider). Both the fused ocg_cjh launch (bench.py's step) and the separate
ocg_cjac / ocg_hess / ocg_c launches are checked.
"""
from __future__ import annotations

import os

import numpy as np
import pytest
import torch

from _oracle import RefEval, RefModel, synth_uniform
from parity import assert_close
from paper_2510_03932_b200 import MODELS, EvalContext, Model

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CONFIGS = [("goddard", 100_000), ("hang_glider", 100_000), ("shuttle", 100_000), ("quadrotor", 100_000),
           ("quadrotor", 1_000_000), ("goddard", 1_000_000)]


def _check_all(name, m, ec, re, x, lam):
    dev = ec.device
    c = torch.full((m.m_con,), float("nan"), dtype=torch.float64, device=dev)
    ec.jac_val.fill_(float("nan"))
    ec.hess_val.fill_(float("nan"))
    assert ec.eval_jac_hess(x, lam, c)  # bench.py's step (ocg_cjh)
    ok1, c_r, j_r = re.constraints_jacobian(x)
    ok2, h_r = re.hessian(x, lam)
    assert ok1 and ok2
    out = {"c": assert_close(c.cpu().numpy(), c_r, f"{name} c (fused)", model=name),
           "jac": assert_close(ec.jac_val.cpu().numpy(), j_r, f"{name} jac (fused)", model=name),
           "hess": assert_close(ec.hess_val.cpu().numpy(), h_r, f"{name} hess (fused)", model=name)}
    # separate launches write the same slots
    c.fill_(float("nan"))
    ec.jac_val.fill_(float("nan"))
    ec.hess_val.fill_(float("nan"))
    assert ec.eval_constraints_jacobian(x, c)
    assert ec.eval_hessian(x, lam)
    assert_close(c.cpu().numpy(), c_r, f"{name} c (cjac)", model=name)
    assert_close(ec.jac_val.cpu().numpy(), j_r, f"{name} jac (cjac)", model=name)
    assert_close(ec.hess_val.cpu().numpy(), h_r, f"{name} hess", model=name)
    c.fill_(float("nan"))
    assert ec.eval_constraints(x, c)
    assert_close(c.cpu().numpy(), c_r, f"{name} c (c only)", model=name)
    return out


# 32: one-warp blocks, TMA bulk copy-in double-buffered on mbarriers (the
# default); 128: four warps per block with LDGSTS staging
BLOCKS = [32, 128]


@pytest.mark.parametrize("block", BLOCKS)
@pytest.mark.parametrize("name,N", CONFIGS)
def test_bench_config_acceptance_recipe(name, N, block):
    src = MODELS[name]
    m, r = Model(src, N), RefModel(src, N)
    x, lam = r.synth_acceptance(20250808)
    ec = EvalContext(m, device=0, block=block)
    re = RefEval(r, parallel=True, workers=os.cpu_count() or 1)
    st = _check_all(name, m, ec, re, x, lam)
    print(name, N, {k: (v["max_rel"], v["bit_exact"]) for k, v in st.items()})


@pytest.mark.parametrize("block", BLOCKS)
@pytest.mark.parametrize("N", [100_000, 1_000_000])
def test_bench_config_quadrotor_recipe(N, block):
    src = MODELS["quadrotor"]
    m, r = Model(src, N), RefModel(src, N)
    x = synth_uniform(11, -0.5, 0.5, m.nvar)
    lam = np.full(m.m_con, 0.25)
    ec = EvalContext(m, device=0, block=block)
    re = RefEval(r, parallel=True, workers=os.cpu_count() or 1)
    _check_all("quadrotor", m, ec, re, x, lam)


@pytest.mark.parametrize("block", BLOCKS)
@pytest.mark.parametrize("name,N", [("goddard", 100_000), ("quadrotor", 100_000)])
def test_bench_config_objective_gradient(name, N, block):
    """f (reference 512-chunk order) and the dense gradient at bench sizes."""
    src = MODELS[name]
    m, r = Model(src, N), RefModel(src, N)
    x, _ = r.synth_acceptance(20250808)
    ec = EvalContext(m, device=0, block=block)
    re = RefEval(r, parallel=True, workers=os.cpu_count() or 1)
    ok_r, f_r = re.objective(x)
    ok, f = ec.eval_objective(x)
    assert ok and ok_r
    assert_close(np.array([f]), np.array([f_r]), f"{name} f", model=name)
    ok_r, g_r, gc_r = re.gradient(x)
    g = torch.empty(m.nvar, dtype=torch.float64, device=ec.device)
    assert ec.eval_gradient(x, g) and ok_r
    assert_close(ec.grad_val.cpu().numpy(), gc_r, f"{name} grad coo", model=name)
    assert_close(g.cpu().numpy(), g_r, f"{name} grad dense", model=name)
