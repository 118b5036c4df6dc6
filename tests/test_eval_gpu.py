"""GPU parity of the evaluation layer against the reference EvalContext.

The checker is the UNMODIFIED reference (oracle/_ref/libref.so) driven on the
same model text and the same inputs. Structure must be bit-identical;
values within 1e-12 relative (tests/parity.py); bool results identical.
Inputs: the acceptance recipe (acceptance_main.cpp:179-193, seed 20250808)
and the quadrotor eval recipe (ipm_test.cpp:394-423, seed 11, lambda = 0.25).
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from _oracle import RefEval, RefModel, synth_uniform
from parity import assert_close
from paper_2510_03932_b200 import MODELS, EvalContext, Model

pytestmark = pytest.mark.gpu

CASES = [(name, N) for name in MODELS for N in (2, 25, 1000)]


def _pair(name, N, scheme="trapezoid"):
    src = MODELS[name]
    m = Model(src, N, scheme)
    r = RefModel(src, N, 1 if scheme == "trapezoid" else 0)
    return m, r


@pytest.mark.parametrize("name,N", CASES)
def test_structure_bit_exact(name, N):
    m, r = _pair(name, N)
    ec, re = EvalContext(m), RefEval(r)
    a, b = ec.structure(), re.structure()
    for k in a:
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("name,N", CASES)
def test_values_acceptance_recipe(name, N):
    m, r = _pair(name, N)
    x, lam = r.synth_acceptance(20250808)
    x2, lam2 = m.synth_acceptance(20250808)
    assert np.array_equal(x, x2) and np.array_equal(lam, lam2)
    ec, re = EvalContext(m), RefEval(r)
    dev = ec.device
    c = torch.empty(m.m_con, dtype=torch.float64, device=dev)

    ok_r, c_r = re.constraints(x)
    assert ec.eval_constraints(x, c) == ok_r
    if ok_r:
        assert_close(c.cpu().numpy(), c_r, f"{name} c", model=name)

    ok_r, c_r, j_r = re.constraints_jacobian(x)
    assert ec.eval_constraints_jacobian(x, c) == ok_r
    if ok_r:
        assert_close(c.cpu().numpy(), c_r, f"{name} c(cjac)", model=name)
        assert_close(ec.jac_val.cpu().numpy(), j_r, f"{name} jac", model=name)

    ok_r, f_r = re.objective(x)
    ok, f = ec.eval_objective(x)
    assert ok == ok_r
    if ok_r:
        assert_close(np.array([f]), np.array([f_r]), f"{name} f", model=name)

    ok_r, g_r, gc_r = re.gradient(x)
    g = torch.empty(m.nvar, dtype=torch.float64, device=dev)
    assert ec.eval_gradient(x, g) == ok_r
    if ok_r:
        assert_close(ec.grad_val.cpu().numpy(), gc_r, f"{name} grad coo", model=name)
        assert_close(g.cpu().numpy(), g_r, f"{name} grad dense", model=name)

    ok_r, h_r = re.hessian(x, lam)
    assert ec.eval_hessian(x, lam) == ok_r
    if ok_r:
        assert_close(ec.hess_val.cpu().numpy(), h_r, f"{name} hess", model=name)
        # max|H| is exact over our own values and within tolerance of the
        # reference's (the entries themselves agree to 1e-12, not bitwise)
        mh = ec.max_abs_hessian()
        assert mh == float(np.max(np.abs(ec.hess_val.cpu().numpy()))) if ec.hess_nnz else mh == 0.0
        assert_close(np.array([mh]), np.array([re.max_abs_hessian()]), f"{name} max|H|", model=name)


@pytest.mark.parametrize("N", [1000])
def test_quadrotor_eval_recipe(N):
    """ipm_test.cpp:394-423: x ~ U(-0.5, 0.5) (mt19937(11)), lambda = 0.25."""
    m, r = _pair("quadrotor", N)
    x = synth_uniform(11, -0.5, 0.5, m.nvar)
    lam = np.full(m.m_con, 0.25)
    ec, re = EvalContext(m), RefEval(r)
    c = torch.empty(m.m_con, dtype=torch.float64, device=ec.device)
    ok_r, c_r, j_r = re.constraints_jacobian(x)
    assert ok_r and ec.eval_constraints_jacobian(x, c)
    st_j = assert_close(ec.jac_val.cpu().numpy(), j_r, "jac", model="quadrotor")
    ok_r, h_r = re.hessian(x, lam)
    assert ok_r and ec.eval_hessian(x, lam)
    st_h = assert_close(ec.hess_val.cpu().numpy(), h_r, "hess", model="quadrotor")
    ok_r, f_r = re.objective(x)
    ok, f = ec.eval_objective(x)
    assert ok and ok_r
    assert_close(np.array([f]), np.array([f_r]), "f", model="quadrotor")
    print("quadrotor bit-exact fractions: jac", st_j["bit_exact"], "hess", st_h["bit_exact"])


@pytest.mark.parametrize("name", ["goddard", "quadrotor", "shuttle"])
def test_fused_jac_hess_matches_separate(name):
    m = Model(MODELS[name], 500)
    x, lam = m.synth_acceptance(7)
    ec = EvalContext(m)
    c1 = torch.empty(m.m_con, dtype=torch.float64, device=ec.device)
    c2 = torch.empty_like(c1)
    assert ec.eval_constraints_jacobian(x, c1)
    assert ec.eval_hessian(x, lam)
    j1, h1 = ec.jac_val.clone(), ec.hess_val.clone()
    ec.jac_val.zero_()
    ec.hess_val.zero_()
    assert ec.eval_jac_hess(x, lam, c2)
    assert torch.equal(c1, c2) and torch.equal(j1, ec.jac_val) and torch.equal(h1, ec.hess_val)


@pytest.mark.parametrize("name", ["goddard", "quadrotor", "hang_glider"])
def test_scaling_matches_reference(name):
    m, r = _pair(name, 200)
    x0 = m.arrays()["x_start"]
    ec, re = EvalContext(m), RefEval(r)
    ec.compute_scaling(x0, True)
    os_r, rs_r = re.compute_scaling(x0, True)
    assert ec.obj_scale == os_r
    assert np.array_equal(ec.row_scale.cpu().numpy(), rs_r)
    # scaled evaluation
    x, lam = r.synth_acceptance(5)
    c = torch.empty(m.m_con, dtype=torch.float64, device=ec.device)
    ok_r, c_r, j_r = re.constraints_jacobian(x)
    assert ec.eval_constraints_jacobian(x, c) == ok_r
    assert_close(ec.jac_val.cpu().numpy(), j_r, "scaled jac", model=name)
    ok_r, h_r = re.hessian(x, lam)
    assert ec.eval_hessian(x, lam) == ok_r
    assert_close(ec.hess_val.cpu().numpy(), h_r, "scaled hess", model=name)
    ok_r, f_r = re.objective(x)
    ok, f = ec.eval_objective(x)
    assert ok == ok_r
    assert_close(np.array([f]), np.array([f_r]), "scaled f", model=name)


def test_domain_errors_flagged():
    """Non-finite intermediates make the call return false, like the reference
    (evaluator.cpp:79-84); here m = 0 divides by zero in Goddard's dynamics."""
    m, r = _pair("goddard", 50)
    x, lam = r.synth_acceptance(3)
    x = x.copy()
    x[1 + 3 * 10 + 2] = 0.0  # m at node 10
    ec, re = EvalContext(m), RefEval(r)
    c = torch.empty(m.m_con, dtype=torch.float64, device=ec.device)
    assert re.constraints_jacobian(x)[0] is False
    assert ec.eval_constraints_jacobian(x, c) is False
    assert re.hessian(x, lam)[0] is False
    assert ec.eval_hessian(x, lam) is False
    # the flag clears: a good point evaluates true again
    x2, _ = r.synth_acceptance(3)
    assert ec.eval_constraints_jacobian(x2, c) is True


def test_euler_scheme():
    for name in ("goddard", "quadrotor", "cart_pendulum"):
        m, r = _pair(name, 40, "euler")
        ec, re = EvalContext(m), RefEval(r)
        a, b = ec.structure(), re.structure()
        for k in a:
            assert np.array_equal(a[k], b[k])
        x, lam = r.synth_acceptance(11)
        c = torch.empty(m.m_con, dtype=torch.float64, device=ec.device)
        ok_r, c_r, j_r = re.constraints_jacobian(x)
        assert ec.eval_constraints_jacobian(x, c) == ok_r
        assert_close(ec.jac_val.cpu().numpy(), j_r, f"{name} euler jac", model=name)
        ok_r, h_r = re.hessian(x, lam)
        assert ec.eval_hessian(x, lam) == ok_r
        assert_close(ec.hess_val.cpu().numpy(), h_r, f"{name} euler hess", model=name)


@pytest.mark.parametrize("name", ["goddard", "quadrotor", "shuttle", "cart_pendulum"])
def test_values_against_c_restatement(name):
    """The same parity through the C restatement of the path (oracle/port),
    itself pinned bit-exact to the reference (tests/test_oracle_port.py)."""
    from _oracle import PortEval
    m, r = _pair(name, 500)
    pe = PortEval(r.structure())
    x, lam = r.synth_acceptance(77)
    ec = EvalContext(m)
    c = torch.empty(m.m_con, dtype=torch.float64, device=ec.device)
    assert ec.eval_jac_hess(x, lam, c)
    ok, c_p, j_p = pe.constraints_jacobian(x)
    ok2, h_p = pe.hessian(x, lam)
    assert ok and ok2
    assert_close(c.cpu().numpy(), c_p, f"{name} c", model=name)
    assert_close(ec.jac_val.cpu().numpy(), j_p, f"{name} jac", model=name)
    assert_close(ec.hess_val.cpu().numpy(), h_p, f"{name} hess", model=name)
