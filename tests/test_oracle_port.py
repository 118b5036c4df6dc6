"""Pinning the C restatement (oracle/port) to the reference: on the same
structure dump and inputs it must reproduce the UNMODIFIED reference
(oracle/_ref/libref.so) bit for bit — values, Jacobian, Hessian, objective,
gradient and the ok flag, including domain errors — on every model, both
schemes, the acceptance recipe (acceptance_main.cpp:179-193) and the
quadrotor eval recipe (ipm_test.cpp:394-423)."""
from __future__ import annotations

import numpy as np
import pytest

from _oracle import PortEval, RefEval, RefModel, synth_uniform
from paper_2510_03932_b200 import MODELS


def _check(st, re, x, lam, rs=None, os_=1.0):
    pe = PortEval(st)
    ok_r, c_r, j_r = re.constraints_jacobian(x)
    ok_p, c_p, j_p = pe.constraints_jacobian(x, rs)
    assert ok_p == ok_r
    if ok_r:
        assert np.array_equal(c_p, c_r) and np.array_equal(j_p, j_r)
    ok_r, h_r = re.hessian(x, lam)
    ok_p, h_p = pe.hessian(x, lam, rs, os_)
    assert ok_p == ok_r
    if ok_r:
        assert np.array_equal(h_p, h_r)
    ok_r, f_r = re.objective(x)
    ok_p, f_p = pe.objective(x, os_)
    assert ok_p == ok_r
    if ok_r:
        assert f_p == f_r
    ok_r, g_r, gc_r = re.gradient(x)
    ok_p, g_p, gc_p = pe.gradient(x, os_)
    assert ok_p == ok_r
    if ok_r:
        assert np.array_equal(gc_p, gc_r) and np.array_equal(g_p, g_r)


@pytest.mark.parametrize("name", sorted(MODELS))
@pytest.mark.parametrize("scheme", [0, 1])
@pytest.mark.parametrize("N", [2, 25, 300])
def test_port_bit_exact_vs_reference(name, scheme, N):
    rm = RefModel(MODELS[name], N, scheme)
    x, lam = rm.synth_acceptance(20250808)
    _check(rm.structure(), RefEval(rm), x, lam)


def test_port_quadrotor_eval_recipe():
    rm = RefModel(MODELS["quadrotor"], 1000)
    x = synth_uniform(11, -0.5, 0.5, rm.nvar)
    _check(rm.structure(), RefEval(rm), x, np.full(rm.m_con, 0.25))


@pytest.mark.parametrize("name", ["goddard", "quadrotor", "hang_glider"])
def test_port_scaled_evaluation(name):
    rm = RefModel(MODELS[name], 60)
    re = RefEval(rm)
    os_, rs = re.compute_scaling(rm.arrays()["x_start"], True)
    x, lam = rm.synth_acceptance(5)
    _check(rm.structure(), re, x, lam, rs, os_)


def test_port_domain_error_matches_reference():
    rm = RefModel(MODELS["goddard"], 50)
    x, lam = rm.synth_acceptance(3)
    x = x.copy()
    x[1 + 3 * 10 + 2] = 0.0  # mass 0 at node 10: division by zero
    _check(rm.structure(), RefEval(rm), x, lam)
