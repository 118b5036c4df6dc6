"""KKT assembly, products and the device factorization against the reference
(oracle/_ref/libref.so): KktAssembler pattern/maps bit-identical, assembled
values within 1e-12 relative (same accumulation order, inputs within 1e-12),
matvec_sym, J^T lambda, and the band LDL^T's inertia and solves."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from _oracle import RefEval, RefKkt, RefModel
from parity import FLOOR, assert_close
from paper_2510_03932_b200 import MODELS, BandLdl, EvalContext, KktAssembler, Model

pytestmark = pytest.mark.gpu


def _setup(name, N, seed=20250808):
    m, r = Model(MODELS[name], N), RefModel(MODELS[name], N)
    ec, re = EvalContext(m), RefEval(r)
    x, lam = r.synth_acceptance(seed)
    c = torch.empty(m.m_con, dtype=torch.float64, device=ec.device)
    assert ec.eval_constraints_jacobian(x, c) and ec.eval_hessian(x, lam)
    assert re.constraints_jacobian(x)[0] and re.hessian(x, lam)[0]
    return m, ec, KktAssembler(m, ec), RefKkt(re)


@pytest.mark.parametrize("name,N", [("double_integrator", 150), ("goddard", 150), ("quadrotor", 150),
                                    ("hang_glider", 150), ("shuttle", 150),
                                    # the free final time's rows gather > 1024 terms: one-block long-row kernels
                                    ("goddard", 1500), ("hang_glider", 1500)])
def test_kkt_pattern_and_assembly(name, N):
    m, ec, k, kr = _setup(name, N)
    assert (k.dim, k.nnz, k.n_free, k.n_slack, k.m) == (kr.dim, kr.nnz, kr.n_free, kr.n_slack, kr.m)
    pa, pr = k.pattern(), kr.pattern()
    assert np.array_equal(pa[0], pr[0]) and np.array_equal(pa[1], pr[1])
    ma, mr = k.maps(), kr.maps()
    for key in mr:
        assert np.array_equal(ma[key], mr[key]), key
    sigma = np.random.default_rng(3).uniform(0.1, 3.0, k.ntot)
    k.assemble(sigma)
    val = k.values().cpu().numpy()
    assert_close(val, kr.assemble(sigma), "K.val", model=name)
    xv = np.random.default_rng(4).standard_normal(k.dim)
    # matvec_sym (sparse.cpp:51-61) sums a row in column-then-mirror order, the
    # device in increasing column order: summation-order cancellation, floored
    assert_close(k.matvec(xv).cpu().numpy(), kr.matvec(val, xv), "K x", floor=FLOOR)
    # J^T lambda (Solver::compute_jt_lambda, solver.cpp:244-257) against numpy
    st = ec.structure()
    jr, jc, jv = st["jac_row"], st["jac_col"], ec.jac_val.cpu().numpy()
    lam = np.random.default_rng(7).standard_normal(k.m)
    ref = np.zeros(k.ntot)
    use = (ma["prim_index"][jc] >= 0) & (ma["dual_index"][jr] >= 0)
    np.add.at(ref, ma["prim_index"][jc[use]], jv[use] * lam[ma["dual_index"][jr[use]]])
    srow = np.nonzero(ma["slack_index"] >= 0)[0]
    ref[k.n_free + ma["slack_index"][srow]] -= lam[ma["dual_index"][srow]]
    assert_close(k.jt_lambda(lam).cpu().numpy(), ref, "J^T lambda", floor=FLOOR)  # numpy add.at order


def _dense(k, val, dw, dc):
    colp, rowi = k.pattern()
    K = np.zeros((k.dim, k.dim))
    for j in range(k.dim):
        for p in range(colp[j], colp[j + 1]):
            K[rowi[p], j] = val[p]
            K[j, rowi[p]] = val[p]
    K[np.arange(k.ntot), np.arange(k.ntot)] += dw
    K[np.arange(k.ntot, k.dim), np.arange(k.ntot, k.dim)] -= dc
    return K


@pytest.mark.parametrize("name", ["double_integrator", "goddard", "quadrotor", "cart_pendulum", "shuttle"])
@pytest.mark.parametrize("segments", ["1", "296"])
def test_band_ldl_inertia_and_solve(name, segments, monkeypatch):
    """One banded block, or the time-partitioned factorization (segments +
    separator system): inertia equal to the dense eigenvalue count, solves
    equal to a dense solve."""
    monkeypatch.setenv("OCG_LDL_SEGMENTS", segments)
    m, ec, k, _ = _setup(name, 60)
    sigma = np.random.default_rng(5).uniform(0.5, 2.0, k.ntot)
    k.assemble(sigma)
    val = k.values().cpu().numpy()
    ldl = BandLdl(k)
    info = ldl.info()
    assert info["dim"] == k.dim and info["bandwidth"] <= 60
    if segments == "1":
        assert info["segments"] == 1
    for dw, dc in [(0.0, 0.0), (1e-2, 0.0), (10.0, 1e-8)]:
        K = _dense(k, val, dw, dc)
        ev = np.linalg.eigvalsh(K)
        tol = 1e-9 * np.abs(ev).max()
        expect = (int((ev > tol).sum()), int((ev < -tol).sum()), int((np.abs(ev) <= tol).sum()))
        got = ldl.factor(dw, dc)
        assert sum(got) == k.dim
        if expect[2] == 0 and got[2] == 0:
            assert got == expect, (dw, dc, got, expect)
            b = np.random.default_rng(6).standard_normal(k.dim)
            xs = ldl.solve(b).cpu().numpy()
            ref = np.linalg.solve(K, b)
            assert np.max(np.abs(xs - ref)) <= 1e-8 * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("name,N,segments", [("goddard", 1500, "64"), ("quadrotor", 400, "29"),
                                             ("shuttle", 500, "40"), ("double_integrator", 3000, "100")])
def test_separator_cyclic_reduction(name, N, segments, monkeypatch):
    """Many separators: the separator system by block cyclic reduction
    (sepcr.cu, several levels, a border for the free-horizon models) against
    the dense inertia and solve, and against the separator system factored as
    one band block (OCG_SEP=band)."""
    monkeypatch.setenv("OCG_LDL_SEGMENTS", segments)
    m, ec, k, _ = _setup(name, N)
    sigma = np.random.default_rng(5).uniform(0.5, 2.0, k.ntot)
    k.assemble(sigma)
    val = k.values().cpu().numpy()
    cr = BandLdl(k)
    assert cr.info()["segments"] > 16
    monkeypatch.setenv("OCG_SEP", "band")
    band = BandLdl(k)
    b = np.random.default_rng(6).standard_normal(k.dim)
    for dw, dc in [(0.0, 0.0), (1e-2, 0.0), (10.0, 1e-8)]:
        K = torch.tensor(_dense(k, val, dw, dc), device="cuda")
        ev = torch.linalg.eigvalsh(K).cpu().numpy()
        tol = 1e-9 * np.abs(ev).max()
        expect = (int((ev > tol).sum()), int((ev < -tol).sum()), int((np.abs(ev) <= tol).sum()))
        got, got_band = cr.factor(dw, dc), band.factor(dw, dc)
        assert sum(got) == k.dim
        if expect[2] == 0 and got[2] == 0:
            assert got == expect == got_band, (dw, dc, got, got_band, expect)
            ref = torch.linalg.solve(K, torch.tensor(b, device="cuda")).cpu().numpy()
            xs = cr.solve(b).cpu().numpy()
            assert np.max(np.abs(xs - ref)) <= 1e-8 * max(1.0, np.max(np.abs(ref)))
            assert np.max(np.abs(xs - band.solve(b).cpu().numpy())) <= 1e-8 * max(1.0, np.max(np.abs(ref)))
