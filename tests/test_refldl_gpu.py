"""Reference-order device LDL^T (ocg_ldl_create_ex(OCG_LDL_REFERENCE),
csrc/refldl.cu) against the reference's sparse::factorize / solve
(proj/src/sparse/ldl.cpp:139-247, oracle/_ref/libref.so) on the same K values:
identical elimination order and pattern of L, identical inertia, D and L within
rounding of the reference's (the summation order inside a pivot differs:
multifrontal vs the reference's up-looking rows), and solves within rounding.
Then the device IPM with this factorization against ipm::solve: the
reference's iteration counts exactly, on Goddard too (proj/test_output.txt:29:
Goddard@1000 = 510), objectives within 1e-8 relative (north_star).
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from _oracle import RefEval, RefKkt, RefModel
from paper_2510_03932_b200 import MODELS, BandLdl, EvalContext, KktAssembler, Model, solve

pytestmark = pytest.mark.gpu


def _setup(name, N, seed=20250808):
    m, r = Model(MODELS[name], N), RefModel(MODELS[name], N)
    ec, re = EvalContext(m), RefEval(r)
    x, lam = r.synth_acceptance(seed)
    c = torch.empty(m.m_con, dtype=torch.float64, device=ec.device)
    assert ec.eval_constraints_jacobian(x, c) and ec.eval_hessian(x, lam)
    assert re.constraints_jacobian(x)[0] and re.hessian(x, lam)[0]
    return m, ec, KktAssembler(m, ec), RefKkt(re)


def _rel(got, ref):
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300))


@pytest.mark.parametrize("name,N", [("double_integrator", 200), ("goddard", 1000), ("quadrotor", 60),
                                    ("cart_pendulum", 100), ("hang_glider", 80), ("shuttle", 50)])
@pytest.mark.parametrize("dw,dc", [(0.0, 0.0), (1e-4, 0.0), (1e-4, 1e-8)])
def test_reference_order_factor_and_solve(name, N, dw, dc):
    m, ec, k, kr = _setup(name, N)
    sigma = np.random.default_rng(5).uniform(0.5, 2.0, k.ntot)
    k.assemble(sigma)
    val = k.values().cpu().numpy()
    ldl = BandLdl(k, order="reference")
    inertia = ldl.factor(dw, dc)
    ref = kr.factorize(val, dw, dc)
    got = ldl.factors()
    sym = kr.symbolic()
    assert np.array_equal(got["perm"], sym["perm"])
    assert np.array_equal(got["Lp"], sym["Lp"]) and np.array_equal(got["Li"], ref["Li"])
    assert inertia == ref["inertia"], f"inertia {inertia} vs reference {ref['inertia']}"
    eD, eL = _rel(got["D"], ref["D"]), _rel(got["Lx"], ref["Lx"])
    # per pivot, relative to the pivot itself where it is not a zero pivot
    nz = np.abs(ref["D"]) > 1e-8 * np.max(np.abs(ref["D"]))
    eDp = float(np.max(np.abs(got["D"][nz] - ref["D"][nz]) / np.abs(ref["D"][nz])))
    print(f"{name}@{N} dw={dw} dc={dc}: inertia {inertia}, D max rel {eD:.2e} (per pivot {eDp:.2e}), "
          f"Lx max rel {eL:.2e}, exact D {np.mean(got['D'] == ref['D']):.3f}")
    # rounding of cancelling pivot sums: bounded against the largest entry,
    # not per pivot (a pivot that cancels to 1e-8 of its terms keeps 1e-8
    # relative noise in any summation order)
    assert eD <= 1e-10 and eL <= 1e-10
    if inertia[2] == 0:
        b = np.random.default_rng(9).standard_normal(k.dim)
        x = ldl.solve(b).cpu().numpy()
        xr = kr.factor_solve(val, b, dw, dc)
        ex = _rel(x, xr)
        print(f"   solve max rel {ex:.2e}")
        assert ex <= 1e-8


@pytest.mark.parametrize("name,N,iters", [("double_integrator", 1000, 4), ("quadrotor", 2000, 6),
                                          ("cart_pendulum", 300, None), ("goddard", 300, None)])
def test_reference_order_solve_matches_reference(name, N, iters):
    ref = RefModel(MODELS[name], N).solve(parallel=False, max_iter=3000)
    got = solve(Model(MODELS[name], N), kkt_order="reference", max_iter=3000)
    print(name, N, "ref", ref["iterations"], ref["factorizations"], ref["objective"], "device", got["iterations"],
          got["factorizations"], got["objective"], f"{got['time_total']:.3f}s")
    assert got["status"] == 0 == ref["status"]
    if iters is not None:
        assert ref["iterations"] == iters
    assert got["iterations"] == ref["iterations"]
    assert got["factorizations"] == ref["factorizations"]
    assert abs(got["objective"] - ref["objective"]) <= 1e-8 * abs(ref["objective"])


@pytest.mark.slow
def test_goddard_1000_reference_trajectory():
    """BASELINE configs[0] pin: Goddard@1000 takes 510 iterations in the
    reference (proj/test_output.txt:29) with 3 factorizations each; the device
    IPM with the reference-order factorization takes the same 510 iterations
    and 1530 factorizations, and ends at the same objective within 1e-8."""
    ref = RefModel(MODELS["goddard"], 1000).solve(parallel=True, max_iter=3000)
    got = solve(Model(MODELS["goddard"], 1000), kkt_order="reference", max_iter=3000)
    print("goddard@1000 ref", ref["iterations"], ref["factorizations"], ref["objective"], f"{ref['time_total']:.2f}s",
          "device", got["iterations"], got["factorizations"], got["objective"], f"{got['time_total']:.2f}s")
    assert ref["iterations"] == 510
    assert got["status"] == 0 == ref["status"]
    assert got["iterations"] == 510
    assert got["factorizations"] == ref["factorizations"]
    assert abs(got["objective"] - ref["objective"]) <= 1e-8 * abs(ref["objective"])


@pytest.mark.slow
def test_goddard_2500_reference_trajectory():
    """A longer trajectory: Goddard@2500 (the reference's cross-grid pin
    J(2500) = 1.0125663, proj/test_output.txt:30) — 1737 iterations and 5211
    factorizations in the oracle build, the same on the device
    (profiles/r2_goddard_parity.jsonl; at N=5000 the two end one iteration
    apart, 2716 vs 2717, objective 1.1e-11 relative: DESIGN.md §6)."""
    import os
    ref = RefModel(MODELS["goddard"], 2500).solve(parallel=True, workers=os.cpu_count() or 1, max_iter=30000)
    got = solve(Model(MODELS["goddard"], 2500), kkt_order="reference", max_iter=30000)
    print("goddard@2500 ref", ref["iterations"], ref["factorizations"], ref["objective"], "device", got["iterations"],
          got["factorizations"], got["objective"])
    assert got["status"] == 0 == ref["status"]
    assert got["iterations"] == ref["iterations"]
    assert got["factorizations"] == ref["factorizations"]
    assert abs(got["objective"] - ref["objective"]) <= 1e-8 * abs(ref["objective"])
    assert abs(got["objective"] - 1.0125663) <= 1e-7  # the published J(2500), 8 digits


@pytest.mark.parametrize("name,N", [("goddard", 1000), ("cart_pendulum", 100), ("quadrotor", 60)])
def test_speculative_candidates_equal_sequential_factorizations(name, N):
    """ocg_ldl_factor_many: every candidate's inertia, factors and solve are
    bit-identical to a sequential ocg_ldl_factor with the same deltas (the IPM
    walks the reference's decision tree over them, ipm.cpp solve_kkt)."""
    m, ec, k, kr = _setup(name, N)
    sigma = np.random.default_rng(7).uniform(0.5, 2.0, k.ntot)
    k.assemble(sigma)
    cands = [(0.0, 0.0), (1e-4, 0.0), (1e-4, 1e-8), (8e-4, 0.0)]
    spec = BandLdl(k, order="reference")
    seq = BandLdl(k, order="reference")
    rhs = torch.tensor(np.random.default_rng(8).standard_normal(k.dim), device=ec.device)
    inertias = spec.factor_many(cands)
    for i, (dw, dc) in enumerate(cands):
        assert seq.factor(dw, dc) == inertias[i], f"candidate {i}"
        spec.select(i)
        a, b = spec.factors(), seq.factors()
        assert np.array_equal(a["D"], b["D"]) and np.array_equal(a["Lx"], b["Lx"]), f"candidate {i} factors"
        assert torch.equal(spec.solve(rhs), seq.solve(rhs)), f"candidate {i} solve"
        spec.select(i)  # swap back: candidate 0's set is current again


def _solve_restated(f, b):
    """proj/src/sparse/ldl.cpp:222-247 (sparse::solve) in plain Python floats:
    the permuted right-hand side, L y = P b by columns (skipping y[k] == 0),
    y *= Dinv, L^T x = y with each column's terms subtracted in entry order."""
    perm, Lp, Li, Lx = f["perm"], f["Lp"], f["Li"], f["Lx"]
    dinv = [0.0 if d == 0.0 else 1.0 / d for d in f["D"].tolist()]
    n = len(perm)
    y = [float(b[perm[k]]) for k in range(n)]
    Lpl, Lil, Lxl = Lp.tolist(), Li.tolist(), Lx.tolist()
    for k in range(n):
        yk = y[k]
        if yk == 0.0:
            continue
        for p in range(Lpl[k], Lpl[k + 1]):
            y[Lil[p]] -= Lxl[p] * yk
    for k in range(n):
        y[k] *= dinv[k]
    for k in range(n - 1, -1, -1):
        s = y[k]
        for p in range(Lpl[k], Lpl[k + 1]):
            s -= Lxl[p] * y[Lil[p]]
        y[k] = s
    x = np.empty(n)
    x[perm] = y
    return x


@pytest.mark.parametrize("name,N", [("double_integrator", 300), ("goddard", 400), ("quadrotor", 60),
                                    ("cart_pendulum", 100), ("hang_glider", 80), ("shuttle", 50)])
def test_sequential_solve_bit_exact(name, N, monkeypatch):
    """seq_solve_k (opt-in OCG_REFLDL_SOLVE=1: one block, the permuted right-
    hand side in shared memory) performs ldl.cpp:222-247's roundings in its
    order: given the device's own factors, its solution equals the plain
    restatement bit for bit."""
    monkeypatch.setenv("OCG_REFLDL_SOLVE", "1")
    m, ec, k, kr = _setup(name, N)
    k.assemble(np.random.default_rng(5).uniform(0.5, 2.0, k.ntot))
    ldl = BandLdl(k, order="reference")
    inertia = ldl.factor(1e-4, 1e-8)
    assert inertia[2] == 0
    b = np.random.default_rng(9).standard_normal(k.dim)
    b[::7] = 0.0  # zero right-hand-side rows take the reference's skip
    x = ldl.solve(b).cpu().numpy()
    want = _solve_restated(ldl.factors(), b)
    assert np.array_equal(x, want), f"{name}: max abs diff {np.max(np.abs(x - want)):.3e}"
