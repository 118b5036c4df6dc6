"""The interior-point vector kernels (SURVEY.md §8a row a18,
csrc/ipm_kernels.cu) on RECORDED iterates of device solves
(OCG_IPM_DUMP / OCG_IPM_DUMP_ITERS, DeviceSolver::dump_iterate) against a
numpy restatement of the reference Solver's loops on the same inputs
(proj/src/ipm/solver.cpp, lines cited per check):
  constraint_residual :209-217, theta_of :219-223, barrier_terms :225-242,
  kkt_error :260-287, sigma :367-373, rhs :381-389, fraction to the boundary
  :399-406, dphi :408-415, dual direction and alpha_z :579-596, the trial
  point :434-441 and the multiplier update with the dual safeguard :598-617.
The device kernels contract products into FMAs and sum in trees, the
reference loops left to right: sums within 1e-12 relative of their terms'
scale; elementwise values within 1e-13 relative; max reductions and the
barrier's validity exactly.
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from paper_2510_03932_b200 import MODELS, Model, solve

pytestmark = pytest.mark.gpu

KAPPA_SIGMA = 1e10  # solver.cpp:48


def _load(d, it):
    meta = json.loads(open(os.path.join(d, f"it{it}_meta.json")).read())
    arr = {}
    for f in os.listdir(d):
        if not f.startswith(f"it{it}_") or f.endswith(".json"):
            continue
        name, ext = f[len(f"it{it}_"):].rsplit(".", 1)
        dt = {"f64": np.float64, "i64": np.int64, "i8": np.int8}[ext]
        arr[name] = np.fromfile(os.path.join(d, f), dtype=dt)
    return meta, arr


def _close(got, ref, what, rtol=1e-13, scale=None):
    got, ref = np.asarray(got, dtype=np.float64), np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, f"{what}: shape {got.shape} vs {ref.shape}"
    if ref.size == 0:
        return
    # scale: the magnitude of the terms the value was computed from (scalar or
    # per entry); a value that cancels is compared against it, not against itself
    s = 1e-3 * np.max(np.abs(ref)) if scale is None else np.asarray(scale, dtype=np.float64)
    err = np.abs(got - ref)
    bound = rtol * np.maximum(np.abs(ref), s) + 1e-300
    assert np.all(err <= bound), f"{what}: worst {np.max(err / bound):.2f}x the bound (rtol {rtol})"


@np.errstate(divide="ignore", invalid="ignore")
def _check(meta, A):
    nf, ntot, m = meta["n_free"], meta["ntot"], meta["m"]
    mu, tau = meta["mu"], meta["tau"]
    x, s = A["x"], A["s"]
    v = np.concatenate([x[A["free_slot"]], s])  # v_at (solver.cpp:194-198)
    lb, ub = A["lb"], A["ub"]
    hl, hu = A["has_lb"].astype(bool), A["has_ub"].astype(bool)
    zl, zu, lam = A["zl"], A["zu"], A["lambda"]
    gradv = np.concatenate([A["grad"][A["free_slot"]], np.zeros(ntot - nf)])
    jt = A["jtlam"]
    dl = np.where(hl, v - lb, 1.0)
    du = np.where(hu, ub - v, 1.0)
    # constraint_residual (:209-217)
    rows = A["dual_row"]
    k = A["slack_index"][rows]
    g_ref = A["c"][rows] - np.where(k >= 0, s[np.maximum(k, 0)] if len(s) else 0.0, A["lcon_s"][rows])
    _close(A["g"], g_ref, "constraint residual g", scale=np.abs(A["c"][rows]) + np.abs(g_ref))
    # theta_of (:219-223): a sum
    _close([meta["theta"]], [np.sum(np.abs(g_ref))], "theta", rtol=1e-12, scale=np.sum(np.abs(g_ref)))
    # barrier_terms (:225-242)
    valid = bool(np.all(dl[hl] > 0) and np.all(du[hu] > 0))
    assert meta["barrier_ok"] == valid
    if valid:
        terms = np.concatenate([np.log(dl[hl]), np.log(du[hu])])
        _close([meta["barrier"]], [np.sum(terms)], "barrier", rtol=1e-12, scale=np.sum(np.abs(terms)))
    # kkt_error parts (:260-287): sums of |z|, |lambda|; max |stationarity|, |g|, |complementarity - mu|
    p = meta["kkt_parts"]
    _close([p[0]], [np.sum(np.abs(zl)) + np.sum(np.abs(zu))], "sum |z|", rtol=1e-12)
    _close([p[1]], [np.sum(np.abs(lam))], "sum |lambda|", rtol=1e-12)
    rd = gradv + jt - zl + zu
    _close([p[2]], [np.max(np.abs(rd)) if ntot else 0.0], "max |stationarity|", rtol=1e-13)
    assert p[3] == (np.max(np.abs(A["g"])) if m else 0.0)  # a max of the same values: exact
    comp = np.concatenate([np.abs(dl * zl - mu)[hl], np.abs(du * zu - mu)[hu]])
    _close([p[4]], [np.max(comp) if comp.size else 0.0], "max |complementarity - mu|", rtol=1e-12, scale=mu)
    # sigma (:367-373)
    sig = np.where(hl, zl / dl, 0.0) + np.where(hu, zu / du, 0.0)
    _close(A["sigma"], sig, "sigma", scale=0.0)
    # rhs (:381-389)
    r = gradv + jt - np.where(hl, mu / dl, 0.0) + np.where(hu, mu / du, 0.0)
    rscale = np.abs(gradv) + np.abs(jt) + np.where(hl, np.abs(mu / dl), 0.0) + np.where(hu, np.abs(mu / du), 0.0)
    _close(A["rhs"], np.concatenate([-r, -A["g"]]), "rhs", scale=np.concatenate([rscale, np.abs(A["g"])]))
    # fraction to the boundary (:399-406)
    step = A["step"]
    dv = step[:ntot]
    cand = [1.0]
    cand += list((-tau * dl / dv)[hl & (dv < 0)])
    cand += list((tau * du / dv)[hu & (dv > 0)])
    _close([meta["alpha_max"]], [min(cand)], "alpha_max")
    # dphi (:408-415): a sum
    gphi = gradv - np.where(hl, mu / dl, 0.0) + np.where(hu, mu / du, 0.0)
    _close([meta["dphi"]], [np.sum(gphi * dv)], "dphi", rtol=1e-12, scale=np.sum(np.abs(gphi * dv)))
    # dual direction, alpha_z (:579-596)
    dzl = np.where(hl, mu / dl - zl - zl / dl * dv, 0.0)
    dzu = np.where(hu, mu / du - zu + zu / du * dv, 0.0)
    _close(A["dzl"], dzl, "dzl", rtol=1e-12, scale=np.where(hl, np.abs(mu / dl) + np.abs(zl) + np.abs(zl / dl * dv), 0))
    _close(A["dzu"], dzu, "dzu", rtol=1e-12, scale=np.where(hu, np.abs(mu / du) + np.abs(zu) + np.abs(zu / du * dv), 0))
    cz = [1.0] + list((-tau * zl / dzl)[(dzl < 0) & (zl > 0)]) + list((-tau * zu / dzu)[(dzu < 0) & (zu > 0)])
    _close([meta["alpha_z"]], [min(cz)], "alpha_z", rtol=1e-12)
    # trial point at alpha_max (:434-441) and the accepted multipliers (:598-617)
    a, az = meta["alpha_max"], meta["alpha_z_used"]
    xt = x.copy()
    xt[A["free_slot"]] = x[A["free_slot"]] + a * dv[:nf]
    st = s + a * dv[nf:]
    dx = np.zeros_like(x)
    dx[A["free_slot"]] = a * dv[:nf]
    _close(A["x_trial"], xt, "trial x", scale=np.abs(x) + np.abs(dx))
    _close(A["s_trial"], st, "trial s", scale=np.abs(s) + np.abs(a * dv[nf:]))
    _close(A["lambda_acc"], lam + a * step[ntot:], "lambda update", scale=np.abs(lam) + np.abs(a * step[ntot:]))
    vn = np.concatenate([xt[A["free_slot"]], st])
    dln, dun = np.where(hl, vn - lb, 1.0), np.where(hu, ub - vn, 1.0)
    zl2 = zl + az * dzl
    zu2 = zu + az * dzu
    zl2 = np.where(hl, np.clip(zl2, mu / (KAPPA_SIGMA * dln), KAPPA_SIGMA * mu / dln), zl2)
    zu2 = np.where(hu, np.clip(zu2, mu / (KAPPA_SIGMA * dun), KAPPA_SIGMA * mu / dun), zu2)
    _close(A["zl_acc"], zl2, "zl update + safeguard", rtol=1e-12, scale=np.abs(zl) + np.abs(az * dzl))
    _close(A["zu_acc"], zu2, "zu update + safeguard", rtol=1e-12, scale=np.abs(zu) + np.abs(az * dzu))


@pytest.mark.parametrize("name,N,iters", [("double_integrator", 400, [0, 2]), ("quadrotor", 200, [0, 3]),
                                          ("goddard", 300, [0, 40]), ("cart_pendulum", 100, [0, 6]),
                                          ("hang_glider", 100, [0, 10])])
def test_vector_kernels_on_recorded_iterates(name, N, iters, tmp_path, monkeypatch):
    monkeypatch.setenv("OCG_IPM_DUMP", str(tmp_path))
    monkeypatch.setenv("OCG_IPM_DUMP_ITERS", ",".join(map(str, iters)))
    monkeypatch.setenv("OCG_IPM_PLAN_CACHE", "0")
    r = solve(Model(MODELS[name], N), max_iter=max(iters) + 1)
    assert r["iterations"] >= min(iters)
    seen = 0
    for it in iters:
        if not os.path.exists(tmp_path / f"it{it}_meta.json"):
            continue
        meta, A = _load(str(tmp_path), it)
        _check(meta, A)
        seen += 1
    assert seen >= 1
