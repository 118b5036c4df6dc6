"""CPU proof of the code generator: the generated sm_100a kernel source,
compiled for the host (glibc libm, no FMA contraction) and run with real
32-lane warp barriers, reproduces the UNMODIFIED reference EvalContext bit for
bit — constraint values, Jacobian, Hessian, objective instance values and
gradient entries — and returns the same ok flag on adversarial points.
On the device the only remaining difference is libdevice vs glibc
transcendentals (tests/test_eval_gpu.py)."""
from __future__ import annotations

import numpy as np
import pytest

from _oracle import RefEval, RefModel
from hostexec import run_all
from paper_2510_03932_b200 import MODELS, Model


def _ref_all(r, x, lam):
    re = RefEval(r)
    out = {}
    out["c_ok"], out["c"] = re.constraints(x)
    out["cjac_ok"], out["c_cjac"], out["jac"] = re.constraints_jacobian(x)
    out["hess_ok"], out["hess"] = re.hessian(x, lam)
    out["grad_ok"], _, out["grad"] = re.gradient(x)
    return out


# input staging modes (ocg_eval_options.input_staging): 1 is the device
# default; N = 100 walks four tiles, so the double buffers alternate
STAGINGS = [(1, 2), (1, 25), (1, 100), (0, 100), (2, 25), (2, 100)]


@pytest.mark.parametrize("name", list(MODELS))
@pytest.mark.parametrize("staging,N", STAGINGS)
@pytest.mark.parametrize("scheme", ["trapezoid", "euler"])
def test_generated_code_bit_exact(name, N, scheme, staging):
    m = Model(MODELS[name], N, scheme)
    r = RefModel(MODELS[name], N, 1 if scheme == "trapezoid" else 0)
    x, lam = r.synth_acceptance(20250808)
    got, ref = run_all(m, x, lam, input_staging=staging), _ref_all(r, x, lam)
    for key in ("c_ok", "cjac_ok", "hess_ok", "grad_ok"):
        assert got[key] == ref[key], key
    flag_of = {"c": "c_ok", "c_cjac": "cjac_ok", "jac": "cjac_ok", "hess": "hess_ok", "grad": "grad_ok"}
    for key, flag in flag_of.items():
        if ref[flag]:
            assert np.array_equal(got[key], ref[key]), f"{name} {key} not bit-identical"


@pytest.mark.parametrize("name", ["goddard", "quadrotor", "shuttle", "hang_glider"])
def test_scaled_evaluation_bit_exact(name):
    """compute_scaling at x_start (eval.cpp:266-286) then scaled evaluation."""
    m, r = Model(MODELS[name], 20), RefModel(MODELS[name], 20)
    re = RefEval(r)
    obj_scale, row_scale = re.compute_scaling(r.arrays()["x_start"], True)
    x, lam = r.synth_acceptance(9)
    got = run_all(m, x, lam, obj_scale, row_scale)
    ok, c, j = re.constraints_jacobian(x)
    ok2, h = re.hessian(x, lam)
    assert ok and ok2 and got["cjac_ok"] and got["hess_ok"]
    assert np.array_equal(got["c_cjac"], c) and np.array_equal(got["jac"], j) and np.array_equal(got["hess"], h)


@pytest.mark.parametrize("name", list(MODELS))
def test_domain_flags_match_reference(name):
    """Points with zeros, sign flips, huge and subnormal values: the generated
    kernels flag exactly when the reference returns false (evaluator.cpp:79-84,
    126, 199, 229), and agree bitwise when both succeed."""
    N = 12
    m, r = Model(MODELS[name], N), RefModel(MODELS[name], N)
    rng = np.random.default_rng(1234)
    for trial in range(12):
        x, lam = r.synth_acceptance(100 + trial)
        idx = rng.choice(m.nvar, size=3, replace=False)
        kind = trial % 4
        if kind == 0:
            x[idx] = 0.0
        elif kind == 1:
            x[idx] = -x[idx]
        elif kind == 2:
            x[idx] = rng.choice([1e200, -1e200, 800.0, -800.0], size=3)
        else:
            x[idx] = rng.choice([1e-320, 1e308], size=3)
        got, ref = run_all(m, x, lam), _ref_all(r, x, lam)
        for key in ("c_ok", "cjac_ok", "hess_ok", "grad_ok"):
            assert got[key] == ref[key], (trial, key)
        if ref["cjac_ok"]:
            assert np.array_equal(got["jac"], ref["jac"])
        if ref["hess_ok"]:
            assert np.array_equal(got["hess"], ref["hess"])


@pytest.mark.parametrize("name", ["goddard", "quadrotor", "shuttle", "cart_pendulum"])
@pytest.mark.parametrize("split", ["0", "1", "2"])
def test_fused_kernel_bit_exact(name, split, monkeypatch):
    """ocg_cjh (one launch for c, J and H) in both copy-out modes: every output
    kind staged in its own shared region, or all kinds through one region."""
    monkeypatch.setenv("OCG_SPLIT", split)
    m = Model(MODELS[name], 70)
    r = RefModel(MODELS[name], 70)
    x, lam = r.synth_acceptance(99)
    got, ref = run_all(m, x, lam), _ref_all(r, x, lam)
    assert got["cjh_ok"] == (ref["cjac_ok"] and ref["hess_ok"])
    assert np.array_equal(got["cjh_c"], ref["c_cjac"])
    assert np.array_equal(got["cjh_jac"], ref["jac"])
    assert np.array_equal(got["cjh_hess"], ref["hess"])

