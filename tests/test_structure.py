"""CPU: the front end (DSL -> transcription -> graphs -> sparsity) builds the
same StructuredNlp as the reference: node lists, input ordinals and
addresses, Jacobian/Hessian patterns, ranges, row bases, bounds and start
point — the inputs every COO offset is derived from."""
from __future__ import annotations

import json
import math
from pathlib import Path

import numpy as np
import pytest

from _oracle import RefModel
from paper_2510_03932_b200 import MODELS, Model

GOLDEN = Path(__file__).resolve().parent / "golden"


def _norm(o):
    """JSON-normalise: the reference dumps +-inf as null."""
    if isinstance(o, dict):
        return {k: _norm(v) for k, v in o.items()}
    if isinstance(o, list):
        return [_norm(v) for v in o]
    if isinstance(o, float) and math.isinf(o):
        return None
    return o


@pytest.mark.parametrize("name", list(MODELS))
@pytest.mark.parametrize("scheme", ["trapezoid", "euler"])
@pytest.mark.parametrize("N", [1, 2, 7, 100])
def test_structure_matches_reference(name, scheme, N):
    m = Model(MODELS[name], N, scheme)
    r = RefModel(MODELS[name], N, 1 if scheme == "trapezoid" else 0)
    assert _norm(m.structure()) == _norm(r.structure())
    a, b = m.arrays(), r.arrays()
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_boxes_as_bounds_option():
    m = Model(MODELS["goddard"], 50, boxes_as_bounds=True)
    r = RefModel(MODELS["goddard"], 50, boxes_as_bounds=True)
    assert _norm(m.structure()) == _norm(r.structure())
    assert m.nvar + m.m_con == 7 * 50 + 9  # transcribe_test.cpp:340-352


def test_problem_sizes():
    """transcribe_test.cpp:109-125: DI 9/8 at N=2; Goddard 10N+12; quadrotor 22N+22."""
    di = Model(MODELS["double_integrator"], 2)
    assert (di.nvar, di.m_con) == (9, 8)
    for N in (10, 100, 1000):
        g, q = Model(MODELS["goddard"], N), Model(MODELS["quadrotor"], N)
        assert g.nvar + g.m_con == 10 * N + 12
        assert q.nvar + q.m_con == 22 * N + 22


def test_golden_double_integrator_dump():
    """proj/tests/golden/double_integrator_n2_nlp.json (committed copy of the
    reference's --dump-nlp golden): layout, input addresses and labels, nnz per
    group, row bases, ranges, bounds, start point."""
    gold = json.loads((GOLDEN / "double_integrator_n2_nlp.json").read_text())
    st = Model(MODELS["double_integrator"], 2).structure()
    assert st["nvar"] == gold["nvar"] and st["m_con"] == gold["m_con"]
    assert [s[2] for s in st["layout"]] == [s["base"] for s in gold["layout"]]
    for g, gg in zip(st["con_groups"], gold["constraint_groups"]):
        assert [[i[0], i[1], i[2]] for i in g["inputs"]] == [[i["base"], i["stride"], i["label"]]
                                                            for i in gg["kernel"]["inputs"]]
        assert len(g["jac"]) == gg["kernel"]["jac_nnz"] and len(g["hess"]) == gg["kernel"]["hess_nnz"]
        assert g["row_base"] == gg["row_base"] and g["label"] == gg["label"]
        assert g["range"] == [gg["range"]["lo"], gg["range"]["hi"], gg["range"]["endpoints_only"]]
    for g, gg in zip(st["obj_groups"], gold["objective_groups"]):
        assert g["weight"] == gg["weight"] and g["label"] == gg["label"]
        assert len(g["jac"]) == gg["kernel"]["jac_nnz"] and len(g["hess"]) == gg["kernel"]["hess_nnz"]
    assert Model(MODELS["double_integrator"], 2).arrays()["x_start"].tolist() == gold["x_start"]


@pytest.mark.parametrize("src,needle", [
    ("t in [0, 1], time\nx in R^2, state\nu in R, control\nx(0) == [1, 2, 3]\n"
     "derivative(x1)(t) == x2(t)\nderivative(x2)(t) == u(t)\nintegral(u(t)^2) => min\n", "wrong bound dimension"),
    ("t in [0, 1], time\nx in R^2, state\nu in R, control\nderivative(x1)(t) == x2(t)\n"
     "integral(u(t)^2) => min\n", "missing dynamics"),
    ("x in R, state\n", "missing time"),
])
def test_parse_errors(src, needle):
    with pytest.raises(Exception) as ei:
        Model(src, 4)
    assert needle in str(ei.value)
