"""Reference-order symbolic analysis (host only, no GPU): the product's
ordering + pivot_after_ deferral + analyze_ordered (ocg_ldl_ref_symbolic,
csrc/refldl.cpp) against the reference's own KktAssembler::symbolic()
(proj/src/ipm/eval.cpp:442-471, proj/src/sparse/ldl.cpp:54-137) compiled in
oracle/_ref/libref.so: the elimination order, the elimination tree and the
pattern of L must be identical, for every model and both schemes.
"""
from __future__ import annotations

import numpy as np
import pytest

from _oracle import RefEval, RefKkt, RefModel
from paper_2510_03932_b200 import MODELS, ref_symbolic

CASES = [("double_integrator", 50, 1), ("goddard", 10, 1), ("goddard", 1000, 1), ("goddard", 300, 0),
         ("quadrotor", 40, 1), ("cart_pendulum", 60, 1), ("hang_glider", 30, 1), ("shuttle", 25, 1),
         ("goddard", 20000, 1)]


@pytest.mark.parametrize("name,N,scheme", CASES)
def test_ref_symbolic_equals_reference(name, N, scheme):
    rm = RefModel(MODELS[name], N, scheme=scheme)
    rk = RefKkt(RefEval(rm))
    colp, rowi = rk.pattern()
    ref = rk.symbolic()
    got = ref_symbolic(colp, rowi, rk.n_free, rk.ntot)
    assert np.array_equal(got["perm"], ref["perm"]), f"{name}@{N}: elimination order differs"
    assert np.array_equal(got["parent"], ref["parent"]), f"{name}@{N}: elimination tree differs"
    assert np.array_equal(got["Lp"], ref["Lp"]), f"{name}@{N}: column counts of L differ"
    assert len(got["Li"]) == ref["lnz"]


@pytest.mark.parametrize("name,N", [("goddard", 200), ("quadrotor", 30)])
def test_ref_symbolic_li_equals_reference_factor_pattern(name, N):
    """Li (rows of each column, ascending) is the pattern sparse::factorize fills."""
    rm = RefModel(MODELS[name], N)
    rk = RefKkt(RefEval(rm))
    colp, rowi = rk.pattern()
    got = ref_symbolic(colp, rowi, rk.n_free, rk.ntot)
    f = rk.factorize(np.ones(rk.nnz), 1.0, 1.0)
    assert np.array_equal(got["Li"], f["Li"])
