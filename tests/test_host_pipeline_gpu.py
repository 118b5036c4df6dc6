"""ocg_eval_jac_hess_host: the fused J+H evaluation from page-locked host
buffers to host buffers, pipelined over node-range chunks (chunk q's kernel on
the caller's stream, its c / jac_val / hess_val segments back on a second
stream while chunk q+1 computes). Every chunking must give exactly the values
of one whole-grid ocg_eval_jac_hess launch (same kernel, same inputs: bit-
identical), fill every output slot (host buffers start as NaN), and report
the bytes it moved; the values themselves are checked against the reference
EvalContext (tests/parity.py) at a size the oracle runs quickly.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from _oracle import RefEval, RefModel
from parity import assert_close
from paper_2510_03932_b200 import MODELS, EvalContext, Model

pytestmark = pytest.mark.gpu


def _host_buffers(m, ec):
    nan = float("nan")
    return (torch.full((m.m_con,), nan, dtype=torch.float64).pin_memory(),
            torch.full((ec.jac_nnz,), nan, dtype=torch.float64).pin_memory(),
            torch.full((ec.hess_nnz,), nan, dtype=torch.float64).pin_memory())


@pytest.mark.parametrize("name,N", [("goddard", 100_000), ("quadrotor", 100_000), ("shuttle", 20_000),
                                    ("hang_glider", 20_000), ("cart_pendulum", 5_000), ("goddard", 37)])
@pytest.mark.parametrize("block", [32, 128])
def test_pipelined_host_equals_device(name, N, block):
    m = Model(MODELS[name], N)
    x, lam = m.synth_acceptance(20250808)
    ec = EvalContext(m, device=0, block=block)
    xd = torch.as_tensor(x, device="cuda:0")
    ld = torch.as_tensor(lam, device="cuda:0")
    c = torch.empty(m.m_con, dtype=torch.float64, device="cuda:0")
    assert ec.eval_jac_hess(xd, ld, c)
    want = (c.cpu(), ec.jac_val.cpu(), ec.hess_val.cpu())
    xh, lh = torch.as_tensor(x).pin_memory(), torch.as_tensor(lam).pin_memory()
    for chunks in (1, 2, 3, 8, 1000):
        ch, jh, hh = _host_buffers(m, ec)
        ec.jac_val.fill_(float("nan"))
        ec.hess_val.fill_(float("nan"))
        stream = torch.cuda.current_stream()
        nbytes = ec.launch_jac_hess_host(xh, lh, ch, jh, hh, chunks=chunks, stream=stream)
        stream.synchronize()
        assert ec.status(), (name, chunks)
        for got, ref, what in zip((ch, jh, hh), want, ("c", "jac", "hess")):
            assert torch.equal(got, ref), (name, N, block, chunks, what)
        assert nbytes == 8 * (m.nvar + 2 * m.m_con + ec.jac_nnz + ec.hess_nnz), (nbytes, chunks)


@pytest.mark.parametrize("name", ["goddard", "shuttle"])
def test_pipelined_host_against_reference(name):
    N = 1500
    m, r = Model(MODELS[name], N), RefModel(MODELS[name], N)
    x, lam = r.synth_acceptance(20250808)
    ec, re = EvalContext(m, device=0), RefEval(r)
    ch, jh, hh = _host_buffers(m, ec)
    stream = torch.cuda.current_stream()
    ec.launch_jac_hess_host(torch.as_tensor(x).pin_memory(), torch.as_tensor(lam).pin_memory(), ch, jh, hh,
                            chunks=5, stream=stream)
    stream.synchronize()
    assert ec.status()
    ok1, c_r, j_r = re.constraints_jacobian(x)
    ok2, h_r = re.hessian(x, lam)
    assert ok1 and ok2
    assert_close(ch.numpy(), c_r, f"{name} c (host pipeline)", model=name)
    assert_close(jh.numpy(), j_r, f"{name} jac (host pipeline)", model=name)
    assert_close(hh.numpy(), h_r, f"{name} hess (host pipeline)", model=name)
    assert not np.isnan(hh.numpy()).any()
