"""Sharded evaluation inside the library (ocg_eval_create_sharded,
csrc/shard.cpp) against one unsharded context on the same
inputs: each rank uploads only the x slots it owns and the multiplier rows of
its instances, receives its halo over the communicator, and its outputs (c,
J, H of its instances) are bit-identical to the unsharded context's; the
objective over all ranks (chunk partials, masked sum, fixed-order combine)
equals the unsharded objective bit for bit, and the ok flag is reduced.

- Comm.nccl at world 1 (the only NCCL size one GPU allows);
- Comm.host over gloo with two processes sharing the GPU: the halo exchange
  and the reductions through the library's host-callback path.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _segments(st, lo, hi, specials):
    from test_shard_plan import _rank_segments
    return _rank_segments(st, lo, hi, specials)


def _check_rank(name, N, comm, device=0):
    from paper_2510_03932_b200 import MODELS, EvalContext, Model
    m = Model(MODELS[name], N)
    x, lam = m.synth_acceptance(20250808)
    ref = EvalContext(m, device=device)
    dev = ref.device
    xd, ld = torch.as_tensor(x, device=dev), torch.as_tensor(lam, device=dev)
    c_ref = torch.empty(m.m_con, dtype=torch.float64, device=dev)
    assert ref.eval_jac_hess(xd, ld, c_ref)
    ok_f, f_ref = ref.eval_objective(xd)
    assert ok_f

    ec = EvalContext(m, device=device, comm=comm)
    sh = ec.shard()
    # device buffers start as NaN: whatever the rank neither owns nor receives stays NaN
    xs = torch.full((m.nvar,), float("nan"), dtype=torch.float64, device=dev)
    ls = torch.full((m.m_con,), float("nan"), dtype=torch.float64, device=dev)
    c = torch.full((m.m_con,), float("nan"), dtype=torch.float64, device=dev)
    h2d_x = ec.scatter_x(x, xs)
    h2d_l = ec.scatter_rows(lam, ls)
    torch.cuda.synchronize()
    assert h2d_x < 8 * m.nvar or sh["world"] == 1
    assert ec.eval_jac_hess(xs, ls, c)
    assert ec.status_all()
    seg = _segments(m.structure(), sh["idx_lo"], sh["idx_hi"], bool(sh["specials"]))
    for a, b in seg["rows"]:
        assert torch.equal(c[a:b], c_ref[a:b])
    for a, b in seg["jac"]:
        assert torch.equal(ec.jac_val[a:b], ref.jac_val[a:b])
    for a, b in seg["hess"]:
        assert torch.equal(ec.hess_val[a:b], ref.hess_val[a:b])
    ok, f = ec.objective_all(xs)
    assert ok and f == f_ref, (f, f_ref)
    return sh, h2d_x, h2d_l


@pytest.mark.parametrize("name", ["goddard", "quadrotor"])
def test_sharded_nccl_world1(name):
    from paper_2510_03932_b200 import Comm
    uid = Comm.nccl_unique_id()
    comm = Comm.nccl(0, 1, 0, uid)
    sh, _, _ = _check_rank(name, 3000, comm)
    assert sh["world"] == 1 and sh["halo_doubles"] == 0


def _host_worker(rank, world, port, name, N, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(__file__))
        from paper_2510_03932_b200 import Comm
        comm = Comm.host(0)
        sh, h2d_x, h2d_l = _check_rank(name, N, comm)
        q.put((rank, sh, h2d_x, h2d_l, None))
    except Exception as ex:  # noqa: BLE001
        import traceback
        q.put((rank, None, 0, 0, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,N", [("goddard", 6000), ("quadrotor", 4000), ("cart_pendulum", 3000)])
def test_sharded_host_comm_two_ranks_one_gpu(name, N):
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_host_worker, args=(r, 2, port, name, N, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=120)
    for rank, sh, h2d_x, h2d_l, err in res:
        assert err is None, f"rank {rank}:\n{err}"
        assert sh["world"] == 2
    assert res[0][1]["halo_doubles"] > 0  # rank 0 reads its right neighbour's first node (and node N)
    # the two ranks uploaded about half of x each (plus the shared free variables)
    assert abs(res[0][2] - res[1][2]) < 0.2 * (res[0][2] + res[1][2])
