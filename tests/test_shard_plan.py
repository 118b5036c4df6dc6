"""Node-range shard plans (host only, csrc/shard.cpp): every
slot of x is uploaded by exactly one rank, every exchange a rank expects is
one its peer sends (same runs, same order), every slot a rank's instances
read — the columns of its Jacobian and Hessian entries — is owned or
received, the constraint rows of its instances are uploaded, and every
objective chunk (reference par_reduce, backend.cpp:119-133) is owned by
exactly one rank. Plus the torch.distributed host callbacks of Comm.host
over gloo with two processes."""
from __future__ import annotations

import os

import numpy as np
import pytest

from paper_2510_03932_b200 import MODELS, Model, shard_plan


def _rank_segments(st, lo, hi, specials):
    """jac / hess entry ranges and c rows of the instances of one rank."""
    segs = {"jac": [], "hess": [], "rows": []}
    joff = hoff = 0
    for g in st["con_groups"]:
        a, b, ends = g["range"]
        cnt = 2 if ends else b - a
        nj, nh, od = len(g["jac"]), len(g["hess"]), g["out_dim"]
        k0, k1 = ((0, cnt) if specials else (0, 0)) if ends else (max(0, max(a, lo) - a), max(0, min(b, hi) - a))
        if k1 > k0:
            segs["jac"].append((joff + k0 * nj, joff + k1 * nj))
            segs["hess"].append((hoff + k0 * nh, hoff + k1 * nh))
            segs["rows"].append((g["row_base"] + k0 * od, g["row_base"] + k1 * od))
        joff += cnt * nj
        hoff += cnt * nh
    for g in st["obj_groups"]:
        a, b, ends = g["range"]
        cnt = 2 if ends else b - a
        nh = len(g["hess"])
        k0, k1 = ((0, cnt) if specials else (0, 0)) if ends else (max(0, max(a, lo) - a), max(0, min(b, hi) - a))
        if k1 > k0:
            segs["hess"].append((hoff + k0 * nh, hoff + k1 * nh))
        hoff += cnt * nh
    return segs


def _mask(n, runs):
    m = np.zeros(n, dtype=np.int32)
    for off, ln in runs:
        m[off:off + ln] += 1
    return m


@pytest.mark.parametrize("name", ["goddard", "quadrotor", "double_integrator", "hang_glider", "shuttle", "cart_pendulum"])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_plan_consistent(name, world):
    N = 5000
    m = Model(MODELS[name], N)
    st = m.structure()
    plans = [shard_plan(m, q, world) for q in range(world)]
    # every node slot uploaded by exactly one rank, the free variables (e.g. tf) by every rank
    up = sum(_mask(m.nvar, p["x_own"]) for p in plans)
    free = np.zeros(m.nvar, dtype=bool)
    for kind, dim, base, nodes in st["layout"]:
        if nodes == 1:
            free[base:base + dim] = True
    assert np.all(up[~free] == 1), f"node slots uploaded {up[~free].min()}..{up[~free].max()} times"
    assert np.all(up[free] == world)
    # exchanges match pairwise, in order
    for q in range(world):
        for o in range(world):
            assert plans[q]["recv_from"][o] == plans[o]["send_to"][q]
    # ranges partition the main grid; chunks owned once
    assert plans[0]["lo"] == min(p["lo"] for p in plans)
    for q in range(world - 1):
        assert plans[q]["hi"] == plans[q + 1]["lo"]
    assert all(p["objective_exact"] for p in plans)
    owned = np.sum([np.array(p["chunk_owned"], dtype=np.int32) for p in plans], axis=0)
    assert np.all(owned == 1)
    # what a rank reads is owned or received
    cols = st_cols(m)
    for q, p in enumerate(plans):
        seg = _rank_segments(st, p["lo"], p["hi"], p["specials"])
        have = (_mask(m.nvar, p["x_own"]) + _mask(m.nvar, [r for runs in p["recv_from"] for r in runs])) > 0
        read = np.zeros(m.nvar, dtype=bool)
        for a, b in seg["jac"]:
            read[cols["jac_col"][a:b]] = True
        for a, b in seg["hess"]:
            read[cols["hess_row"][a:b]] = True
            read[cols["hess_col"][a:b]] = True
        missing = np.nonzero(read & ~have)[0]
        assert missing.size == 0, f"rank {q} reads slots it neither owns nor receives: {missing[:8]}"
        rows = _mask(m.m_con, p["rows"]) > 0
        for a, b in seg["rows"]:
            assert rows[a:b].all()
        if world > 1:  # the halo is small: a node per neighbour (+ node N on rank 0)
            assert p["halo_doubles"] <= 2 * m.nvar // (N + 1) + 64


def st_cols(m):
    """Columns of the model's COO entries from the structure JSON (the
    groups' inputs and patterns); no device needed."""
    if True:
        st = m.structure()
        jc, hr, hc = [], [], []
        for g in st["con_groups"]:
            a, b, ends = g["range"]
            for k in ([a, b] if ends else range(a, b)):
                for (r, i) in g["jac"]:
                    jc.append(_slot(g, i, k))
                for (j, i) in g["hess"]:
                    hr.append(_slot(g, i, k))
                    hc.append(_slot(g, j, k))
        for g in st["obj_groups"]:
            a, b, ends = g["range"]
            for k in ([a, b] if ends else range(a, b)):
                for (j, i) in g["hess"]:
                    hr.append(_slot(g, i, k))
                    hc.append(_slot(g, j, k))
        return {"jac_col": np.array(jc, dtype=np.int64), "hess_row": np.array(hr, dtype=np.int64),
                "hess_col": np.array(hc, dtype=np.int64)}


def _slot(g, i, k):
    base, stride = g["inputs"][i][:2]
    return base + stride * k


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ctypes as C

        from paper_2510_03932_b200 import _lib
        from paper_2510_03932_b200.evaluation import host_comm_callbacks
        ar_f, ar_i, sr = host_comm_callbacks(None)
        buf = np.array([rank + 0.5, 10.0 * rank], dtype=np.float64)
        assert ar_f(None, buf.ctypes.data_as(C.POINTER(C.c_double)), 2) == 0
        ib = np.array([rank, -rank], dtype=np.int32)
        assert ar_i(None, ib.ctypes.data_as(C.POINTER(C.c_int32)), 2) == 0
        # each rank sends its rank-stamped vector to the next, receives from the previous
        to, frm = (rank + 1) % world, (rank - 1) % world
        send = np.full(3, 100.0 + rank)
        recv = np.zeros(3)
        assert sr(None, send.ctypes.data_as(C.POINTER(C.c_double)), 3, to,
                  recv.ctypes.data_as(C.POINTER(C.c_double)), 3, frm) == 0
        # zero-length in one direction must not communicate
        z = np.zeros(0)
        if rank == 0:
            assert sr(None, send.ctypes.data_as(C.POINTER(C.c_double)), 3, 1,
                      z.ctypes.data_as(C.POINTER(C.c_double)), 0, 1) == 0
        else:
            got = np.zeros(3)
            assert sr(None, z.ctypes.data_as(C.POINTER(C.c_double)), 0, 0,
                      got.ctypes.data_as(C.POINTER(C.c_double)), 3, 0) == 0
            assert np.array_equal(got, np.full(3, 100.0))
        # plans: my sends to the peer are the peer's expected receives
        m = Model(MODELS["goddard"], 3000)
        p = shard_plan(m, rank, world)
        n_send = np.array([sum(ln for _, ln in p["send_to"][to])], dtype=np.int64)
        n_recv = np.zeros(1, dtype=np.int64)
        reqs = [dist.isend(torch.from_numpy(n_send), to), dist.irecv(torch.from_numpy(n_recv), frm)]
        for r_ in reqs:
            r_.wait()
        ok = n_recv[0] == sum(ln for _, ln in p["recv_from"][frm])
        _ = _lib
        q.put((rank, buf.tolist(), ib.tolist(), recv.tolist(), bool(ok)))
    finally:
        dist.destroy_process_group()


def test_host_comm_callbacks_gloo_world2():
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=180) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, buf, ib, recv, ok in res:
        assert buf == [0.5 + 1.5, 0.0 + 10.0]
        assert ib == [1, 0]
        assert recv == [100.0 + (rank - 1) % 2] * 3
        assert ok
