"""Node-range sharding: host-side partition logic with a
world-size-2 gloo process group on CPU, and on the GPU the union of per-shard
evaluations reproducing the single-context evaluation bit for bit."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
from paper_2510_03932_b200 import MODELS, Model


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _covers(st, world, n_per):
    """Per rank: shard, bytes, output segments; checks disjoint full coverage."""
    out = []
    for r in range(world):
        a, b = bench.shard_of(st, r, world, n_per)
        out.append((a, b, bench.output_segments(st, a, b, r == 0)))
    return out


@pytest.mark.parametrize("name", ["goddard", "quadrotor", "cart_pendulum"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_shards_partition_every_output_once(name, world):
    n_per = 50
    m = Model(MODELS[name], n_per * world)
    st = m.structure()
    sizes = {"c": m.m_con}
    jac = sum(len(g["jac"]) * (g["range"][1] - g["range"][0] if not g["range"][2] else 2) for g in st["con_groups"])
    hess = sum(len(g["hess"]) * (g["range"][1] - g["range"][0] if not g["range"][2] else 2)
               for g in st["con_groups"] + st["obj_groups"])
    sizes.update(jac=jac, hess=hess)
    cover = {k: np.zeros(v, dtype=np.int64) for k, v in sizes.items()}
    lo, hi = bench.main_space(st)
    prev_b = lo
    for a, b, segs in _covers(st, world, n_per):
        assert a == prev_b
        prev_b = b
        for buf, s0, n in segs:
            cover[buf][s0:s0 + n] += 1
    assert prev_b == hi
    for k, v in cover.items():
        assert np.all(v == 1), f"{k}: entries covered {np.unique(v)} times"
    # algorithmic bytes add up to the single-shard figure except the halo nodes
    total = sum(bench.algorithmic_bytes(st, a, b, r == 0) for r, (a, b, _) in enumerate(_covers(st, world, n_per)))
    single = bench.algorithmic_bytes(st, lo, hi, True)
    halo = 8 * sum(d for _, d, _, nodes in st["layout"] if nodes > 1) * (world - 1)
    assert total == single + halo


def _worker(rank, world, port, name, n_per, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = Model(MODELS[name], n_per * world)
    st = m.structure()
    a, b = bench.shard_of(st, rank, world, n_per)
    nbytes = bench.algorithmic_bytes(st, a, b, rank == 0)
    # the bench's max-over-ranks reduction and the union of owned outputs
    t = torch.tensor([float(rank + 1), float(nbytes)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    segs = bench.output_segments(st, a, b, rank == 0)
    owned = torch.tensor([sum(n for _, _, n in segs)], dtype=torch.int64)
    dist.all_reduce(owned, op=dist.ReduceOp.SUM)
    if rank == 0:
        q.put((float(t[0]), int(owned[0])))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_reduction_and_ownership():
    world, n_per, name = 2, 40, "goddard"
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, n_per, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    tmax, owned = q.get(timeout=10)
    assert tmax == float(world)
    m = Model(MODELS[name], n_per * world)
    st = m.structure()
    lo, hi = bench.main_space(st)
    assert owned == sum(n for _, _, n in bench.output_segments(st, lo, hi, True))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["goddard", "quadrotor", "shuttle"])
def test_shard_union_equals_full_evaluation(name):
    """Two shard contexts (node ranges + the one-node halo read from x) write
    exactly the entries of the full evaluation, with identical values."""
    from paper_2510_03932_b200 import EvalContext
    N = 777
    m = Model(MODELS[name], N)
    st = m.structure()
    x, lam = m.synth_acceptance(20250808)
    full = EvalContext(m)
    dev = full.device
    xd, ld = torch.as_tensor(x, device=dev), torch.as_tensor(lam, device=dev)
    c_full = torch.zeros(m.m_con, dtype=torch.float64, device=dev)
    assert full.eval_jac_hess(xd, ld, c_full)
    c_sh = torch.full_like(c_full, float("nan"))
    jac = torch.full_like(full.jac_val, float("nan"))
    hess = torch.full_like(full.hess_val, float("nan"))
    world, n_per = 2, 400
    for r in range(world):
        a, b = bench.shard_of(st, r, world, n_per)
        ec = EvalContext(m, idx_lo=a, idx_hi=b if r < world - 1 else -1, specials=r == 0)
        ec.jac_val.fill_(float("nan"))
        ec.hess_val.fill_(float("nan"))
        c = torch.full_like(c_full, float("nan"))
        assert ec.eval_jac_hess(xd, ld, c)
        for buf, s0, n in bench.output_segments(st, a, b, r == 0):
            src = {"c": c, "jac": ec.jac_val, "hess": ec.hess_val}[buf]
            dst = {"c": c_sh, "jac": jac, "hess": hess}[buf]
            dst[s0:s0 + n] = src[s0:s0 + n]
    assert torch.equal(c_sh, c_full)
    assert torch.equal(jac, full.jac_val)
    assert torch.equal(hess, full.hess_val)


# ---- the objective over shards: chunk partials + exact masked sum + combine ----

def _split_points(st, world, per_chunks=2):
    """Shard boundaries on 512-chunk boundaries of the range objective group."""
    lo, hi = bench.main_space(st)
    g0 = min(g["range"][0] for g in st["obj_groups"] if not g["range"][2])
    cuts = [g0 + 512 * per_chunks * (r + 1) for r in range(world - 1)]
    return [lo] + cuts + [hi]


@pytest.mark.parametrize("name", ["quadrotor", "cart_pendulum", "goddard"])
@pytest.mark.parametrize("world", [2, 3])
def test_objective_chunks_owned_once(name, world):
    from paper_2510_03932_b200 import objective_chunk_owners
    m = Model(MODELS[name], 512 * 2 * world + 77)
    st = m.structure()
    cuts = _split_points(st, world)
    owners = [objective_chunk_owners(st, cuts[r], cuts[r + 1], r == 0) for r in range(world)]
    assert len({len(o) for o in owners}) == 1
    assert np.all(np.sum(owners, axis=0) == 1)


def test_objective_chunk_straddle_rejected():
    from paper_2510_03932_b200 import objective_chunk_owners
    st = Model(MODELS["quadrotor"], 3000).structure()
    with pytest.raises(ValueError):
        objective_chunk_owners(st, 0, 700, True)


def _combine_worker(rank, world, port, q):
    """Each rank holds stale garbage (NaN/inf) outside its own chunks; the
    masked SUM all-reduce must reproduce the full partials bit for bit."""
    from paper_2510_03932_b200 import objective_chunk_owners
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    st = Model(MODELS["quadrotor"], 512 * 2 * world + 77).structure()
    cuts = _split_points(st, world)
    own = torch.as_tensor(objective_chunk_owners(st, cuts[rank], cuts[rank + 1], rank == 0))
    full = torch.as_tensor(np.random.default_rng(5).standard_normal(len(own)) * 1e3)
    full[0] = -0.0
    stale = torch.full_like(full, float("nan"))
    stale[1::2] = float("inf")
    part = torch.where(own, full, stale)
    part = torch.where(own, part, torch.zeros((), dtype=torch.float64))
    dist.all_reduce(part, op=dist.ReduceOp.SUM)
    if rank == 0:
        q.put(bool(np.array_equal(part.numpy(), full.numpy())))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_objective_combine_exact():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_combine_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["quadrotor", "cart_pendulum", "goddard"])
def test_shard_objective_equals_full(name):
    """Per-shard chunk partials, masked and summed (the all-reduce, done here
    on one GPU), then combined: bit-identical to the unsharded objective."""
    from paper_2510_03932_b200 import EvalContext, objective_chunk_owners
    world = 3
    m = Model(MODELS[name], 512 * 2 * world + 77)
    st = m.structure()
    x, _ = m.synth_acceptance(20250808)
    full = EvalContext(m)
    ok, f_full = full.eval_objective(x)
    assert ok
    xd = torch.as_tensor(x, device=full.device)
    cuts = _split_points(st, world)
    total = None
    ctxs = []
    for r in range(world):
        ec = EvalContext(m, idx_lo=cuts[r], idx_hi=cuts[r + 1] if r < world - 1 else -1, specials=r == 0)
        ctxs.append(ec)
        part = torch.full((max(1, ec.objective_chunks),), float("nan"), dtype=torch.float64, device=ec.device)
        ec.launch_objective_partials(xd, part)
        own = torch.as_tensor(objective_chunk_owners(st, cuts[r], cuts[r + 1], r == 0), device=ec.device)
        part = torch.where(own, part, torch.zeros((), dtype=torch.float64, device=ec.device))
        total = part if total is None else total + part
    f = torch.empty(1, dtype=torch.float64, device=full.device)
    ctxs[0].launch_objective_combine(total, f)
    assert f.item() == f_full or (np.isnan(f_full) and np.isnan(f.item()))
    assert np.float64(f.item()).tobytes() == np.float64(f_full).tobytes()
    # single-rank path of the convenience wrapper
    ok2, f2 = full.eval_objective_sharded(x, torch.as_tensor(objective_chunk_owners(st, *bench.main_space(st), True)))
    assert ok2 and np.float64(f2).tobytes() == np.float64(f_full).tobytes()
