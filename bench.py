#!/usr/bin/env python
"""bench.py — the derivative-evaluation hot path of arXiv 2510.03932's `octrans`
on B200, in the driver's one-JSON-line contract.

Step = one fused `eval_constraints_jacobian` + `eval_hessian` pass (the
reference's EvalContext J+H node-step) over every time node of
the configured OCP, through the C ABI (include/octgpu.h: ocg_eval_jac_hess).
Default workload = BASELINE.json configs[1]: Goddard rocket, trapezoidal
transcription, N = 1e5 nodes per GPU (weak scaling: N per GPU fixed, the
problem has N x world nodes, each rank evaluates its contiguous node range).

metric "jac+hess eval ns/node" (lower is better): max-over-ranks device time
per step / total nodes. Inputs are the reference's acceptance recipe
(acceptance_main.cpp:179-193, mt19937(20250808)); L2 is flushed (a 512 MiB
read) before every timed step, outside the events.

--impl reference: the reference's own CPU EvalContext (oracle/_ref/libref.so,
the unmodified reference sources) with its parallel Backend on all host
cores, same model/N/metric; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent
L2_FLUSH_BYTES = 512 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", default="goddard")
    ap.add_argument("--N", type=int, default=100_000, help="time nodes per GPU")
    ap.add_argument("--scheme", default="trapezoid")
    # one-warp blocks: 16.5-16.6 us per Goddard N=1e5 step against 17.2-17.3
    # with four-warp blocks, alternated on one box (profiles/r2_block_ab.jsonl);
    # both are parity-tested at every bench config (test_eval_bench_configs.py)
    ap.add_argument("--block", type=int, default=32)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--lib-shard", action="store_true",
                    help="use the library's sharded context (NCCL communicator) even on one rank")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the other eval configs (quadrotor 1e6 and 1e5, hang glider, shuttle; 'extra' key)")
    ap.add_argument("--solve", default="quadrotor:100000",
                    help="model:N of the full IPM solve leg ('ipm_solve' key; 'none' to skip)")
    ap.add_argument("--goddard-solve", default="100000:10",
                    help="N[:ref_iters] of the Goddard full device solve (BASELINE config 2, 'goddard_solve' key); the "
                         "reference runs ref_iters iterations for a per-iteration comparison; 'none' to skip")
    ap.add_argument("--goddard-parity", default="1000",
                    help="N of the Goddard solve with the reference-order factorization (BASELINE configs[0]: "
                         "iterations, factorizations and objective against the reference's; "
                         "'goddard_parity_solve' key; 'none' to skip)")
    ap.add_argument("--batch", default="4096:500",
                    help="instances:N of the batched cart-pendulum solve leg (BASELINE config 5, 'batch_solve' "
                         "key; 'none' to skip)")
    return ap.parse_args()


def peaks() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            for k in ("hbm_gbs", "hbm_GBs", "hbm"):
                if k in d:
                    return float(d[k]), "measured"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback"


# ---------------------------------------------------------------------------
# workload geometry: shard ranges and algorithmic bytes
# ---------------------------------------------------------------------------

def main_space(st: dict) -> tuple[int, int]:
    lo, hi = None, None
    for g in st["con_groups"] + st["obj_groups"]:
        a, b, ends = g["range"]
        if ends:
            continue
        lo = a if lo is None else min(lo, a)
        hi = b if hi is None else max(hi, b)
    return lo or 0, hi or 0


def shard_of(st: dict, rank: int, world: int, n_per: int) -> tuple[int, int]:
    lo, hi = main_space(st)
    a = lo + rank * n_per
    b = hi if rank == world - 1 else lo + (rank + 1) * n_per
    return a, b


def _is_tail(g: dict) -> bool:
    return bool(g["range"][2]) or g.get("kind", -1) == 2


def _count(g: dict, a: int, b: int, specials: bool) -> int:
    lo, hi, ends = g["range"]
    if _is_tail(g):
        return (2 if ends else hi - lo) if specials else 0
    return max(0, min(hi, b) - max(lo, a))


def algorithmic_bytes(st: dict, a: int, b: int, specials: bool) -> int:
    """8 x [x reads + lambda reads + row_scale reads + c writes + J + H] for
    the shard's instances (SURVEY.md §8d B_node; index arrays not counted)."""
    words = 0
    for kind, dim, base, nodes in st["layout"]:
        if nodes > 1:
            words += dim * max(0, min(nodes, b + 1) - a)  # node slab incl. the one-node halo
        elif specials:
            words += dim * nodes
    for g in st["con_groups"]:
        n = _count(g, a, b, specials)
        od = g["out_dim"]
        words += n * (2 * od + len(g["jac"]) + len(g["hess"]) + (od if g["hess"] else 0))
    for g in st["obj_groups"]:
        words += _count(g, a, b, specials) * len(g["hess"])
    return 8 * words


def output_segments(st: dict, a: int, b: int, specials: bool) -> list[tuple[str, int, int]]:
    """(buffer, start, count) of every COO/c segment this shard writes; adjacent
    segments merged. Used for the end-to-end device->host copies."""
    segs = []
    joff = hoff = 0
    for g in st["con_groups"]:
        lo, hi, _ = g["range"]
        cnt = (hi - lo) if not g["range"][2] else 2
        nj, nh, od = len(g["jac"]), len(g["hess"]), g["out_dim"]
        if _is_tail(g):
            k0, k1 = (0, cnt) if specials else (0, 0)
        else:
            k0, k1 = max(0, max(lo, a) - lo), max(0, min(hi, b) - lo)
        if k1 > k0:
            segs.append(("c", g["row_base"] + k0 * od, (k1 - k0) * od))
            segs.append(("jac", joff + k0 * nj, (k1 - k0) * nj))
            segs.append(("hess", hoff + k0 * nh, (k1 - k0) * nh))
        joff += cnt * nj
        hoff += cnt * nh
    for g in st["obj_groups"]:
        lo, hi, ends = g["range"]
        cnt = (hi - lo) if not ends else 2
        nh = len(g["hess"])
        if _is_tail(g):
            k0, k1 = (0, cnt) if specials else (0, 0)
        else:
            k0, k1 = max(0, max(lo, a) - lo), max(0, min(hi, b) - lo)
        if k1 > k0 and nh:
            segs.append(("hess", hoff + k0 * nh, (k1 - k0) * nh))
        hoff += cnt * nh
    merged: list[list] = []
    for buf, s, n in sorted((x for x in segs if x[2] > 0), key=lambda t: (t[0], t[1])):
        if merged and merged[-1][0] == buf and merged[-1][1] + merged[-1][2] == s:
            merged[-1][2] += n
        else:
            merged.append([buf, s, n])
    return [tuple(m) for m in merged]


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------

class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self._t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU legs: the reference EvalContext (oracle/_ref/libref.so)
# ---------------------------------------------------------------------------

def _ref_modules():
    sys.path.insert(0, str(ROOT / "tests"))
    from _oracle import RefEval, RefModel  # noqa: E402  (checker: cpu_baseline / reference arm only)
    return RefEval, RefModel


def load_models():
    """models.py (model TEXT only, no imports) loaded by path, so that the
    reference arm never imports the package (which maps libocgpu.so)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("_ocg_model_texts", ROOT / "paper_2510_03932_b200" / "models.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def bench_config(args, world: int) -> dict:
    """The workload both arms report: identical dict (the driver compares them)."""
    N = args.N * world
    return {"workload": f"{args.model} {args.scheme} N={N} ({args.N} nodes/GPU) J+H eval "
                        "(EvalContext::eval_constraints_jacobian + eval_hessian)",
            "model": args.model, "N": N, "nodes_per_gpu": args.N, "scheme": args.scheme,
            "parallelism": f"node-range shards x{world}",
            "l2": "device: flushed (512 MiB read) before every timed step",
            "inputs": "acceptance recipe mt19937(20250808)"}


def _median_steps(re, x, lam, reps: int, warmup: int = 1) -> list[float]:
    for _ in range(max(warmup, 1)):
        t1, ok = re.step_seconds(x, lam, 1)
        assert ok, "reference evaluation failed on the synthetic point"
    return [re.step_seconds(x, lam, 1)[0] for _ in range(reps)]


def cpu_reference_eval(src: str, N: int, scheme: str, reps: int = 5, serial: bool = True,
                       outputs: bool = False) -> dict:
    """the reference EvalContext J+H step (eval_constraints_jacobian
    + eval_hessian) with Backend::parallel on every host core and with
    Backend::serial, median of `reps` after one warm-up each."""
    RefEval, RefModel = _ref_modules()
    cores = os.cpu_count() or 1
    rm = RefModel(src, N, 1 if scheme == "trapezoid" else 0)
    x, lam = rm.synth_acceptance(20250808)
    re = RefEval(rm, parallel=True, workers=cores)
    par = _median_steps(re, x, lam, reps)
    out = {"parallel": {"median_s": float(np.median(par)), "times_s": par, "workers": int(re.L.ref_eval_workers(re.h))},
           "cpu_model": cpu_model(), "nproc": cores, "reps": reps}
    if serial:
        rs = RefEval(rm, parallel=False)
        ser = _median_steps(rs, x, lam, reps)
        out["serial"] = {"median_s": float(np.median(ser)), "times_s": ser, "workers": 1}
        del rs
    if outputs:
        ok1, c_r, j_r = re.constraints_jacobian(x)
        ok2, h_r = re.hessian(x, lam)
        out["outputs"] = (ok1 and ok2, c_r, j_r, h_r)
    return out


def dropin_e2e(src: str, N: int, scheme: str, steps: int, warmup: int) -> dict | None:
    """End to end through the REFERENCE's API: EvalContext::eval_constraints_jacobian
    + eval_hessian of the drop-in build (integration/_out/libref_accel.so: the
    reference's own classes with integration/octrans_accel.cpp in place of
    proj/src/ipm/eval.cpp), host std::vectors in and out, as the reference's
    Solver calls them. Each call uploads x (and lambda), runs the device
    kernels and copies c / jac_val / hess_val back before returning."""
    try:
        sys.path.insert(0, str(ROOT / "tests"))
        from _oracle import RefEval, RefModel  # noqa: E402
        rm = RefModel(src, N, 1 if scheme == "trapezoid" else 0, lib="accel")
    except Exception as ex:  # drop-in not built on this box
        return {"unavailable": str(ex)}
    x, lam = rm.synth_acceptance(20250808)
    re = RefEval(rm)
    for _ in range(max(warmup, 1)):
        assert re.step_seconds(x, lam, 1)[1]
    ts = [re.step_seconds(x, lam, 1)[0] for _ in range(steps)]
    sz = np.zeros(3, dtype=np.int64)
    re.L.ref_eval_sizes(re.h, sz.ctypes.data)
    jn, hn = int(sz[0]), int(sz[1])
    return {"median_s": float(np.median(ts)), "mean_s": float(np.mean(ts)), "steps": steps,
            "h2d": 8 * (2 * rm.nvar + rm.m_con), "d2h": 8 * (rm.m_con + jn + hn)}


def dropin_e2e_isolated(name: str, N: int, scheme: str, steps: int, warmup: int) -> dict | None:
    """dropin_e2e in a fresh process: in the bench process the drop-in's host
    copy threads competed with the (spinning) thread pools left by the
    measurements before it — 14.5 ns/node alone, 17.7-24.2 in-process on the
    same box. The measurement itself is unchanged."""
    try:
        r = subprocess.run([sys.executable, str(Path(__file__).resolve()), "--dropin-e2e-child",
                            f"{name}:{N}:{scheme}:{steps}:{warmup}"], capture_output=True, text=True, timeout=600)
        return json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as ex:
        return {"unavailable": f"drop-in child process: {ex}"}


def batch_solve_isolated(spec: str, with_reference: bool) -> dict:
    """batch_solve_leg in a fresh process: the batched solver's host thread
    issues ~1800 launch groups per batch, and in the bench process it competed
    with the spinning thread pools the reference measurements leave behind
    (whole-batch walls 1.1-2.2 s against a steady 0.86 s alone on the same
    box, device time unchanged). The measurement itself is unchanged."""
    try:
        r = subprocess.run([sys.executable, str(Path(__file__).resolve()), "--batch-child",
                            f"{spec}:{int(with_reference)}"], capture_output=True, text=True, timeout=1200)
        return json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as ex:
        return {"unavailable": f"batch child process: {ex}"}


def parity_of(name: str, got: dict, ref: tuple) -> dict:
    """max relative error of the device c / jac / hess against the reference
    EvalContext on the same inputs (tests/parity.py rule with the model's floor)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from parity import floor_for, rel_errors  # noqa: E402
    ok, c_r, j_r, h_r = ref
    fl = floor_for(name)
    res = {"reference_ok": bool(ok), "floor": fl, "tolerance": 1e-12}
    worst, worst0, exact, n = 0.0, 0.0, 0, 0
    for k, r in (("c", c_r), ("jac", j_r), ("hess", h_r)):
        g = got[k]
        e = rel_errors(g, r, fl)
        e0 = rel_errors(g, r, 0.0)
        res[f"max_rel_err_{k}"] = float(e.max()) if e.size else 0.0
        worst = max(worst, res[f"max_rel_err_{k}"])
        worst0 = max(worst0, float(e0.max()) if e0.size else 0.0)
        exact += int(np.sum(g == r))
        n += r.size
    res["max_rel_err"] = worst
    res["max_rel_err_nofloor"] = worst0
    res["bit_exact_frac"] = exact / max(n, 1)
    res["entries"] = n
    return res


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    src = load_models().MODELS[args.model]
    world = args.gpus
    N = args.N * world
    RefEval, RefModel = _ref_modules()
    cores = os.cpu_count() or 1
    rm = RefModel(src, N, 1 if args.scheme == "trapezoid" else 0)
    x, lam = rm.synth_acceptance(20250808)
    re = RefEval(rm, parallel=True, workers=cores)
    for _ in range(max(args.warmup, 1)):
        re.step_seconds(x, lam, 1)
    times = [re.step_seconds(x, lam, 1)[0] for _ in range(args.steps)]
    workers = int(re.L.ref_eval_workers(re.h))
    t = float(np.mean(times))
    val = t * 1e9 / N
    line = {
        "metric": "jac+hess eval ns/node", "value": val, "unit": "ns/node", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args, world),
        "cpu_baseline": {"value": val, "unit": "ns/node", "cores": workers, "kind": "reference",
                         "cpu_model": cpu_model(), "nproc": cores,
                         "median_ns_per_node": float(np.median(times)) * 1e9 / N,
                         "sample": f"full workload (N={N}), {args.steps} steps after {args.warmup} warm-up, "
                                   f"reference EvalContext (oracle/_ref/libref.so) with Backend::parallel "
                                   f"x{workers} workers"},
        "e2e": {"value": val, "unit": "ns/node", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def time_eval_config(ec, xd, ld, c, flush, sink, stream, steps: int, warmup: int, halo: bool = False):
    """Per-step CUDA events around exactly one fused J+H launch — preceded, on
    a sharded context, by the halo exchange over the communicator (ncclSend /
    ncclRecv on the same stream); the L2 flush (a 512 MiB read) runs before
    each step outside the events."""
    import torch
    for _ in range(warmup):
        torch.sum(flush, dim=0, out=sink)
        if halo:
            ec.halo_exchange(xd, stream)
        ec.launch_jac_hess(xd, ld, c, stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    n0 = ec.launch_count
    for s, e in ev:
        torch.sum(flush, dim=0, out=sink)
        s.record(stream)
        if halo:
            ec.halo_exchange(xd, stream)
        ec.launch_jac_hess(xd, ld, c, stream)
        e.record(stream)
    stream.synchronize()
    launches = ec.launch_count - n0
    return [s.elapsed_time(e) * 1e-3 for s, e in ev], launches


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2510_03932_b200 import MODELS, EvalContext, Model

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ngpu = torch.cuda.device_count()
    if world > 1:
        if ngpu >= world:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            # fewer GPUs than ranks (a functional check of the sharded path on
            # one device): ranks share devices, host-side collectives over gloo
            local = local % max(1, ngpu)
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)

    # the batched-solve leg first, in a child process, before this process has
    # started any reference thread pools (they keep spinning afterwards and
    # the batch's host launch loop competed with them even from a child:
    # whole-batch walls 1.1-2.5 s against a steady 0.86 s otherwise)
    batch_early = None
    if args.batch != "none" and world == 1:
        batch_early = batch_solve_isolated(args.batch, not args.no_cpu_baseline)
    src = MODELS[args.model]
    N = args.N * world
    m = Model(src, N, args.scheme)
    st = m.structure()
    x, lam = m.synth_acceptance(20250808)
    sharded = world > 1 or args.lib_shard
    comm = None
    if sharded:
        # node-range shards inside the library (ocg_eval_create_sharded): NCCL
        # when every rank has its own GPU, else torch.distributed callbacks
        from paper_2510_03932_b200 import Comm
        if world == 1 or dist.get_backend() == "nccl":
            uid = [Comm.nccl_unique_id() if rank == 0 else None]
            if world > 1:
                dist.broadcast_object_list(uid, src=0)
            comm = Comm.nccl(rank, world, local, uid[0])
        else:
            comm = Comm.host(local)
        ec = EvalContext(m, device=local, block=args.block, comm=comm)
        sh = ec.shard()
        a, b, specials = sh["idx_lo"], sh["idx_hi"], bool(sh["specials"])
        xd = torch.full((m.nvar,), float("nan"), dtype=torch.float64, device=dev)
        ld = torch.full((m.m_con,), float("nan"), dtype=torch.float64, device=dev)
        ec.scatter_x(x, xd, stream)  # owned slots + halo over the communicator
        ec.scatter_rows(lam, ld, stream)
    else:
        a, b = shard_of(st, 0, 1, args.N)
        specials = True
        ec = EvalContext(m, device=local, block=args.block)
        xd = torch.as_tensor(x, device=dev)
        ld = torch.as_tensor(lam, device=dev)
    c = torch.zeros(m.m_con, dtype=torch.float64, device=dev)
    assert ec.eval_jac_hess(xd, ld, c), "evaluation flagged a domain error on the synthetic point"
    if sharded:
        assert ec.status_all(stream)
    flush = torch.ones(L2_FLUSH_BYTES // 8, dtype=torch.float64, device=dev)
    sink = torch.zeros((), dtype=torch.float64, device=dev)

    clocks = ClockSampler(local)
    clocks.start()
    # warm-up, then exactly K timed steps bracketed by barrier + synchronize
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t_wall0 = time.perf_counter()
    times, launches = time_eval_config(ec, xd, ld, c, flush, sink, stream, args.steps, args.warmup,
                                       halo=sharded)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - t_wall0
    t_local = float(np.mean(times))
    ok = ec.status_all(stream) if sharded else ec.status(stream)
    dev_out = {"c": c.cpu().numpy(), "jac": ec.jac_val.cpu().numpy(), "hess": ec.hess_val.cpu().numpy()}

    # end to end through the public API with host buffers: pinned x, lambda in;
    # c, jac_val, hess_val segments this rank owns back to pinned host memory
    segs = output_segments(st, a, b, specials)
    xh = torch.as_tensor(x).pin_memory()
    lh = torch.as_tensor(lam).pin_memory()
    host = {"c": torch.empty(m.m_con, dtype=torch.float64).pin_memory(),
            "jac": torch.empty(ec.jac_nnz, dtype=torch.float64).pin_memory(),
            "hess": torch.empty(ec.hess_nnz, dtype=torch.float64).pin_memory()}
    devbuf = {"c": c, "jac": ec.jac_val, "hess": ec.hess_val}
    h2d = 8 * (m.nvar + m.m_con)
    d2h = 8 * sum(n for _, _, n in segs)
    e2e_steps = max(3, min(args.steps, 20))
    xh_np, lh_np = xh.numpy(), lh.numpy()

    def e2e_step():
        nonlocal h2d
        if sharded:  # this rank's slots and rows only, the halo over the communicator
            h2d = ec.scatter_x(xh_np, xd, stream) + ec.scatter_rows(lh_np, ld, stream)
        else:
            xd.copy_(xh, non_blocking=True)
            ld.copy_(lh, non_blocking=True)
        ec.launch_jac_hess(xd, ld, c, stream)
        for buf, s0, n in segs:
            host[buf][s0:s0 + n].copy_(devbuf[buf][s0:s0 + n], non_blocking=True)

    for _ in range(args.warmup):
        torch.sum(flush, dim=0, out=sink)
        e2e_step()
    stream.synchronize()
    e2e_t = []
    for _ in range(e2e_steps):
        torch.sum(flush, dim=0, out=sink)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        e2e_step()
        e.record(stream)
        e.synchronize()
        e2e_t.append(s.elapsed_time(e) * 1e-3)
    ok = ok and (ec.status_all(stream) if sharded else ec.status(stream))
    clk = clocks.stop()
    # a result read back must match the device copy
    for buf, s0, n in segs[:3]:
        assert torch.equal(host[buf][s0:s0 + n], devbuf[buf][s0:s0 + n].cpu())

    t_e2e_local = float(np.mean(e2e_t))
    tt = torch.tensor([t_local, t_e2e_local, 0.0 if ok else 1.0], dtype=torch.float64,
                      device=dev if dist.is_initialized() and dist.get_backend() == "nccl" else "cpu")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_max, t_e2e_max, bad = (float(v) for v in tt.cpu())

    nbytes = algorithmic_bytes(st, a, b, specials)
    peak, peak_kind = peaks()
    achieved = nbytes / t_local / 1e9

    out = None
    if rank == 0:
        value = t_max * 1e9 / N
        out = {
            "metric": "jac+hess eval ns/node", "value": value, "unit": "ns/node", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max * 1e3, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(args, world),
            "launch": {"block": ec_block(ec), "kernel": "ocg_cjh"},
            "ok": not bad,
            "nodes_per_s": N / t_max,
            "hbm_gbs": achieved,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind, "frac_of_nominal_8000": achieved / 8000.0,
                         "traffic": None, "kernel": "ocg_cjh (generated per model, NVRTC sm_100a)",
                         "algorithmic_bytes_per_launch": nbytes,
                         "bytes_per_node": nbytes / max(1, b - a)},
            "e2e": {"value": t_e2e_max * 1e9 / N, "unit": "ns/node", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "path": "C ABI ocg_eval_jac_hess (fused kernel) through the Python EvalContext mirror; pinned "
                            "host x, lambda in, c / jac_val / hess_val out, per rank"},
            "gpu_launches": launches,
            "clocks": clk,
            "wall_s_timed_region": wall,
        }
        prof = ROOT / "profiles" / "ncu_traffic.json"
        if prof.exists():
            try:
                d = json.loads(prof.read_text())
                key = f"{args.model}:{N}"
                if key in d:
                    out["roofline"]["traffic"] = d[key]["dram_bytes_per_launch"]
                    out["roofline"]["traffic_source"] = d[key].get("source")
            except Exception:
                pass
        if world == 1:
            # the headline e2e goes through the reference's own EvalContext API
            # (the drop-in); the C-ABI number above stays as e2e_c_abi
            dr = dropin_e2e_isolated(args.model, N, args.scheme, e2e_steps, args.warmup)
            if dr and "median_s" in dr:
                out["e2e_c_abi"] = out["e2e"]
                out["e2e"] = {"value": dr["median_s"] * 1e9 / N, "unit": "ns/node", "h2d_bytes_per_step": dr["h2d"],
                              "d2h_bytes_per_step": dr["d2h"], "steps": dr["steps"],
                              "path": "reference API: EvalContext::eval_constraints_jacobian + eval_hessian of the "
                                      "drop-in build (integration/_out/libref_accel.so) with host std::vectors; "
                                      "median of the timed steps (steady_clock around the two calls)"}
            elif dr:
                out["e2e"]["dropin"] = dr
        if world == 1 and not args.no_cpu_baseline:
            try:
                r = cpu_reference_eval(src, N, args.scheme, reps=5, serial=True, outputs=True)
                tp, ts = r["parallel"]["median_s"], r["serial"]["median_s"]
                out["cpu_baseline"] = {
                    "value": tp * 1e9 / N, "unit": "ns/node", "cores": r["parallel"]["workers"], "kind": "reference",
                    "serial_value": ts * 1e9 / N, "cpu_model": r["cpu_model"], "nproc": r["nproc"],
                    "sample": f"full workload (N={N}), median of {r['reps']} J+H evaluations after one warm-up, "
                              f"reference EvalContext (oracle/_ref/libref.so): value = Backend::parallel "
                              f"({r['parallel']['workers']} workers), serial_value = Backend::serial",
                    "parallel_times_s": r["parallel"]["times_s"], "serial_times_s": r["serial"]["times_s"]}
                out["parity"] = parity_of(args.model, dev_out, r["outputs"])
                out["max_rel_err"] = out["parity"]["max_rel_err"]
            except Exception as ex:  # the checker library is missing on this box
                out["cpu_baseline"] = {"value": None, "unit": "ns/node", "cores": 0, "kind": "reference",
                                       "sample": f"unavailable: {ex}"}
        if not args.no_secondary and world == 1:
            out["extra"] = secondary(dev, stream, flush, sink, peak, not args.no_cpu_baseline)
        if args.solve != "none" and world == 1:
            out["ipm_solve"] = ipm_solve_leg(args.solve, not args.no_cpu_baseline)
        if args.goddard_solve != "none" and world == 1:  # BASELINE config 2
            n, cap = (args.goddard_solve.split(":") + ["3"])[:2]
            out["goddard_solve"] = ipm_solve_leg(f"goddard:{n}", not args.no_cpu_baseline, int(cap))
        if args.goddard_parity != "none" and world == 1:  # BASELINE configs[0]: the reference's trajectory
            out["goddard_parity_solve"] = ipm_solve_leg(f"goddard:{args.goddard_parity}", not args.no_cpu_baseline,
                                                        order="reference", reps=1)
        if args.batch != "none" and world == 1:
            out["batch_solve"] = batch_early
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def ipm_solve_leg(spec: str, with_reference: bool, ref_max_iter: int = 0, order: str = "band", reps: int = 3) -> dict:
    """Full interior-point solve (BASELINE metric: "IPM solve time at N=1e5"):
    ocg_ipm_solve — the reference's filter line-search IPM with evaluations,
    KKT assembly, vector work and the time-partitioned band LDL^T all on the
    device — against the reference's own ipm::solve (oracle/_ref/libref.so,
    Backend::parallel on all host cores, its CPU LDL^T). Wall times of the
    solve call; the device time includes the one-time NVRTC compile of the
    model's kernels (reported separately as jit_s); device_s is the median
    wall of three further solves, each building its plans anew.
    ref_max_iter > 0 caps the reference's run (Goddard at N=1e5 needs ~N/2
    iterations, hours on the host: SURVEY.md D6); the two are then
    compared per iteration. order="reference" factors the KKT matrices in
    the reference's elimination order (ocg_ldl_create_ex OCG_LDL_REFERENCE),
    which reproduces the reference's iterate trajectory on Goddard too."""
    from paper_2510_03932_b200 import MODELS, Model, solve
    name, N = spec.split(":")
    N = int(N)
    m = Model(MODELS[name], N)
    os.environ["OCG_IPM_PLAN_CACHE"] = "0"  # first two solves build their plans in the call
    try:
        t0 = time.perf_counter()
        d = solve(m, kkt_order=order)  # cold: NVRTC compile + plans
        t_first = time.perf_counter() - t0
        t0 = time.perf_counter()
        solve(m, kkt_order=order)  # kernels compiled, plans built again
        t_plans = time.perf_counter() - t0
    finally:
        os.environ.pop("OCG_IPM_PLAN_CACHE", None)
    solve(m, kkt_order=order)  # builds the plans ocg_ipm_solve keeps for this model
    walls, d2 = [], None
    for _ in range(reps):  # plans reused; median of the further solves
        t0 = time.perf_counter()
        d2 = solve(m, kkt_order=order)
        walls.append(time.perf_counter() - t0)
    t_second = float(np.median(walls))
    out = {"model": name, "N": N, "status": d2["status_name"], "iterations": d2["iterations"],
           "objective": d2["objective"], "device_s": t_second, "device_s_all": walls,
           "device_s_incl_jit": t_first, "device_s_rebuilding_plans": t_plans,
           "timing": "device_s: wall of a solve reusing the model's cached plans (median); "
                     "device_s_rebuilding_plans: plans built in the call; device_s_incl_jit: first solve of the "
                     "process (NVRTC compile + plans)",
           "jit_s": max(0.0, t_first - t_second), "factorizations": d2["factorizations"],
           "time_factorize_s": d2["time_factorize"], "time_solve_s": d2["time_solve"],
           "time_derivatives_s": d2["time_derivatives"], "time_total_s": d2["time_total"],
           "time_setup_s": d2["time_setup"], "plan_s": {"eval": d2["time_plan_eval"], "kkt": d2["time_plan_kkt"],
                                                       "ldl": d2["time_plan_ldl"]},
           "factorization": ("time-partitioned band LDL^T (device)" if order == "band" else
                             "reference-order LDL^T (device; AMD-equivalent order + pivot_after_, 1x1 pivots)")}
    if with_reference:
        RefEval, RefModel = _ref_modules()
        cores = os.cpu_count() or 1
        rm = RefModel(MODELS[name], N)
        t0 = time.perf_counter()
        r = rm.solve(parallel=True, workers=cores, max_iter=ref_max_iter)
        out["reference"] = {"wall_s": time.perf_counter() - t0, "iterations": int(r["iterations"]),
                            "objective": r["objective"], "status": int(r["status"]), "cores": cores,
                            "time_factorize_s": r["time_factorize"], "time_derivatives_s": r["time_derivatives"]}
        if ref_max_iter > 0:
            out["reference"]["capped_at"] = ref_max_iter
            out["reference"]["s_per_iter"] = out["reference"]["wall_s"] / max(1, int(r["iterations"]))
            out["device_s_per_iter"] = d2["time_total"] / max(1, d2["iterations"])
            out["speedup_per_iter"] = out["reference"]["s_per_iter"] / out["device_s_per_iter"]
        else:
            out["iterations_match"] = int(r["iterations"]) == d2["iterations"]
            out["reference"]["factorizations"] = int(r["factorizations"])
            out["factorizations_match"] = int(r["factorizations"]) == d2["factorizations"]
            out["objective_rel_diff"] = abs(r["objective"] - d2["objective"]) / max(abs(r["objective"]), 1e-300)
            out["speedup_vs_reference"] = out["reference"]["wall_s"] / t_second
            out["speedup_vs_reference_rebuilding_plans"] = out["reference"]["wall_s"] / t_plans
    return out


def batch_solve_leg(spec: str, with_reference: bool, ref_sample: int = 64) -> dict:
    """BASELINE config 5: cart-pendulum instances b = 0..B-1 at N (terminal
    target p(2) = 1 + b/4096) solved by ocg_ipm_batch_solve — every instance
    the reference's IPM decisions, every device step one launch over all
    instances — against the reference ipm::solve run one instance per host
    core (Backend::serial each, all cores busy) on an evenly spaced sample.
    Instance data (their terminal-target rows) and the reference models are
    prepared outside both timed regions."""
    from paper_2510_03932_b200 import Model, solve_batch
    from paper_2510_03932_b200.models import cart_pendulum_instance
    B, N = (int(v) for v in spec.split(":"))
    base = Model(cart_pendulum_instance(0, 4096), N)
    insts = [Model(cart_pendulum_instance(b, 4096), N) for b in range(B)]
    arrs = [m.arrays() for m in insts]
    lcon = np.ascontiguousarray(np.stack([r["lcon"] for r in arrs]))
    ucon = np.ascontiguousarray(np.stack([r["ucon"] for r in arrs]))
    solve_batch(base, insts[:2])  # kernels into the compile cache
    # five whole-batch solves, the median wall reported (single walls vary
    # 0.85-2.5 s on some boxes with the solver's own time_total unchanged at
    # 0.82-0.84 s: host-side noise outside the solve, profiles/r2_batch_wall.txt)
    walls = []
    for _ in range(5):
        t0 = time.perf_counter()
        res = solve_batch(base, lcon=lcon, ucon=ucon)
        walls.append(time.perf_counter() - t0)
    wall = float(np.median(walls))
    out = {"model": "cart_pendulum", "N": N, "instances": B, "wall_s": wall, "wall_s_all": walls,
           "batch_time_total_s": res[0]["time_total"], "instances_per_s": B / wall,
           "optimal": sum(1 for r in res if r["status"] == 0),
           "mean_iterations": float(np.mean([r["iterations"] for r in res])),
           "launch_rounds": res[0]["rounds"], "launch_groups": res[0]["launch_groups"],
           "batch_setup_s": res[0]["time_setup"],
           "plan_s": res[0]["time_plan_eval"] + res[0]["time_plan_kkt"] + res[0]["time_plan_ldl"]}
    if with_reference:
        from concurrent.futures import ThreadPoolExecutor
        RefEval, RefModel = _ref_modules()
        cores = os.cpu_count() or 1
        sample = list(range(0, B, max(1, B // ref_sample)))[:ref_sample]
        models = {b: RefModel(cart_pendulum_instance(b, 4096), N) for b in sample}

        def one(b):
            r = models[b].solve(parallel=False)
            return b, int(r["status"]), int(r["iterations"]), r["objective"]

        t0 = time.perf_counter()
        with ThreadPoolExecutor(cores) as ex:  # one solve per core (the harness releases the GIL)
            refs = list(ex.map(one, sample))
        rwall = time.perf_counter() - t0
        match = sum(1 for b, st, it, obj in refs
                    if st == res[b]["status"] and it == res[b]["iterations"]
                    and abs(obj - res[b]["objective"]) <= 1e-8 * abs(obj))
        out["reference"] = {"sample": len(sample), "cores": cores, "wall_s": rwall,
                            "instances_per_s": len(sample) / rwall}
        out["parity"] = {"compared": len(refs), "status_iterations_objective_match": match}
        out["speedup_vs_reference"] = out["instances_per_s"] / out["reference"]["instances_per_s"]
    return out


def ec_block(ec) -> int:
    return getattr(ec, "block", 128)


def secondary(dev, stream, flush, sink, peak, with_reference: bool) -> list[dict]:
    """The other eval-only configs (BASELINE.json configs[2..3]) at N=1 GPU:
    Goddard and quadrotor N=1e6 (north_star's >= 60% of HBM roofline at
    N >= 1e6),
    quadrotor N=1e5, hang glider and shuttle N=1e5; each timed like the
    headline and checked against the reference EvalContext (max_rel_err)."""
    import torch

    from paper_2510_03932_b200 import MODELS, EvalContext, Model
    res = []
    # launch block per model: the faster of one- and four-warp blocks,
    # alternated twice on one box (profiles/r2_sec_block_ab.jsonl): one-warp
    # blocks for Goddard N=1e6 (96.4 vs 101.3 us), hang glider (36.9 vs 38.8)
    # and shuttle (65.4 vs 67.6); four-warp blocks for the quadrotor (35.9 vs
    # 36.8 us at N=1e5, 283.6 vs 304.8 at N=1e6)
    block_of = {"quadrotor": 128}
    for name, N in (("goddard", 1_000_000), ("quadrotor", 1_000_000), ("quadrotor", 100_000),
                    ("hang_glider", 100_000), ("shuttle", 100_000)):
        m = Model(MODELS[name], N)
        st = m.structure()
        ec = EvalContext(m, device=dev.index, block=block_of.get(name, 32))
        x, lam = m.synth_acceptance(20250808)
        xd, ld = torch.as_tensor(x, device=dev), torch.as_tensor(lam, device=dev)
        c = torch.zeros(m.m_con, dtype=torch.float64, device=dev)
        ok = ec.eval_jac_hess(xd, ld, c)
        ts, launches = time_eval_config(ec, xd, ld, c, flush, sink, stream, 20, 3)
        t = float(np.mean(ts))
        nb = algorithmic_bytes(st, *main_space(st), True)
        row = {"model": name, "N": N, "ok": ok and ec.status(stream), "ns_per_node": t * 1e9 / N,
               "us_per_step": t * 1e6, "gbs": nb / t / 1e9, "frac": nb / t / 1e9 / peak, "bytes_per_node": nb / N,
               "steps": 20, "warmup": 3, "gpu_launches": launches, "block": ec.block}
        if with_reference:
            got = {"c": c.cpu().numpy(), "jac": ec.jac_val.cpu().numpy(), "hess": ec.hess_val.cpu().numpy()}
            del ec
            r = cpu_reference_eval(MODELS[name], N, "trapezoid", reps=1, serial=False, outputs=True)
            row["parity"] = parity_of(name, got, r["outputs"])
            row["max_rel_err"] = row["parity"]["max_rel_err"]
            row["cpu_baseline_ns_per_node"] = r["parallel"]["median_s"] * 1e9 / N
        else:
            del ec
        res.append(row)
    return res


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--dropin-e2e-child":
        # the drop-in measurement in a process of its own (see dropin_e2e_isolated)
        src_name, N, scheme, steps, warmup = sys.argv[2].split(":")
        print(json.dumps(dropin_e2e(load_models().MODELS[src_name], int(N), scheme, int(steps), int(warmup))))
        return
    if len(sys.argv) > 2 and sys.argv[1] == "--batch-child":
        # the batched-solve leg in a process of its own (see batch_solve_isolated)
        B, N, ref = sys.argv[2].split(":")
        print(json.dumps(batch_solve_leg(f"{B}:{N}", ref == "1")))
        return
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
