"""Python host mirror of the reference evaluation interface.

`Model` is transcribe::StructuredNlp built from model text
(/root/reference/proj/src/transcribe/transcribe.cpp:180), `EvalContext` is
ipm::detail::EvalContext (/root/reference/proj/src/ipm/ipm_internal.hpp:40-95)
and `KktAssembler` is Reduction + KktAssembler (ipm_internal.hpp:102-146):
same member names, same argument meaning, same bool results. Values live in
device memory (torch CUDA tensors bound into the library); every computation
runs in libocgpu.so's sm_100a kernels — there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import json

import numpy as np
import torch

from . import _lib
from ._lib import LIB, check

SCHEMES = {"euler": 0, "trapezoid": 1}


def _ptr(t) -> int:
    return t.data_ptr()


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class Model:
    """Parsed + transcribed OCP (dsl::parse_ocp + transcribe::transcribe)."""

    def __init__(self, source: str, N: int, scheme: str = "trapezoid", boxes_as_bounds: bool = False):
        h = C.c_void_p()
        check(LIB.ocg_model_create(source.encode(), SCHEMES[scheme], int(N), int(boxes_as_bounds), C.byref(h)),
              "ocg_model_create")
        self._h = h
        self.source = source
        self.N = int(N)
        self.scheme = scheme
        self.nvar = LIB.ocg_model_nvar(h)
        self.m_con = LIB.ocg_model_mcon(h)

    def __del__(self):
        if getattr(self, "_h", None):
            LIB.ocg_model_destroy(self._h)
            self._h = None

    def arrays(self) -> dict:
        nv, m = self.nvar, self.m_con
        out = {k: np.empty(nv) for k in ("lvar", "uvar", "x_start", "clip_lo", "clip_hi")}
        out.update({k: np.empty(m) for k in ("lcon", "ucon")})
        check(LIB.ocg_model_arrays(self._h, *[out[k].ctypes.data for k in
                                               ("lvar", "uvar", "x_start", "clip_lo", "clip_hi", "lcon", "ucon")]))
        return out

    def structure(self) -> dict:
        return json.loads(_lib.take_string(LIB.ocg_model_structure_json(self._h)))

    def synth_acceptance(self, seed: int = 20250808) -> tuple[np.ndarray, np.ndarray]:
        x, lam = np.empty(self.nvar), np.empty(self.m_con)
        check(LIB.ocg_model_synth_acceptance(self._h, seed, x.ctypes.data, lam.ctypes.data))
        return x, lam

    def generated_source(self, fma: bool = False, block: int = 128, input_staging: int = 0) -> str:
        return _lib.take_string(LIB.ocg_debug_generated_source_ex(self._h, int(fma), block, int(input_staging)))


def synth_uniform(seed: int, lo: float, hi: float, n: int) -> np.ndarray:
    out = np.empty(n)
    check(LIB.ocg_synth_uniform(seed, lo, hi, n, out.ctypes.data))
    return out


def host_comm_callbacks(group=None):
    """The three ocg_comm_host_fns callbacks over torch.distributed (host
    buffers as ctypes pointers; return 0 on success). A zero count does not
    communicate (both sides of an exchange know the sizes)."""
    import torch.distributed as dist

    def to_global(r):
        return r if group is None else dist.get_global_rank(group, r)

    def allreduce_sum(ctx, buf, n):
        try:
            if n > 0:
                dist.all_reduce(torch.from_numpy(np.ctypeslib.as_array(buf, shape=(n,))), op=dist.ReduceOp.SUM,
                                group=group)
            return 0
        except Exception:  # noqa: BLE001 (reported to the library as a failed call)
            return 1

    def allreduce_max(ctx, buf, n):
        try:
            if n > 0:
                dist.all_reduce(torch.from_numpy(np.ctypeslib.as_array(buf, shape=(n,))), op=dist.ReduceOp.MAX,
                                group=group)
            return 0
        except Exception:  # noqa: BLE001
            return 1

    def sendrecv(ctx, sbuf, ns, to, rbuf, nr, frm):
        try:
            ops = []
            if ns > 0:
                ops.append(dist.P2POp(dist.isend, torch.from_numpy(np.ctypeslib.as_array(sbuf, shape=(ns,)).copy()),
                                      to_global(to), group))
            if nr > 0:
                ops.append(dist.P2POp(dist.irecv, torch.from_numpy(np.ctypeslib.as_array(rbuf, shape=(nr,))),
                                      to_global(frm), group))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            return 0
        except Exception:  # noqa: BLE001
            return 1

    return allreduce_sum, allreduce_max, sendrecv


class Comm:
    """Communicator between the ranks of one sharded evaluation (ocg_comm):
    Comm.nccl(...) — NCCL inside the library (ncclSend/Recv halos, ncclAllReduce),
    or Comm.host(...) — the library's collectives through torch.distributed
    (any backend, e.g. gloo) on host buffers."""

    def __init__(self, h, rank: int, world: int, keep=None):
        self._h, self.rank, self.world, self._keep = h, rank, world, keep

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        check(LIB.ocg_comm_nccl_unique_id(buf), "ocg_comm_nccl_unique_id")
        return bytes(buf)

    @classmethod
    def nccl(cls, rank: int, world: int, device: int, unique_id: bytes) -> "Comm":
        buf = (C.c_ubyte * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        check(LIB.ocg_comm_create_nccl(buf, rank, world, device, C.byref(h)), "ocg_comm_create_nccl")
        return cls(h, rank, world)

    @classmethod
    def host(cls, device: int, group=None) -> "Comm":
        """Collectives over torch.distributed (the default group unless given)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        ar_f, ar_i, sr = host_comm_callbacks(group)
        fns = _lib.CommHostFns(None, _lib.ALLREDUCE_F64(ar_f), _lib.ALLREDUCE_I32(ar_i), _lib.SENDRECV_F64(sr))
        h = C.c_void_p()
        check(LIB.ocg_comm_create_host(C.byref(fns), rank, world, device, C.byref(h)), "ocg_comm_create_host")
        return cls(h, rank, world, keep=fns)

    def __del__(self):
        if getattr(self, "_h", None):
            LIB.ocg_comm_destroy(self._h)
            self._h = None


def shard_plan(model: "Model", rank: int, world: int) -> dict:
    """Host-only: the node-range shard plan of `rank` (ocg_shard_plan_json)."""
    p = LIB.ocg_shard_plan_json(model._h, rank, world)
    if not p:
        raise _lib.OcgError(LIB.ocg_last_error().decode())
    return json.loads(_lib.take_string(p))


class EvalContext:
    """Device EvalContext: COO structure bit-identical to the reference's; values
    in `jac_val`, `hess_val`, `grad_val` (CUDA tensors); `obj_scale`/`row_scale`
    as in the reference. Methods return the reference's bool."""

    def __init__(self, model: Model, device: int = 0, fma: bool = False, block: int = 128,
                 idx_lo: int = 0, idx_hi: int = -1, specials: bool = True, min_blocks: int = 0,
                 split_kinds: int = -1, comm: Comm | None = None, input_staging: int = -1):
        """comm: a sharded context (ocg_eval_create_sharded) — this rank's
        node range, endpoint instances on rank 0; idx_lo/idx_hi/specials are
        then derived from the rank."""
        if not torch.cuda.is_available():
            raise RuntimeError("octgpu EvalContext needs a CUDA device (no CPU fallback)")
        self.model = model
        self.device = torch.device("cuda", device)
        self.block = block
        torch.cuda.set_device(self.device)
        opts = _lib.EvalOptions(device, int(fma), block, idx_lo, idx_hi, int(specials), int(min_blocks),
                                int(split_kinds), int(input_staging))
        h = C.c_void_p()
        self.comm = comm
        if comm is None:
            check(LIB.ocg_eval_create(model._h, C.byref(opts), C.byref(h)), "ocg_eval_create")
        else:
            check(LIB.ocg_eval_create_sharded(model._h, C.byref(opts), comm._h, C.byref(h)),
                  "ocg_eval_create_sharded")
        self._h = h
        j, hh, g = C.c_int64(), C.c_int64(), C.c_int64()
        check(LIB.ocg_eval_sizes(h, C.byref(j), C.byref(hh), C.byref(g)))
        self.jac_nnz, self.hess_nnz, self.grad_nnz = j.value, hh.value, g.value
        f64 = dict(dtype=torch.float64, device=self.device)
        self.jac_val = torch.zeros(max(self.jac_nnz, 1), **f64)[: self.jac_nnz]
        self.hess_val = torch.zeros(max(self.hess_nnz, 1), **f64)[: self.hess_nnz]
        self.grad_val = torch.zeros(max(self.grad_nnz, 1), **f64)[: self.grad_nnz]
        self._rs = torch.ones(max(model.m_con, 1), **f64)
        self.row_scale = self._rs[: model.m_con]
        for which, t in ((_lib.OCG_BUF_JAC, self.jac_val), (_lib.OCG_BUF_HESS, self.hess_val),
                         (_lib.OCG_BUF_GRAD, self.grad_val), (_lib.OCG_BUF_ROWSCALE, self._rs)):
            check(LIB.ocg_eval_bind_buffer(h, which, _ptr(t)), "bind")
        self._f = torch.zeros(1, **f64)
        self._scratch = torch.zeros(1, **f64)
        self.obj_scale = 1.0
        self.time_derivatives = 0.0
        self._structure = None

    def __del__(self):
        if getattr(self, "_h", None):
            LIB.ocg_eval_destroy(self._h)
            self._h = None

    # ---- node-range shards (comm=...) ----
    def shard(self) -> dict:
        o = np.zeros(6, dtype=np.int64)
        check(LIB.ocg_eval_shard(self._h, o.ctypes.data))
        return dict(zip(["idx_lo", "idx_hi", "specials", "rank", "world", "halo_doubles"], (int(v) for v in o)))

    def scatter_x(self, x_host: np.ndarray, x_dev: torch.Tensor, stream=None) -> int:
        """x_dev <- the slots this rank owns of x_host, then the halo from the
        owners; returns the host->device bytes."""
        x_host = np.ascontiguousarray(x_host, dtype=np.float64)
        nb = C.c_int64()
        check(LIB.ocg_eval_scatter_x(self._h, x_host.ctypes.data, _ptr(x_dev), C.byref(nb), _stream(stream)),
              "ocg_eval_scatter_x")
        return nb.value

    def scatter_rows(self, lam_host: np.ndarray, lam_dev: torch.Tensor, stream=None) -> int:
        lam_host = np.ascontiguousarray(lam_host, dtype=np.float64)
        nb = C.c_int64()
        check(LIB.ocg_eval_scatter_rows(self._h, lam_host.ctypes.data, _ptr(lam_dev), C.byref(nb), _stream(stream)),
              "ocg_eval_scatter_rows")
        return nb.value

    def halo_exchange(self, x_dev: torch.Tensor, stream=None) -> None:
        check(LIB.ocg_eval_halo_exchange(self._h, _ptr(x_dev), _stream(stream)), "ocg_eval_halo_exchange")

    def status_all(self, stream=None) -> bool:
        return check(LIB.ocg_eval_status_all(self._h, _stream(stream)), "ocg_eval_status_all") == _lib.OCG_OK

    def objective_all(self, x_dev: torch.Tensor, stream=None) -> tuple[bool, float]:
        f = C.c_double()
        rc = check(LIB.ocg_eval_objective_all(self._h, _ptr(x_dev), C.byref(f), _stream(stream)),
                   "ocg_eval_objective_all")
        return rc == _lib.OCG_OK, f.value

    # ---- structure queries (host int64, EvalContext's public members) ----
    def structure(self) -> dict:
        if self._structure is None:
            a = [np.empty(n, dtype=np.int64) for n in
                 (self.jac_nnz, self.jac_nnz, self.hess_nnz, self.hess_nnz, self.grad_nnz)]
            check(LIB.ocg_eval_structure(self._h, *[v.ctypes.data for v in a]))
            self._structure = dict(zip(["jac_row", "jac_col", "hess_row", "hess_col", "grad_col"], a))
        return self._structure

    @property
    def jac_row(self):
        return self.structure()["jac_row"]

    @property
    def jac_col(self):
        return self.structure()["jac_col"]

    @property
    def hess_row(self):
        return self.structure()["hess_row"]

    @property
    def hess_col(self):
        return self.structure()["hess_col"]

    @property
    def grad_col(self):
        return self.structure()["grad_col"]

    # ---- scaling ----
    def set_scaling(self, obj_scale: float, row_scale=None) -> None:
        rs = None if row_scale is None else np.ascontiguousarray(row_scale, dtype=np.float64)
        check(LIB.ocg_eval_set_scaling(self._h, float(obj_scale), None if rs is None else rs.ctypes.data))
        self.obj_scale = float(obj_scale)

    def compute_scaling(self, x0, enabled: bool = True) -> None:
        x0 = self._dev(x0)
        check(LIB.ocg_eval_compute_scaling(self._h, _ptr(x0), int(enabled), _stream()))
        o = C.c_double()
        check(LIB.ocg_eval_get_scaling(self._h, C.byref(o), None))
        self.obj_scale = o.value

    # ---- evaluation (reference bool semantics) ----
    def _dev(self, a) -> torch.Tensor:
        if isinstance(a, torch.Tensor):
            return a.to(device=self.device, dtype=torch.float64).contiguous()
        return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=self.device)

    def status(self, stream=None) -> bool:
        return check(LIB.ocg_eval_status(self._h, _stream(stream))) == _lib.OCG_OK

    def eval_constraints(self, x, c_scaled: torch.Tensor) -> bool:
        x = self._dev(x)
        check(LIB.ocg_eval_constraints(self._h, _ptr(x), _ptr(c_scaled), _stream()))
        return self.status()

    def eval_constraints_jacobian(self, x, c_scaled: torch.Tensor) -> bool:
        x = self._dev(x)
        check(LIB.ocg_eval_constraints_jacobian(self._h, _ptr(x), _ptr(c_scaled), _stream()))
        return self.status()

    def eval_objective(self, x) -> tuple[bool, float]:
        x = self._dev(x)
        check(LIB.ocg_eval_objective(self._h, _ptr(x), _ptr(self._f), _stream()))
        ok = self.status()
        return ok, float(self._f.item())

    def eval_gradient(self, x, grad_dense: torch.Tensor) -> bool:
        x = self._dev(x)
        check(LIB.ocg_eval_gradient(self._h, _ptr(x), _ptr(grad_dense), _stream()))
        return self.status()

    def eval_hessian(self, x, lambda_scaled) -> bool:
        x, lam = self._dev(x), self._dev(lambda_scaled)
        check(LIB.ocg_eval_hessian(self._h, _ptr(x), _ptr(lam), _stream()))
        return self.status()

    def eval_jac_hess(self, x, lambda_scaled, c_scaled: torch.Tensor) -> bool:
        """Fused eval_constraints_jacobian + eval_hessian at one point."""
        x, lam = self._dev(x), self._dev(lambda_scaled)
        check(LIB.ocg_eval_jac_hess(self._h, _ptr(x), _ptr(lam), _ptr(c_scaled), _stream()))
        return self.status()

    def max_abs_hessian(self) -> float:
        check(LIB.ocg_eval_max_abs_hessian(self._h, _ptr(self._scratch), _stream()))
        return float(self._scratch.item())

    # ---- raw async entry points (device pointers, caller's stream) ----
    def launch_constraints_jacobian(self, x: torch.Tensor, c: torch.Tensor, stream=None) -> None:
        check(LIB.ocg_eval_constraints_jacobian(self._h, _ptr(x), _ptr(c), _stream(stream)))

    def launch_hessian(self, x: torch.Tensor, lam: torch.Tensor, stream=None) -> None:
        check(LIB.ocg_eval_hessian(self._h, _ptr(x), _ptr(lam), _stream(stream)))

    def launch_jac_hess(self, x: torch.Tensor, lam: torch.Tensor, c: torch.Tensor, stream=None) -> None:
        check(LIB.ocg_eval_jac_hess(self._h, _ptr(x), _ptr(lam), _ptr(c), _stream(stream)))

    def launch_jac_hess_host(self, x_host: torch.Tensor, lam_host: torch.Tensor, c_host: torch.Tensor,
                             jac_host: torch.Tensor, hess_host: torch.Tensor, chunks: int = 1, stream=None) -> int:
        """ocg_eval_jac_hess_host: host (page-locked) buffers in and out,
        pipelined over `chunks` node ranges; returns the bytes copied. The
        host outputs are complete once `stream` is."""
        for t in (x_host, lam_host, c_host, jac_host, hess_host):
            assert t.device.type == "cpu" and t.dtype == torch.float64 and t.is_contiguous()
        assert jac_host.numel() >= self.jac_nnz and hess_host.numel() >= self.hess_nnz
        nb = C.c_int64(0)
        check(LIB.ocg_eval_jac_hess_host(self._h, _ptr(x_host), _ptr(lam_host), _ptr(c_host), _ptr(jac_host),
                                         _ptr(hess_host), int(chunks), C.byref(nb), _stream(stream)))
        return int(nb.value)

    def launch_constraints(self, x: torch.Tensor, c: torch.Tensor, stream=None) -> None:
        check(LIB.ocg_eval_constraints(self._h, _ptr(x), _ptr(c), _stream(stream)))

    def launch_objective(self, x: torch.Tensor, f: torch.Tensor, stream=None) -> None:
        check(LIB.ocg_eval_objective(self._h, _ptr(x), _ptr(f), _stream(stream)))

    def launch_gradient(self, x: torch.Tensor, g: torch.Tensor, stream=None) -> None:
        check(LIB.ocg_eval_gradient(self._h, _ptr(x), _ptr(g), _stream(stream)))

    # ---- node-range shards: the objective as chunk partials + combine ----
    @property
    def objective_chunks(self) -> int:
        return int(LIB.ocg_eval_objective_chunks(self._h))

    def launch_objective_partials(self, x: torch.Tensor, partials: torch.Tensor, stream=None) -> None:
        check(LIB.ocg_eval_objective_partials(self._h, _ptr(x), _ptr(partials), _stream(stream)))

    def launch_objective_combine(self, partials: torch.Tensor, f: torch.Tensor, stream=None) -> None:
        check(LIB.ocg_eval_objective_combine(self._h, _ptr(partials), _ptr(f), _stream(stream)))

    def eval_objective_sharded(self, x, owners: torch.Tensor, group=None) -> tuple[bool, float]:
        """eval_objective over node-range shards, one context per rank: each
        rank's chunk partials are kept where `owners` (objective_chunk_owners)
        says the chunk is its own and zeroed elsewhere, summed over the ranks
        (each chunk has one nonzero term, so the sum is exact) and combined in
        the reference's fixed order (backend.cpp:119-133) — bit-identical to an
        unsharded eval_objective. Without an initialised process group this is
        the single-rank case."""
        import torch.distributed as dist
        x = self._dev(x)
        n = max(1, self.objective_chunks)
        part = torch.empty(n, dtype=torch.float64, device=self.device)
        self.launch_objective_partials(x, part)
        part = torch.where(owners.to(self.device), part, torch.zeros((), dtype=torch.float64, device=self.device))
        if dist.is_available() and dist.is_initialized():
            dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)
        ok = self.status()  # this shard's domain errors, then every rank's
        if dist.is_available() and dist.is_initialized():
            t = torch.tensor([int(ok)], dtype=torch.int32, device=self.device)
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
            ok = bool(t.item())
        self.launch_objective_combine(part, self._f)
        ok = self.status() and ok
        return ok, float(self._f.item())

    @property
    def launch_count(self) -> int:
        return LIB.ocg_eval_launch_count(self._h)


def objective_chunk_owners(structure: dict, idx_lo: int, idx_hi: int, specials: bool) -> np.ndarray:
    """Which of the objective's 512-instance chunks (in EvalContext order:
    objective groups in model order, chunks in index order) a shard evaluating
    grid indices [idx_lo, idx_hi) — plus the endpoint instances when
    `specials` — computes in full. A chunk the shard only partly covers is an
    error: shard boundaries must fall on chunk boundaries of every objective
    group (multiples of 512 from the group's first index)."""
    owned = []
    for g in structure["obj_groups"]:
        lo, hi, ends = g["range"]
        count = 2 if ends else hi - lo
        for j in range((count + 511) // 512):
            if ends:
                owned.append(bool(specials))
                continue
            a, b = lo + 512 * j, min(hi, lo + 512 * (j + 1))
            inside = idx_lo <= a and b <= idx_hi
            if not inside and max(a, idx_lo) < min(b, idx_hi):
                raise ValueError(f"objective chunk [{a}, {b}) straddles the shard [{idx_lo}, {idx_hi})")
            owned.append(inside)
    return np.array(owned, dtype=bool)


class KktAssembler:
    """Reduction + KktAssembler on the device: K (lower CSC) with the reference's
    pattern; `assemble(sigma)` rewrites K.val from the EvalContext's buffers."""

    def __init__(self, model: Model, ec: EvalContext):
        h = C.c_void_p()
        check(LIB.ocg_kkt_create(model._h, ec._h, C.byref(h)), "ocg_kkt_create")
        self._h, self.ec, self.model = h, ec, model
        d = np.zeros(7, dtype=np.int64)
        check(LIB.ocg_kkt_dims(h, d.ctypes.data))
        self.n_free, self.n_slack, self.ntot, self.m, self.dim, self.nnz, contra = (int(v) for v in d)
        self.contradictory = bool(contra)

    def __del__(self):
        if getattr(self, "_h", None):
            LIB.ocg_kkt_destroy(self._h)
            self._h = None

    def pattern(self) -> tuple[np.ndarray, np.ndarray]:
        colp, rowi = np.empty(self.dim + 1, dtype=np.int64), np.empty(self.nnz, dtype=np.int64)
        check(LIB.ocg_kkt_pattern(self._h, colp.ctypes.data, rowi.ctypes.data))
        return colp, rowi

    def maps(self) -> dict:
        nv, m = self.model.nvar, self.model.m_con
        out = dict(prim_index=np.empty(nv, dtype=np.int64), slack_index=np.empty(m, dtype=np.int64),
                   dual_index=np.empty(m, dtype=np.int64), row_slot=np.empty(m, dtype=np.int64),
                   xlo=np.empty(nv), xhi=np.empty(nv))
        check(LIB.ocg_kkt_maps(self._h, *[out[k].ctypes.data for k in
                                           ("prim_index", "slack_index", "dual_index", "row_slot", "xlo", "xhi")]))
        return out

    def values(self) -> torch.Tensor:
        """K.val copied into a tensor."""
        ptr = LIB.ocg_kkt_values(self._h)
        out = torch.empty(self.nnz, dtype=torch.float64, device=self.ec.device)
        torch.cuda.current_stream().synchronize()
        _cuda_memcpy_d2d(_ptr(out), ptr, self.nnz * 8)
        return out

    def assemble(self, sigma) -> None:
        s = self.ec._dev(sigma)
        check(LIB.ocg_kkt_assemble(self._h, _ptr(s), _stream()))
        torch.cuda.current_stream().synchronize()

    def matvec(self, x) -> torch.Tensor:
        x = self.ec._dev(x)
        y = torch.empty(self.dim, dtype=torch.float64, device=self.ec.device)
        check(LIB.ocg_kkt_matvec(self._h, _ptr(x), _ptr(y), _stream()))
        return y

    def jt_lambda(self, lam) -> torch.Tensor:
        lam = self.ec._dev(lam)
        out = torch.empty(self.ntot, dtype=torch.float64, device=self.ec.device)
        check(LIB.ocg_kkt_jt_lambda(self._h, _ptr(lam), _ptr(out), _stream()))
        return out


def _cuda_memcpy_d2d(dst: int, src: int, nbytes: int) -> None:
    cudart = C.CDLL("libcudart.so.12")
    cudart.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
    rc = cudart.cudaMemcpy(dst, src, nbytes, 3)
    if rc != 0:
        raise RuntimeError(f"cudaMemcpy failed ({rc})")


class BandLdl:
    """Device LDL^T of the KKT matrix (include/octgpu.h ocg_ldl_*): the
    stand-in for sparse::factorize/solve and for cuDSS. order="band" (default)
    is the time-partitioned band; order="reference" keeps the reference's
    elimination order and 1x1 pivots (ocg_ldl_create_ex, OCG_LDL_REFERENCE)."""

    def __init__(self, kkt: KktAssembler, order: str = "band"):
        h = C.c_void_p()
        code = {"band": _lib.OCG_LDL_BAND, "reference": _lib.OCG_LDL_REFERENCE}[order]
        check(LIB.ocg_ldl_create_ex(kkt._h, code, C.byref(h)), "ocg_ldl_create_ex")
        self._h, self.kkt, self.order = h, kkt, order

    def factors(self) -> dict:
        """order="reference": the last factorization in the reference's LdlFactor
        layout: perm, Lp, Li, D (by pivot position), Lx."""
        dim, lnz = self.kkt.dim, int(LIB.ocg_ldl_factor_nnz(self._h))
        out = dict(perm=np.empty(dim, dtype=np.int64), Lp=np.empty(dim + 1, dtype=np.int64),
                   Li=np.empty(max(lnz, 1), dtype=np.int64), D=np.empty(dim), Lx=np.empty(max(lnz, 1)))
        check(LIB.ocg_ldl_factors(self._h, *(out[k].ctypes.data for k in ("perm", "Lp", "Li", "D", "Lx"))),
              "ocg_ldl_factors")
        out["Li"], out["Lx"] = out["Li"][:lnz], out["Lx"][:lnz]
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            LIB.ocg_ldl_destroy(self._h)
            self._h = None

    def info(self) -> dict:
        o = np.zeros(5, dtype=np.int64)
        check(LIB.ocg_ldl_info(self._h, o.ctypes.data))
        return dict(zip(["dim", "segments", "bandwidth", "border", "factorizations"], (int(v) for v in o)))

    def factor(self, delta_w: float = 0.0, delta_c: float = 0.0) -> tuple[int, int, int]:
        """Factor the assembled K.val; returns the inertia (positive, negative, zero)."""
        inertia = np.zeros(3, dtype=np.int64)
        check(LIB.ocg_ldl_factor(self._h, float(delta_w), float(delta_c), inertia.ctypes.data, _stream()))
        return tuple(int(v) for v in inertia)

    def factor_many(self, deltas) -> list[tuple[int, int, int]]:
        """order="reference": factor the candidate regularizations [(delta_w,
        delta_c), ...] concurrently (ocg_ldl_factor_many); candidate 0 is then
        current. Returns every candidate's inertia."""
        n = len(deltas)
        dw = (C.c_double * n)(*[float(d[0]) for d in deltas])
        dc = (C.c_double * n)(*[float(d[1]) for d in deltas])
        inertia = np.zeros(3 * n, dtype=np.int64)
        check(LIB.ocg_ldl_factor_many(self._h, n, dw, dc, inertia.ctypes.data_as(C.POINTER(C.c_int64)), _stream()),
              "ocg_ldl_factor_many")
        return [tuple(int(v) for v in inertia[3 * i:3 * i + 3]) for i in range(n)]

    def select(self, i: int) -> None:
        """Make candidate i of the last factor_many current."""
        check(LIB.ocg_ldl_select(self._h, int(i)), "ocg_ldl_select")

    def solve(self, rhs) -> torch.Tensor:
        r = self.kkt.ec._dev(rhs)
        x = torch.empty_like(r)
        check(LIB.ocg_ldl_solve(self._h, _ptr(r), _ptr(x), _stream()))
        return x


STATUS = {0: "optimal", 1: "max_iter", 2: "infeasible_detected", 3: "eval_error"}


def ref_symbolic(colp, rowi, n_free: int, ntot: int) -> dict:
    """Host-only reference-order symbolic analysis (ocg_ldl_ref_symbolic):
    KktAssembler::symbolic + sparse::analyze_ordered on a lower-CSC KKT
    pattern -> perm, parent (etree), Lp, Li. No device needed."""
    colp = np.ascontiguousarray(colp, dtype=np.int64)
    rowi = np.ascontiguousarray(rowi, dtype=np.int64)
    dim = len(colp) - 1
    lnz = np.zeros(1, dtype=np.int64)
    out = dict(perm=np.empty(dim, dtype=np.int64), parent=np.empty(dim, dtype=np.int64),
               Lp=np.empty(dim + 1, dtype=np.int64))
    check(LIB.ocg_ldl_ref_symbolic(dim, colp.ctypes.data, rowi.ctypes.data, int(n_free), int(ntot),
                                   out["perm"].ctypes.data, out["parent"].ctypes.data, out["Lp"].ctypes.data, None,
                                   lnz.ctypes.data), "ocg_ldl_ref_symbolic")
    Li = np.empty(max(int(lnz[0]), 1), dtype=np.int64)
    check(LIB.ocg_ldl_ref_symbolic(dim, colp.ctypes.data, rowi.ctypes.data, int(n_free), int(ntot), None, None, None,
                                   Li.ctypes.data, lnz.ctypes.data), "ocg_ldl_ref_symbolic")
    out["Li"] = Li[:int(lnz[0])]
    return out


def _kkt_order(options: dict) -> dict:
    """kkt_order may be given as "band" / "reference" (IpmOptions.kkt_order)."""
    v = options.get("kkt_order")
    if isinstance(v, str):
        options = dict(options)
        options["kkt_order"] = {"band": _lib.OCG_LDL_BAND, "reference": _lib.OCG_LDL_REFERENCE}[v]
    return options


def solve(model: Model, device: int = 0, return_x: bool = False, **options) -> dict:
    """ipm::solve on the device (include/octgpu.h ocg_ipm_solve): the
    reference's filter line-search IPM (proj/src/ipm/solver.cpp) with every
    vector, evaluation, the KKT assembly and the factorization on the B200.
    Options are IpmOptions fields (solver.hpp:31-56); reg_* flatten `reg`."""
    if not torch.cuda.is_available():
        raise RuntimeError("octgpu solve needs a CUDA device (no CPU fallback)")
    o = _lib.IpmOptions()
    LIB.ocg_ipm_default_options(C.byref(o))
    for k, v in _kkt_order(options).items():
        if not hasattr(o, k):
            raise TypeError(f"unknown IPM option {k!r}")
        setattr(o, k, type(getattr(o, k))(v))
    r = _lib.IpmResult()
    x = np.empty(model.nvar) if return_x else None
    check(LIB.ocg_ipm_solve(model._h, C.byref(o), int(device), C.byref(r),
                            None if x is None else x.ctypes.data), "ocg_ipm_solve")
    out = {name: getattr(r, name) for name, _ in r._fields_}
    out["status_name"] = STATUS.get(r.status, "unknown")
    if x is not None:
        out["x"] = x
    return out


def solve_batch(model: Model, instances: list[Model] | None = None, n: int | None = None, device: int = 0,
                return_x: bool = False, lvar=None, uvar=None, x_start=None, lcon=None, ucon=None,
                **options) -> list[dict]:
    """Batched device IPM (include/octgpu.h ocg_ipm_batch_solve): instances of
    `model`'s structure solved together, every device step one launch over
    all instances. The instances are given as Models of the same structure
    (e.g. models.cart_pendulum_instance(b)), or as [n][nvar] / [n][m_con]
    arrays of their bounds and start points (None = the model's own), or as
    `n` copies of `model`. Each result dict is what solve() returns for that
    instance; time_total is the batch's wall time."""
    if not torch.cuda.is_available():
        raise RuntimeError("octgpu solve_batch needs a CUDA device (no CPU fallback)")
    o = _lib.IpmOptions()
    LIB.ocg_ipm_default_options(C.byref(o))
    for k, v in _kkt_order(options).items():
        if not hasattr(o, k):
            raise TypeError(f"unknown IPM option {k!r}")
        setattr(o, k, type(getattr(o, k))(v))
    given = {"lvar": lvar, "uvar": uvar, "x_start": x_start, "lcon": lcon, "ucon": ucon}
    if instances is not None:
        base = model.arrays()
        arrs = [m.arrays() for m in instances]
        for key in given:
            stacked = np.stack([r[key] for r in arrs])
            # arrays every instance shares with the model are passed as NULL
            given[key] = None if np.array_equal(stacked, np.broadcast_to(base[key], stacked.shape)) else stacked
        nb = len(instances)
    else:
        sizes = [len(v) for v in given.values() if v is not None]
        nb = sizes[0] if sizes else int(n or 1)
    keep, ptrs = [], []
    for key, v in given.items():
        if v is None:
            ptrs.append(None)
            continue
        width = model.nvar if key in ("lvar", "uvar", "x_start") else model.m_con
        a = np.ascontiguousarray(v, dtype=np.float64)
        if a.shape != (nb, width):
            raise ValueError(f"{key}: expected shape {(nb, width)}, got {a.shape}")
        keep.append(a)
        ptrs.append(a.ctypes.data)
    res = (_lib.IpmResult * nb)()
    x = np.empty((nb, model.nvar)) if return_x else None
    check(LIB.ocg_ipm_batch_solve(model._h, C.byref(o), int(device), nb, *ptrs, res,
                                  None if x is None else x.ctypes.data), "ocg_ipm_batch_solve")
    out = []
    for b in range(nb):
        d = {name: getattr(res[b], name) for name, _ in res[b]._fields_}
        d["status_name"] = STATUS.get(res[b].status, "unknown")
        d["rounds"] = int(d.pop("time_derivatives"))
        d["launch_groups"] = int(d.pop("time_solve"))
        if x is not None:
            d["x"] = x[b]
        out.append(d)
    return out


class Solver:
    """Reusable device IPM context (ocg_ipm_ctx_*): plans built once for a
    model structure; solve() takes an instance's bounds / start point."""

    def __init__(self, model: Model, device: int = 0):
        if not torch.cuda.is_available():
            raise RuntimeError("octgpu Solver needs a CUDA device (no CPU fallback)")
        h = C.c_void_p()
        check(LIB.ocg_ipm_ctx_create(model._h, int(device), C.byref(h)), "ocg_ipm_ctx_create")
        self._h, self.model = h, model

    def __del__(self):
        if getattr(self, "_h", None):
            LIB.ocg_ipm_ctx_destroy(self._h)
            self._h = None

    def solve(self, instance: Model | None = None, return_x: bool = False, **options) -> dict:
        o = _lib.IpmOptions()
        LIB.ocg_ipm_default_options(C.byref(o))
        for k, v in _kkt_order(options).items():
            if not hasattr(o, k):
                raise TypeError(f"unknown IPM option {k!r}")
            setattr(o, k, type(getattr(o, k))(v))
        ptrs = [None] * 5
        keep = None
        if instance is not None:
            keep = instance.arrays()
            ptrs = [keep[k].ctypes.data for k in ("lvar", "uvar", "x_start", "lcon", "ucon")]
        r = _lib.IpmResult()
        x = np.empty(self.model.nvar) if return_x else None
        check(LIB.ocg_ipm_ctx_solve(self._h, C.byref(o), *ptrs, C.byref(r), None if x is None else x.ctypes.data),
              "ocg_ipm_ctx_solve")
        out = {name: getattr(r, name) for name, _ in r._fields_}
        out["status_name"] = STATUS.get(r.status, "unknown")
        if x is not None:
            out["x"] = x
        return out
