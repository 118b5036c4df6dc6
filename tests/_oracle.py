"""Test-side access to the checkers under oracle/ (never imported by the product).

- RefModel/RefEval/RefKkt: ctypes over oracle/_ref/libref.so, the UNMODIFIED
  reference sources compiled by oracle/Makefile plus oracle/ref_harness.cpp.
- The same classes over integration/_out/libref_accel.so (lib="accel"): the
  reference's own front end, Solver and factorization linked with the drop-in
  device evaluation layer (integration/octrans_accel.cpp) in place of
  proj/src/ipm/eval.cpp — the product seen through the reference's API.
"""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF_SO = ROOT / "oracle" / "_ref" / "libref.so"
ACCEL_SO = ROOT / "integration" / "_out" / "libref_accel.so"
PORT_SO = ROOT / "oracle" / "_ref" / "liboracle.so"

_libs: dict = {}


def ref_lib(which: str = "ref") -> C.CDLL:
    if which not in _libs:
        path = REF_SO if which == "ref" else ACCEL_SO
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run __graft_entry__.build() (needs /root/reference)")
        L = C.CDLL(str(path))
        vp, i64, i32, dp = C.c_void_p, C.c_int64, C.c_int, C.c_void_p
        sig = {
            "ref_free": (None, [vp]),
            "ref_model_create": (vp, [C.c_char_p, i32, i64, i32, C.c_char_p, i32]),
            "ref_model_destroy": (None, [vp]),
            "ref_model_nlp_ptr": (vp, [vp]),
            "ref_model_nvar": (i64, [vp]),
            "ref_model_mcon": (i64, [vp]),
            "ref_model_arrays": (None, [vp] + [dp] * 7),
            "ref_model_json": (vp, [vp]),
            "ref_eval_create": (vp, [vp, i32, i32]),
            "ref_eval_destroy": (None, [vp]),
            "ref_eval_workers": (i32, [vp]),
            "ref_eval_sizes": (None, [vp, dp]),
            "ref_eval_structure": (None, [vp] + [dp] * 5),
            "ref_eval_set_scaling": (None, [vp, C.c_double, dp]),
            "ref_eval_compute_scaling": (None, [vp, dp, i32]),
            "ref_eval_get_scaling": (None, [vp, dp, dp]),
            "ref_eval_c": (i32, [vp, dp, dp]),
            "ref_eval_cjac": (i32, [vp, dp, dp, dp]),
            "ref_eval_obj": (i32, [vp, dp, dp]),
            "ref_eval_grad": (i32, [vp, dp, dp, dp]),
            "ref_eval_hess": (i32, [vp, dp, dp, dp]),
            "ref_eval_max_abs_hessian": (C.c_double, [vp]),
            "ref_eval_step_seconds": (C.c_double, [vp, dp, dp, i32, dp]),
            "ref_kkt_create": (vp, [vp]),
            "ref_kkt_destroy": (None, [vp]),
            "ref_kkt_dims": (None, [vp, dp]),
            "ref_kkt_pattern": (None, [vp, dp, dp]),
            "ref_kkt_maps": (None, [vp] + [dp] * 6),
            "ref_kkt_assemble": (None, [vp, dp, dp]),
            "ref_kkt_matvec": (None, [vp, dp, dp, dp]),
            "ref_kkt_symbolic_sizes": (None, [vp, dp]),
            "ref_kkt_symbolic": (None, [vp, dp, dp, dp]),
            "ref_kkt_factorize": (None, [vp, dp, C.c_double, C.c_double, dp, dp, dp, dp]),
            "ref_kkt_factor_solve": (i32, [vp, dp, C.c_double, C.c_double, dp, dp]),
            "ref_solve": (i32, [vp, i32, i32, i32, C.c_double, dp]),
            "ref_synth_acceptance": (None, [vp, C.c_uint32, dp, dp]),
            "ref_synth_uniform": (None, [C.c_uint32, C.c_double, C.c_double, i64, dp]),
        }
        if which == "accel":
            sig["octrans_accel_nlp_json"] = (vp, [vp])
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        _libs[which] = L
    return _libs[which]


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


class RefModel:
    def __init__(self, source: str, N: int, scheme: int = 1, boxes_as_bounds: bool = False, lib: str = "ref"):
        self.lib = lib
        self.L = L = ref_lib(lib)
        err = C.create_string_buffer(512)
        self.h = L.ref_model_create(source.encode(), scheme, N, int(boxes_as_bounds), err, 512)
        if not self.h:
            raise ValueError(err.value.decode())
        self.nvar = L.ref_model_nvar(self.h)
        self.m_con = L.ref_model_mcon(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_model_destroy(self.h)

    def structure(self) -> dict:
        L = self.L
        p = L.ref_model_json(self.h)
        s = C.cast(p, C.c_char_p).value.decode()
        L.ref_free(p)
        return json.loads(s)

    def arrays(self) -> dict:
        nv, m = self.nvar, self.m_con
        out = {k: np.empty(nv) for k in ("lvar", "uvar", "x_start", "clip_lo", "clip_hi")}
        out.update({k: np.empty(m) for k in ("lcon", "ucon")})
        self.L.ref_model_arrays(self.h, *[_p(out[k]) for k in
                                             ("lvar", "uvar", "x_start", "clip_lo", "clip_hi", "lcon", "ucon")])
        return out

    def synth_acceptance(self, seed: int = 20250808):
        x, lam = np.empty(self.nvar), np.empty(self.m_con)
        self.L.ref_synth_acceptance(self.h, seed, _p(x), _p(lam))
        return x, lam

    def solve(self, parallel: bool = True, workers: int = 0, max_iter: int = 0, tol: float = 0.0) -> dict:
        out = np.zeros(10)
        st = self.L.ref_solve(self.h, int(parallel), workers, max_iter, tol, _p(out))
        keys = ["objective", "iterations", "time_total", "time_derivatives", "time_factorize", "time_solve",
                "factorizations", "kkt_nnz", "factor_nnz", "theta"]
        d = dict(zip(keys, out.tolist()))
        d["status"] = st
        return d


def synth_uniform(seed: int, lo: float, hi: float, n: int) -> np.ndarray:
    out = np.empty(n)
    ref_lib().ref_synth_uniform(seed, lo, hi, n, _p(out))
    return out


class RefEval:
    def __init__(self, model: RefModel, parallel: bool = False, workers: int = 0):
        self.model = model
        self.L = model.L
        self.h = self.L.ref_eval_create(model.h, int(parallel), workers)
        s = np.zeros(3, dtype=np.int64)
        self.L.ref_eval_sizes(self.h, _p(s))
        self.jac_nnz, self.hess_nnz, self.grad_nnz = (int(v) for v in s)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_eval_destroy(self.h)

    def structure(self):
        a = [np.empty(n, dtype=np.int64) for n in
             (self.jac_nnz, self.jac_nnz, self.hess_nnz, self.hess_nnz, self.grad_nnz)]
        self.L.ref_eval_structure(self.h, *[_p(v) for v in a])
        return dict(zip(["jac_row", "jac_col", "hess_row", "hess_col", "grad_col"], a))

    def set_scaling(self, obj_scale: float, row_scale=None):
        rs = None if row_scale is None else np.ascontiguousarray(row_scale, dtype=np.float64)
        self.L.ref_eval_set_scaling(self.h, obj_scale, None if rs is None else _p(rs))

    def compute_scaling(self, x0, enabled=True):
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        self.L.ref_eval_compute_scaling(self.h, _p(x0), int(enabled))
        o = np.zeros(1)
        rs = np.empty(self.model.m_con)
        self.L.ref_eval_get_scaling(self.h, _p(o), _p(rs))
        return float(o[0]), rs

    def constraints(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        c = np.empty(self.model.m_con)
        ok = self.L.ref_eval_c(self.h, _p(x), _p(c))
        return bool(ok), c

    def constraints_jacobian(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        c, j = np.empty(self.model.m_con), np.empty(self.jac_nnz)
        ok = self.L.ref_eval_cjac(self.h, _p(x), _p(c), _p(j))
        return bool(ok), c, j

    def objective(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        f = np.zeros(1)
        ok = self.L.ref_eval_obj(self.h, _p(x), _p(f))
        return bool(ok), float(f[0])

    def gradient(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        g, gc = np.empty(self.model.nvar), np.empty(self.grad_nnz)
        ok = self.L.ref_eval_grad(self.h, _p(x), _p(g), _p(gc))
        return bool(ok), g, gc

    def hessian(self, x, lam):
        x = np.ascontiguousarray(x, dtype=np.float64)
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        h = np.empty(self.hess_nnz)
        ok = self.L.ref_eval_hess(self.h, _p(x), _p(lam), _p(h))
        return bool(ok), h

    def max_abs_hessian(self) -> float:
        return self.L.ref_eval_max_abs_hessian(self.h)

    def step_seconds(self, x, lam, reps: int = 1) -> tuple[float, bool]:
        ok = np.zeros(1, dtype=np.int32)
        t = self.L.ref_eval_step_seconds(self.h, _p(x), _p(lam), reps, _p(ok))
        return t, bool(ok[0])


class RefKkt:
    def __init__(self, ev: RefEval):
        self.ev = ev
        self.L = ev.L
        self.h = self.L.ref_kkt_create(ev.h)
        d = np.zeros(7, dtype=np.int64)
        self.L.ref_kkt_dims(self.h, _p(d))
        self.n_free, self.n_slack, self.ntot, self.m, self.dim, self.nnz, self.contradictory = (int(v) for v in d)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_kkt_destroy(self.h)

    def pattern(self):
        colp, rowi = np.empty(self.dim + 1, dtype=np.int64), np.empty(self.nnz, dtype=np.int64)
        self.L.ref_kkt_pattern(self.h, _p(colp), _p(rowi))
        return colp, rowi

    def maps(self):
        nv, m = self.ev.model.nvar, self.ev.model.m_con
        out = dict(prim_index=np.empty(nv, dtype=np.int64), slack_index=np.empty(m, dtype=np.int64),
                   dual_index=np.empty(m, dtype=np.int64), row_slot=np.empty(m, dtype=np.int64),
                   xlo=np.empty(nv), xhi=np.empty(nv))
        self.L.ref_kkt_maps(self.h, *[_p(out[k]) for k in
                                         ("prim_index", "slack_index", "dual_index", "row_slot", "xlo", "xhi")])
        return out

    def assemble(self, sigma):
        sigma = np.ascontiguousarray(sigma, dtype=np.float64)
        val = np.empty(self.nnz)
        self.L.ref_kkt_assemble(self.h, _p(sigma), _p(val))
        return val

    def matvec(self, val, x):
        val = np.ascontiguousarray(val, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.dim)
        self.L.ref_kkt_matvec(self.h, _p(val), _p(x), _p(y))
        return y

    def symbolic(self) -> dict:
        """KktAssembler::symbolic() (eval.cpp:442-471): perm, etree parent, Lp."""
        sz = np.zeros(2, dtype=np.int64)
        self.L.ref_kkt_symbolic_sizes(self.h, _p(sz))
        n, lnz = (int(v) for v in sz)
        out = dict(perm=np.empty(n, dtype=np.int64), parent=np.empty(n, dtype=np.int64),
                   Lp=np.empty(n + 1, dtype=np.int64))
        self.L.ref_kkt_symbolic(self.h, _p(out["perm"]), _p(out["parent"]), _p(out["Lp"]))
        out["lnz"] = lnz
        return out

    def factorize(self, val, delta_w: float = 0.0, delta_c: float = 0.0) -> dict:
        """sparse::factorize (ldl.cpp:139-213): D, Li, Lx in pivot order, inertia."""
        lnz = self.symbolic()["lnz"]
        val = np.ascontiguousarray(val, dtype=np.float64)
        D, Li, Lx = np.empty(self.dim), np.empty(lnz, dtype=np.int64), np.empty(lnz)
        inertia = np.zeros(3, dtype=np.int64)
        self.L.ref_kkt_factorize(self.h, _p(val), float(delta_w), float(delta_c), _p(D), _p(Li), _p(Lx),
                                 _p(inertia))
        return dict(D=D, Li=Li, Lx=Lx, inertia=tuple(int(v) for v in inertia))

    def factor_solve(self, val, b, delta_w: float = 0.0, delta_c: float = 0.0):
        """sparse::factorize + sparse::solve (ldl.cpp:222-247); None on zero pivots."""
        val = np.ascontiguousarray(val, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(self.dim)
        ok = self.L.ref_kkt_factor_solve(self.h, _p(val), float(delta_w), float(delta_c), _p(b), _p(x))
        return x if ok else None


# ---- the C restatement (oracle/port, liboracle.so) ---------------------------

class _OcGroup(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("op", C.c_void_p), ("a", C.c_void_p), ("b", C.c_void_p), ("c", C.c_void_p),
                ("n_inputs", C.c_int32), ("base", C.c_void_p), ("stride", C.c_void_p), ("out_dim", C.c_int32),
                ("roots", C.c_void_p), ("n_jac", C.c_int32), ("jac", C.c_void_p), ("n_hess", C.c_int32),
                ("hess", C.c_void_p), ("lo", C.c_int64), ("hi", C.c_int64), ("endpoints", C.c_int32),
                ("row_base", C.c_int64), ("weight", C.c_double)]


class _OcNlp(C.Structure):
    _fields_ = [("nvar", C.c_int64), ("m_con", C.c_int64), ("n_con", C.c_int32), ("n_obj", C.c_int32),
                ("con", C.c_void_p), ("obj", C.c_void_p)]


_port = None


def port_lib() -> C.CDLL:
    global _port
    if _port is None:
        if not PORT_SO.exists():
            raise FileNotFoundError(f"{PORT_SO} missing: run `make -C oracle port`")
        L = C.CDLL(str(PORT_SO))
        vp, dp = C.c_void_p, C.c_void_p
        L.oc_constraints_jacobian.restype = C.c_int
        L.oc_constraints_jacobian.argtypes = [vp, dp, dp, dp, dp]
        L.oc_hessian.restype = C.c_int
        L.oc_hessian.argtypes = [vp, dp, dp, dp, C.c_double, dp]
        L.oc_objective.restype = C.c_int
        L.oc_objective.argtypes = [vp, dp, C.c_double, dp]
        L.oc_gradient.restype = C.c_int
        L.oc_gradient.argtypes = [vp, dp, C.c_double, dp, dp]
        _port = L
    return _port


class PortEval:
    """The C restatement over a structure dump (ref_model_json /
    ocg_model_structure_json format): EvalContext's evaluation calls."""

    def __init__(self, st: dict):
        self.st = st
        self._keep = []
        self.nvar, self.m_con = int(st["nvar"]), int(st["m_con"])

        def arr(v, dt):
            a = np.ascontiguousarray(np.asarray(v, dtype=dt))
            if a.size == 0:
                a = np.zeros(1, dtype=dt)
            self._keep.append(a)
            return a.ctypes.data

        def group(g):
            nodes = g["nodes"]
            o = _OcGroup()
            o.n_nodes = len(nodes)
            o.op = arr([n[0] for n in nodes], np.int32)
            o.a = arr([n[1] for n in nodes], np.int32)
            o.b = arr([n[2] for n in nodes], np.int32)
            o.c = arr([n[3] for n in nodes], np.float64)
            o.n_inputs = len(g["inputs"])
            o.base = arr([i[0] for i in g["inputs"]], np.int64)
            o.stride = arr([i[1] for i in g["inputs"]], np.int64)
            o.out_dim = len(g["roots"])
            o.roots = arr(g["roots"], np.int32)
            o.n_jac = len(g["jac"])
            o.jac = arr([v for p in g["jac"] for v in p], np.int32)
            o.n_hess = len(g["hess"])
            o.hess = arr([v for p in g["hess"] for v in p], np.int32)
            o.lo, o.hi, o.endpoints = int(g["range"][0]), int(g["range"][1]), int(bool(g["range"][2]))
            o.row_base = int(g.get("row_base", 0))
            o.weight = float(g.get("weight", 1.0))
            return o

        cons = (_OcGroup * max(1, len(st["con_groups"])))(*[group(g) for g in st["con_groups"]])
        objs = (_OcGroup * max(1, len(st["obj_groups"])))(*[group(g) for g in st["obj_groups"]])
        self._keep += [cons, objs]
        self.nlp = _OcNlp(self.nvar, self.m_con, len(st["con_groups"]), len(st["obj_groups"]),
                          C.addressof(cons), C.addressof(objs))

        def count(g):
            lo, hi, ends = g["range"]
            return (1 if lo == hi else 2) if ends else hi - lo

        self.jac_nnz = sum(len(g["jac"]) * count(g) for g in st["con_groups"])
        self.hess_nnz = sum(len(g["hess"]) * count(g) for g in st["con_groups"] + st["obj_groups"])
        self.grad_nnz = sum(len(g["jac"]) * count(g) for g in st["obj_groups"])

    def _rs(self, row_scale):
        return np.ones(self.m_con) if row_scale is None else np.ascontiguousarray(row_scale, dtype=np.float64)

    def constraints_jacobian(self, x, row_scale=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        rs = self._rs(row_scale)
        c, j = np.zeros(max(self.m_con, 1)), np.zeros(max(self.jac_nnz, 1))
        ok = port_lib().oc_constraints_jacobian(C.byref(self.nlp), _p(x), _p(rs), _p(c), _p(j))
        return bool(ok), c[: self.m_con], j[: self.jac_nnz]

    def hessian(self, x, lam, row_scale=None, obj_scale=1.0):
        x = np.ascontiguousarray(x, dtype=np.float64)
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        rs = self._rs(row_scale)
        h = np.zeros(max(self.hess_nnz, 1))
        ok = port_lib().oc_hessian(C.byref(self.nlp), _p(x), _p(lam), _p(rs), float(obj_scale), _p(h))
        return bool(ok), h[: self.hess_nnz]

    def objective(self, x, obj_scale=1.0):
        x = np.ascontiguousarray(x, dtype=np.float64)
        f = np.zeros(1)
        ok = port_lib().oc_objective(C.byref(self.nlp), _p(x), float(obj_scale), _p(f))
        return bool(ok), float(f[0])

    def gradient(self, x, obj_scale=1.0):
        x = np.ascontiguousarray(x, dtype=np.float64)
        gc, gd = np.zeros(max(self.grad_nnz, 1)), np.zeros(self.nvar)
        ok = port_lib().oc_gradient(C.byref(self.nlp), _p(x), float(obj_scale), _p(gc), _p(gd))
        return bool(ok), gd, gc[: self.grad_nnz]
