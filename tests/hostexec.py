"""Test-only: execute the GENERATED kernel source on the host CPU.

The generated CUDA is compiled as plain C++ (g++, glibc libm, no FMA
contraction) with a tiny shim for the CUDA built-ins, and every thread of the
launch is run in a loop. Because the generator mirrors the reference
evaluator's operation order, this host execution must agree with the
reference bit for bit — which separates code-generation errors (any
difference here) from device-math differences (libdevice vs glibc) seen on
the GPU. This is a checker for the code generator, never a product path.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import subprocess
from pathlib import Path

import numpy as np

CACHE = Path(__file__).resolve().parent / ".hostexec"

PRELUDE = r"""
#include <cmath>
#include <cstring>
#define __device__
#define __forceinline__ inline
#define __global__
#define __launch_bounds__(...)
#define OCG_HOST 1
#define __restrict__ __restrict
#define __shared__
#define __syncthreads() ((void)0)
#include <barrier>
#include <thread>
#include <vector>
static std::barrier<>* ocg_warp_barrier = nullptr;
#define __syncwarp() ocg_warp_barrier->arrive_and_wait()
#define __align__(n) __attribute__((aligned(n)))
alignas(16) double smem_all[1 << 18];  // one warp (OCG_BLOCK = 32) on the host: 32 std::threads
struct ocg_dim3 { unsigned x, y, z; };
static thread_local ocg_dim3 blockIdx, threadIdx, gridDim;
static inline double __fma_rn(double a, double b, double c) { return std::fma(a, b, c); }
template <class T> static inline T __ldg(const T* p) { return *p; }
// asynchronous copies complete immediately on the host
static inline void ocg_cp8(double* s, const double* g) { *s = *g; }
static inline void ocg_cp_wait() {}
static inline void ocg_cp_commit() {}
static inline void ocg_cp_wait1() {}
static inline int ocg_shift(const double* g, const double* s) { return (int)((((unsigned long long)g) ^ ((unsigned long long)s)) >> 3) & 1; }
static inline void ocg_fence_async() {}
static inline void ocg_bulk_store(double* g, const double* s, int n) { for (int i = 0; i < n; ++i) g[i] = s[i]; }
static inline void ocg_bulk_commit() {}
static inline void ocg_bulk_wait_read() {}
static inline void ocg_bulk_wait_all() {}
static inline void ocg_mbar_init(unsigned long long*) {}
static inline void ocg_mbar_arrive(unsigned long long*) {}
static inline void ocg_mbar_wait(unsigned long long*, unsigned) {}
static inline void ocg_bulk_load(double* p, const double* g, long long n, unsigned long long*) { for (long long i = 0; i < n; ++i) p[i] = g[i]; }
static inline double __longlong_as_double(long long v) { double d; std::memcpy(&d, &v, 8); return d; }
// the reference evaluates sin and cos separately with glibc
static inline void ocg_sincos(double a, double* s, double* c) { *s = std::sin(a); *c = std::cos(a); }
#define sincos ocg_sincos
using std::exp; using std::log; using std::tan; using std::sqrt; using std::pow; using std::fabs;
// the reference calls libm pow for every constant exponent
#define OCG_HOST_POW 1
static inline double ocg_pow_libm(double a, double b) { volatile double bb = b; return std::pow(a, bb); }
// volatile exponents: keep g++ from folding pow(a, 2.0) into a*a (glibc's pow
// is not always the correctly rounded square, e.g. a = 61.36577005930618)
static volatile double ocg_e2 = 2.0, ocg_em1 = -1.0, ocg_e05 = 0.5;
static inline double ocg_pow2(double a) { return std::pow(a, ocg_e2); }
static inline double ocg_powm1(double a) { return std::pow(a, ocg_em1); }
static inline double ocg_pow05(double a) { return std::pow(a, ocg_e05); }
#define pow ocg_pow_libm
"""

KERNELS = {
    "ocg_c": "const double* x, const double* rs, double* c, int* flag",
    "ocg_cjac": "const double* x, const double* rs, double* c, double* jac, int* flag",
    "ocg_hess": "const double* x, const double* lam, const double* rs, const double* objw, double* hess, int* flag",
    "ocg_objv": "const double* x, double* objv, int* flag",
    "ocg_grad": "const double* x, const double* objw, double* g, int* flag",
    "ocg_cjh": "const double* x, const double* lam, const double* rs, const double* objw, double* c, double* jac, "
               "double* hess, int* flag",
}


def _driver(name: str, params: str) -> str:
    args = ", ".join(p.split()[-1].lstrip("*") for p in params.split(","))
    return (f'extern "C" void run_{name}(const long long* pv, {params}, long long i0, long long n_main,'
            f" long long n_spec, long long total, int ys) {{\n"
            f"  OcgParams prm; for (size_t i = 0; i < sizeof prm.v / sizeof prm.v[0]; ++i) prm.v[i] = (OIX)pv[i];\n"
            f"  (void)total; (void)ys;\n"
            f"  // persistent warp-synchronous kernel: one block of one warp walks every\n"
            f"  // tile; lanes are real threads meeting at __syncwarp\n"
            f"  std::barrier<> bar(32); ocg_warp_barrier = &bar;\n"
            f"  std::vector<std::thread> lanes;\n"
            f"  for (unsigned l = 0; l < 32; ++l) lanes.emplace_back([&, l] {{\n"
            f"    gridDim.x = 1; blockIdx.x = 0; blockIdx.y = 0; blockIdx.z = 0; threadIdx.x = l;\n"
            f"    {name}(prm, {args}, i0, n_main, n_spec, OcgBatch{{}}); }});\n"
            f"  for (auto& th : lanes) th.join();\n}}\n")


def compile_generated(source: str) -> C.CDLL:
    CACHE.mkdir(exist_ok=True)
    body = PRELUDE + source + "".join(_driver(k, v) for k, v in KERNELS.items())
    key = hashlib.sha1(body.encode()).hexdigest()[:16]
    so = CACHE / f"gen_{key}.so"
    if not so.exists():
        cpp = CACHE / f"gen_{key}.cpp"
        cpp.write_text(body)
        subprocess.run(["g++", "-std=c++20", "-O1", "-pthread", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                        "-w", "-o", str(so), str(cpp)], check=True)
    return C.CDLL(str(so))


class HostKernels:
    """Runs the generated kernels for a Model on the CPU (layout from the model)."""

    def __init__(self, model, layout: dict, input_staging: int = 1):

        # satisfied by sequential execution
        src = model.generated_source(fma=False, block=32, input_staging=input_staging)
        meta = src[src.rindex("// ocg-meta ") + len("// ocg-meta "):]
        import json
        self.meta = json.loads(meta)
        self.params = np.array(self.meta.pop("params"), dtype=np.int64)
        self.lib = compile_generated(src)
        self.model = model
        self.lay = layout

    def _p(self, a):
        return C.c_void_p(a.ctypes.data)

    def _launch(self, name, *arrays):
        flag = np.zeros(1, dtype=np.int32)
        fn = getattr(self.lib, f"run_{name}")
        ys, tail, _smem = self.meta[name]
        n_main = self.lay["n_main"]
        total = max(n_main, tail)
        args = [self._p(self.params)] + [self._p(a) for a in arrays] + [self._p(flag), C.c_longlong(self.lay["idx_lo"]),
                                               C.c_longlong(n_main), C.c_longlong(tail),
                                               C.c_longlong(total), C.c_int(ys)]
        fn(*args)
        return flag[0] == 0

    def cjac(self, x, rs, jac_nnz):
        c, jac = np.zeros(self.model.m_con), np.zeros(max(jac_nnz, 1))
        ok = self._launch("ocg_cjac", x, rs, c, jac)
        return ok, c, jac[:jac_nnz]

    def hess(self, x, lam, rs, objw, hess_nnz):
        h = np.zeros(max(hess_nnz, 1))
        ok = self._launch("ocg_hess", x, lam, rs, objw, h)
        return ok, h[:hess_nnz]


def layout_from_structure(st: dict) -> dict:
    """Thread mapping and COO sizes of a model (mirrors plan make_layout)."""
    main = [g["range"] for g in st["con_groups"] + st["obj_groups"] if not g["range"][2]]
    lo = min(r[0] for r in main)
    hi = max(r[1] for r in main)

    def count(r):
        return (1 if r[0] == r[1] else 2) if r[2] else r[1] - r[0]

    n_spec = sum(count(g["range"]) for g in st["con_groups"] + st["obj_groups"] if g["range"][2])
    jac = sum(len(g["jac"]) * count(g["range"]) for g in st["con_groups"])
    hess = sum(len(g["hess"]) * count(g["range"]) for g in st["con_groups"] + st["obj_groups"])
    return {"idx_lo": lo, "n_main": hi - lo, "n_spec": n_spec, "jac_nnz": jac, "hess_nnz": hess}


def run_all(model, x, lam, obj_scale: float = 1.0, row_scale=None, input_staging: int = 1):
    """Host execution of every generated kernel: c, c+jac, hess, objective
    instance values and gradient COO, with the reference's unit (or given)
    scaling. input_staging: 0 LDGSTS once per tile, 1 double-buffered LDGSTS
    (the default on the device), 2 TMA bulk copies on mbarriers."""
    st = model.structure()
    lay = layout_from_structure(st)
    hk = HostKernels(model, lay, input_staging)
    rs = np.ones(model.m_con) if row_scale is None else np.ascontiguousarray(row_scale, dtype=np.float64)
    objw = np.array([obj_scale * g["weight"] for g in st["obj_groups"]] or [0.0])
    out = {}
    c = np.zeros(model.m_con)
    out["c_ok"] = hk._launch("ocg_c", x, rs, c)
    out["c"] = c
    out["cjac_ok"], out["c_cjac"], out["jac"] = hk.cjac(x, rs, lay["jac_nnz"])
    out["hess_ok"], out["hess"] = hk.hess(x, lam, rs, objw, lay["hess_nnz"])
    nobjv = sum((1 if g["range"][0] == g["range"][1] else 2) if g["range"][2] else g["range"][1] - g["range"][0]
                for g in st["obj_groups"])
    ov = np.zeros(max(nobjv, 1))
    out["objv_ok"] = hk._launch("ocg_objv", x, ov)
    out["objv"] = ov[:nobjv]
    ngrad = sum(len(g["jac"]) * ((1 if g["range"][0] == g["range"][1] else 2) if g["range"][2]
                                 else g["range"][1] - g["range"][0]) for g in st["obj_groups"])
    gv = np.zeros(max(ngrad, 1))
    out["grad_ok"] = hk._launch("ocg_grad", x, objw, gv)
    out["grad"] = gv[:ngrad]
    # the fused c + J + H kernel
    c2, j2, h2 = np.zeros(model.m_con), np.zeros(max(lay["jac_nnz"], 1)), np.zeros(max(lay["hess_nnz"], 1))
    out["cjh_ok"] = hk._launch("ocg_cjh", x, lam, rs, objw, c2, j2, h2)
    out["cjh_c"], out["cjh_jac"], out["cjh_hess"] = c2, j2[:lay["jac_nnz"]], h2[:lay["hess_nnz"]]
    return out
