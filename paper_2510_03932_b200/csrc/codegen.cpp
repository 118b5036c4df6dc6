// Graph -> straight-line fp64 CUDA for the per-node evaluation kernels.
//
// The generated code performs, operation for operation, what the reference's
// tape interpreter does (/root/reference/proj/src/kernel/evaluator.cpp):
//   forward values + local partials            evaluator.cpp:47-87
//   one reverse sweep per Jacobian row          evaluator.cpp:96-130
//   forward dual + reverse adjoint/adjoint-dual
//     sweep per Hessian direction j             evaluator.cpp:145-233
// but at code-generation time, so the interpreter, the zero-adjoint skips and
// every structurally-zero seed disappear. Only folds that are exact in IEEE
// arithmetic are applied (x*1, x*(-1), x+0, 0*x for finite x, constant
// arithmetic done in the same double precision on the host), so with FMA
// contraction off the device performs the same roundings in the same order as
// the x86 reference; only the libm/libdevice transcendentals differ (<=2 ulp).
//
// Thread mapping: blockIdx.x % slices selects a grid-indexed group, one thread per grid
// index of it, with shared-memory staging of the node slabs and of the COO
// outputs (see Generator::kernel). Endpoint-pair and single-index instances
// run on a short tail of threads. All grid-size-dependent integers are kernel
// parameters, so one compiled module serves every N of a model.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <functional>
#include <sstream>

#include "plan.hpp"

namespace ocg {

Layout make_layout(const Nlp& nlp) {
  Layout L;
  Index jac = 0, hess = 0, grad = 0, objv = 0;
  bool any_main = false;
  Index lo = 0, hi = 0;
  auto cover = [&](const Range& r) {
    if (r.endpoints) return;
    if (!any_main) {
      lo = r.lo;
      hi = r.hi;
      any_main = true;
    } else {
      lo = std::min(lo, r.lo);
      hi = std::max(hi, r.hi);
    }
  };
  for (size_t g = 0; g < nlp.cons.size(); ++g) {
    const Group& grp = nlp.cons[g];
    L.jac_off.push_back(jac);
    L.hess_off_con.push_back(hess);
    jac += static_cast<Index>(grp.pattern.jac.size()) * grp.range.count();
    hess += static_cast<Index>(grp.pattern.hess.size()) * grp.range.count();
    cover(grp.range);
    if (grp.range.endpoints)
      for (Index k = 0; k < grp.range.count(); ++k) L.specials.push_back({false, static_cast<int>(g), k});
  }
  for (size_t g = 0; g < nlp.objs.size(); ++g) {
    const Group& grp = nlp.objs[g];
    L.grad_off.push_back(grad);
    L.hess_off_obj.push_back(hess);
    L.objv_off.push_back(objv);
    grad += static_cast<Index>(grp.pattern.jac.size()) * grp.range.count();
    hess += static_cast<Index>(grp.pattern.hess.size()) * grp.range.count();
    objv += grp.range.count();
    cover(grp.range);
    if (grp.range.endpoints)
      for (Index k = 0; k < grp.range.count(); ++k) L.specials.push_back({true, static_cast<int>(g), k});
  }
  L.jac_nnz = jac;
  L.hess_nnz = hess;
  L.grad_nnz = grad;
  L.objv_n = objv;
  L.idx_lo = lo;
  L.idx_hi = hi;
  return L;
}

namespace {

struct V {
  bool is_c = true;
  double c = 0.0;
  int id = -1;
  bool zero() const { return is_c && c == 0.0; }
  bool one() const { return is_c && c == 1.0; }
  bool minus_one() const { return is_c && c == -1.0; }
};
V K(double c) { return V{true, c, -1}; }

std::string lit(double c) {
  if (std::isnan(c)) return "__longlong_as_double(0x7ff8000000000000LL)";
  if (std::isinf(c)) return c > 0 ? "__longlong_as_double(0x7ff0000000000000LL)"
                                   : "__longlong_as_double(0xfff0000000000000LL)";
  char buf[64];
  std::snprintf(buf, sizeof buf, "%a", c);
  return std::string("(") + buf + ")";
}

class Emitter {
 public:
  std::string out;
  int depth = 1;

  Emitter() { scopes_.emplace_back(); }

  void line(const std::string& s) {
    out.append(static_cast<size_t>(depth) * 2, ' ');
    out += s;
    out += '\n';
  }
  void open(const std::string& head) {
    line(head + " {");
    ++depth;
    scopes_.emplace_back();
  }
  void close(const std::string& tail = "") {
    --depth;
    line("}" + tail);
    scopes_.pop_back();
  }

  std::string s(V v) const { return v.is_c ? lit(v.c) : "t" + std::to_string(v.id); }

  // SSA temp for an expression, reused if the same key is visible in scope
  V emit(const std::string& key, const std::string& expr) {
    for (auto it = scopes_.rbegin(); it != scopes_.rend(); ++it) {
      auto f = it->find(key);
      if (f != it->end()) return f->second;
    }
    V v{false, 0.0, next_++};
    line("const double t" + std::to_string(v.id) + " = " + expr + ";");
    scopes_.back().emplace(key, v);
    return v;
  }
  // named temp without CSE (e.g. sincos outputs)
  V fresh() { return V{false, 0.0, next_++}; }
  void bind(const std::string& key, V v) { scopes_.back().emplace(key, v); }
  bool lookup(const std::string& key, V& v) const {
    for (auto it = scopes_.rbegin(); it != scopes_.rend(); ++it) {
      auto f = it->find(key);
      if (f != it->end()) {
        v = f->second;
        return true;
      }
    }
    return false;
  }

  V add(V a, V b) {
    if (a.zero()) return b;
    if (b.zero()) return a;
    if (a.is_c && b.is_c) return K(a.c + b.c);
    return emit("+" + s(a) + "," + s(b), s(a) + " + " + s(b));
  }
  V sub(V a, V b) {
    if (b.zero()) return a;
    if (a.zero()) return neg(b);
    if (a.is_c && b.is_c) return K(a.c - b.c);
    return emit("-" + s(a) + "," + s(b), s(a) + " - " + s(b));
  }
  V mul(V a, V b) {
    if (a.zero() || b.zero()) return K(0.0);
    if (a.one()) return b;
    if (b.one()) return a;
    if (a.minus_one()) return neg(b);
    if (b.minus_one()) return neg(a);
    if (a.is_c && b.is_c) return K(a.c * b.c);
    return emit("*" + s(a) + "," + s(b), s(a) + " * " + s(b));
  }
  V div(V a, V b) {
    if (b.one()) return a;
    if (a.is_c && b.is_c) return K(a.c / b.c);
    // division by a power of two is multiplication by its (exact) reciprocal:
    // both round the same real number once, so the result is bit-identical
    if (b.is_c && std::isfinite(b.c) && b.c != 0.0) {
      int e = 0;
      const double mant = std::frexp(b.c, &e);
      if ((mant == 0.5 || mant == -0.5) && e > -1020 && e < 1020) return mul(a, K(1.0 / b.c));
    }
    return emit("/" + s(a) + "," + s(b), s(a) + " / " + s(b));
  }
  V neg(V a) {
    if (a.is_c) return K(-a.c);
    return emit("n" + s(a), "-" + s(a));
  }
  V call(const char* fn, V a) {
    if (a.is_c) {  // only reachable for literal arguments; fold with host libm
      const std::string f(fn);
      if (f == "exp") return K(std::exp(a.c));
      if (f == "log") return K(std::log(a.c));
      if (f == "sqrt") return K(std::sqrt(a.c));
      if (f == "tan") return K(std::tan(a.c));
      if (f == "sin") return K(std::sin(a.c));
      if (f == "cos") return K(std::cos(a.c));
    }
    return emit(std::string(fn) + s(a), std::string(fn) + "(" + s(a) + ")");
  }
  // sin and cos of the same argument from one sincos call
  V trig(bool want_sin, V a) {
    if (a.is_c) return K(want_sin ? std::sin(a.c) : std::cos(a.c));
    V sv, cv;
    const std::string ks = "sin" + s(a), kc = "cos" + s(a);
    if (lookup(want_sin ? ks : kc, sv)) return sv;
    sv = fresh();
    cv = fresh();
    line("double " + s(sv) + ", " + s(cv) + ";");
    line("sincos(" + s(a) + ", &" + s(sv) + ", &" + s(cv) + ");");
    bind(ks, sv);
    bind(kc, cv);
    return want_sin ? sv : cv;
  }
  // pow with a constant exponent; exponents where glibc's pow is provably
  // identical to direct arithmetic are strength-reduced
  V powc(V a, double c) {
    if (c == 0.0) return K(1.0);
    if (c == 1.0) return a;
    if (a.is_c) return K(std::pow(a.c, c));
    // correctly rounded forms of pow for these exponents (device helpers in
    // the module prelude; the host checker maps them back to libm pow)
    if (c == 2.0) return call("ocg_pow2", a);
    if (c == -1.0) return call("ocg_powm1", a);
    if (c == 0.5) return call("ocg_pow05", a);
    return emit("pow" + s(a) + "," + lit(c), "pow(" + s(a) + ", " + lit(c) + ")");
  }

 private:
  int next_ = 0;
  std::vector<std::map<std::string, V>> scopes_;
};

enum class Mode { c, cjac, hess, cjh, objv, grad };

bool mode_values_only(Mode m) { return m == Mode::c || m == Mode::objv; }

// Per-node forward results of one group instance.
struct Fwd {
  std::vector<V> v, p1, p2;
};

struct Check {
  std::vector<int> owners;  // group ordinals (cons: g, objs: 1000+g) that need the value finite
  V v;
};

class Generator {
 public:
  Generator(const Nlp& nlp, const Layout& lay, const GenOptions& opt) : nlp_(nlp), lay_(lay), opt_(opt) {}

  Generated module() {
    Generated out;
    struct KSpec {
      Mode m;
      const char* name;
      const char* params;
    };
    const KSpec ks[] = {
        {Mode::c, "ocg_c",
         "const double* __restrict__ x, const double* __restrict__ rs, double* __restrict__ cout, "
         "int* __restrict__ flag"},
        {Mode::cjac, "ocg_cjac",
         "const double* __restrict__ x, const double* __restrict__ rs, double* __restrict__ cout, "
         "double* __restrict__ jac, int* __restrict__ flag"},
        {Mode::hess, "ocg_hess",
         "const double* __restrict__ x, const double* __restrict__ lam, const double* __restrict__ rs, "
         "const double* __restrict__ objw, double* __restrict__ hess, int* __restrict__ flag"},
        {Mode::cjh, "ocg_cjh",
         "const double* __restrict__ x, const double* __restrict__ lam, const double* __restrict__ rs, "
         "const double* __restrict__ objw, double* __restrict__ cout, double* __restrict__ jac, "
         "double* __restrict__ hess, int* __restrict__ flag"},
        {Mode::objv, "ocg_objv", "const double* __restrict__ x, double* __restrict__ objv, int* __restrict__ flag"},
        {Mode::grad, "ocg_grad",
         "const double* __restrict__ x, const double* __restrict__ objw, double* __restrict__ gout, "
         "int* __restrict__ flag"},
    };
    std::string kernels;
    for (const KSpec& k : ks) {
      int slices = 1, tail = 0;
      smem_out_ = 0;
      const std::string text = kernel(k.m, k.name, k.params, slices, tail);
      kernels += text;
      out.kernels[k.name] = text;
      out.slices[k.name] = slices;
      out.tail[k.name] = tail;
      out.smem[k.name] = static_cast<int>(smem_out_);
    }
    std::ostringstream os;
    os << "// generated by ocgpu codegen: do not edit\n";
    os << "#define OCG_BLOCK " << opt_.block << "\n";
    os << "// grid-size-dependent integers (offsets, ranges, slab bases) arrive by value:\n";
    for (size_t i = 0; i < pkeys_.size(); ++i) os << "//   prm.v[" << i << "] = " << pkeys_[i] << "\n";
    // index arithmetic in 32 bits when every array index of the model fits
    os << "typedef " << (opt_.idx32 ? "int" : "long long") << " OIX;\n";
    os << "struct OcgParams { OIX v[" << std::max<size_t>(1, pkeys_.size()) << "]; };\n";
    // batched launches over independent instances of one structure: block z
    // evaluates instance ids[z]; every array argument advances by its
    // per-instance stride (roles: x, lam, rs, objw, c, jac, hess, objv, grad,
    // flag). ids == NULL: one instance, no offsets.
    os << "struct OcgBatch { const int* ids; long long s[10]; };\n";
    os << "__device__ __forceinline__ bool fin(double v) { return fabs(v) <= 1.7976931348623157e308; }\n";
    os << "#ifndef OCG_HOST_POW\n";
    os << "__device__ __forceinline__ double ocg_pow2(double a) { return a * a; }\n";
    os << "__device__ __forceinline__ double ocg_powm1(double a) { return 1.0 / a; }\n";
    os << "__device__ __forceinline__ double ocg_pow05(double a) { return sqrt(a); }\n";
    os << "#endif\n";
    // 8-byte asynchronous global->shared copies (LDGSTS): a tile's loads are
    // all in flight together and need no registers
    os << "#ifndef OCG_HOST\n";
    os << "__device__ __forceinline__ void ocg_cp8(double* s, const double* g) {\n"
          "  asm volatile(\"cp.async.ca.shared.global [%0], [%1], 8;\\n\" :: \"r\"((unsigned)__cvta_generic_to_shared(s)), \"l\"(g) : \"memory\");\n}\n";
    os << "__device__ __forceinline__ void ocg_cp_wait() { asm volatile(\"cp.async.wait_all;\\n\" ::: \"memory\"); }\n";
    os << "__device__ __forceinline__ void ocg_cp_commit() { asm volatile(\"cp.async.commit_group;\\n\" ::: \"memory\"); }\n";
    os << "__device__ __forceinline__ void ocg_cp_wait1() { asm volatile(\"cp.async.wait_group 1;\\n\" ::: \"memory\"); }\n";
    // TMA bulk copy-out (cp.async.bulk shared::cta -> global, SASS UBLKCP):
    // an 8-byte head/tail goes by plain stores so the bulk part is 16-byte
    // aligned and a multiple of 16 bytes
    os << R"(__device__ __forceinline__ int ocg_shift(const double* g, const double* s) {
  return (int)((((unsigned long long)g) ^ ((unsigned long long)s)) >> 3) & 1;
}
__device__ __forceinline__ void ocg_fence_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void ocg_bulk_store(double* g, const double* s, int n) {
  if (n <= 0) return;
  if (((unsigned long long)g) & 15ull) { *g = *s; ++g; ++s; --n; }
  if (n & 1) { g[n - 1] = s[n - 1]; --n; }
  if (n > 0)
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
                 :: "l"(g), "r"((unsigned)__cvta_generic_to_shared(s)), "r"(n * 8) : "memory");
}
__device__ __forceinline__ void ocg_bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void ocg_bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void ocg_bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
// TMA bulk copy-in (cp.async.bulk global -> shared, SASS UBLKCP) completing
// on an mbarrier: one lane posts the byte count of every copy (expect_tx),
// issues the copies and arrives; the warp waits on the phase parity
__device__ __forceinline__ unsigned ocg_su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void ocg_mbar_init(unsigned long long* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(ocg_su32(b)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void ocg_mbar_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" :: "r"(ocg_su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void ocg_mbar_arrive(unsigned long long* b) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" :: "r"(ocg_su32(b)) : "memory");
}
__device__ __forceinline__ void ocg_mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile("{\n .reg .pred p;\n OCG_W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra OCG_W_%=;\n}\n"
               :: "r"(ocg_su32(b)), "r"(parity) : "memory");
}
// n > 0 doubles from g to shared memory at p, where p and g agree modulo 16
// bytes: the 16-byte chunks holding g[0..n) move whole (every chunk holds a
// valid element, so no page beyond the array is touched)
__device__ __forceinline__ void ocg_bulk_load(double* p, const double* g, long long n, unsigned long long* b) {
  const unsigned long long ga = ((unsigned long long)g) & ~15ull;
  const unsigned long long ge = (((unsigned long long)(g + n)) + 15ull) & ~15ull;
  const unsigned nb = (unsigned)(ge - ga);
  ocg_mbar_tx(b, nb);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               :: "r"(ocg_su32(p - ((((unsigned long long)g) & 15ull) >> 3))), "l"(ga), "r"(nb), "r"(ocg_su32(b))
               : "memory");
}
)";
    os << "#endif\n\n";
    out.prelude = os.str();
    std::string defs;
    for (const KSpec& k : ks) {
      const auto f = opt_.min_blocks.find(k.name);
      defs += "#define OCG_MINB_" + std::string(k.name) + " " +
              std::to_string(f == opt_.min_blocks.end() ? 1 : std::max(1, f->second)) + "\n";
    }
    os << kernels;
    out.source = defs + os.str();
    out.params.assign(pvals_.begin(), pvals_.end());
    if (out.params.empty()) out.params.push_back(0);
    return out;
  }

 private:
  const Nlp& nlp_;
  const Layout& lay_;
  const GenOptions& opt_;
  // staging hooks: shared-memory source of a strided input, and shared-memory
  // target of an output (kind 0 c, 1 jac, 2 grad, 3 objv, 4 hess; e = row /
  // entry); empty string = global memory
  std::function<std::string(const Addr&)> load_from_;
  std::function<std::string(int, Index)> store_to_;
  // predicate of a direct global store inside a tile (lanes outside the
  // group's range must not write); empty = unpredicated
  std::string store_pred_;
  // staged row inputs of the current group: what 0 = row_scale, 1 = lambda;
  // empty string = global memory
  std::function<std::string(int, int)> row_from_;
  Index smem_out_ = 0;  // dynamic shared memory (bytes) of the last kernel
  // finiteness accumulator the checks of the code being emitted go to
  std::string acc_ = "okacc";
  // a group's checks rotate over kAccChains independent accumulators
  // (acc_ + "_0" ...), so the finiteness DFMAs form short chains instead of
  // one serial chain through the whole group
  static constexpr int kAccChains = 4;
  int acc_chains_ = 1, acc_rr_ = 0;
  std::string acc_next() {
    if (acc_chains_ <= 1) return acc_;
    return acc_ + "_" + std::to_string(acc_rr_++ % acc_chains_);
  }
  // called before every shared-memory store of the current group with the
  // output kind: emits the waits/flushes of the staged copy-out
  std::function<void(int)> store_hook_;
  bool first_store_of_tile_ = false;
  std::map<std::string, std::string> slices_;  // range params -> slice variable suffix
  // range bounds as parameters keyed by value, so groups with equal ranges
  // share them (and their per-tile slice)
  std::string range_param(const Range& r, bool lo) {
    const Index v = lo ? r.lo : r.hi;
    return P(std::string(lo ? "range.lo=" : "range.hi=") + std::to_string(v), v);
  }
  std::string slice_of(const Range& r) { return slices_.at(range_param(r, true) + "," + range_param(r, false)); }

  // Grid-size-dependent integers live in a by-value parameter block keyed by
  // their meaning, so the generated source — and its cached cubin — depends
  // only on the model structure, not on N.
  std::vector<std::string> pkeys_;
  std::vector<Index> pvals_;
  std::map<std::string, size_t> pidx_;
  std::string P(const std::string& key, Index v) {
    auto it = pidx_.find(key);
    if (it == pidx_.end()) {
      it = pidx_.emplace(key, pkeys_.size()).first;
      pkeys_.push_back(key);
      pvals_.push_back(v);
    }
    return "prm.v[" + std::to_string(it->second) + "]";
  }
  std::string G(bool objective, int gi, const char* what, Index v) {
    return P(std::string(objective ? "obj" : "con") + std::to_string(gi) + "." + what, v);
  }

  // which parts of a group a mode evaluates
  struct Parts {
    bool values = false, jac = false, hess = false, partials = false, grad = false, objv = false;
    bool any() const { return values || jac || hess || grad || objv; }
  };
  Parts parts(Mode m, bool objective, const Group& g) const {
    Parts p;
    const bool has_h = !g.pattern.hess.empty();
    if (!objective) {
      p.values = m == Mode::c || m == Mode::cjac || m == Mode::cjh;
      p.jac = m == Mode::cjac || m == Mode::cjh;
      p.hess = (m == Mode::hess || m == Mode::cjh) && has_h;
    } else {
      p.hess = (m == Mode::hess || m == Mode::cjh) && has_h;
      p.grad = m == Mode::grad;
      p.objv = m == Mode::objv;
    }
    p.partials = p.jac || p.hess || p.grad;
    return p;
  }

  // Forward values whose finiteness must be tested explicitly. The reference
  // tests every node value (evaluator.cpp:79). A non-finite v always makes a
  // consumer u non-finite when v enters u through +, -, *, the numerator of /,
  // neg, sin, cos, tan, log, sqrt or pow with a positive exponent; so v needs
  // no test of its own when such a consumer is itself tested or covered.
  // (exp, a denominator and negative powers can absorb inf, e.g. 1/inf = 0.)
  static std::vector<char> value_checks(const Graph& gr) {
    const auto& nodes = gr.nodes();
    std::vector<char> covered(nodes.size(), 0), check(nodes.size(), 0);
    std::vector<std::vector<int>> feeds(nodes.size());  // v -> propagating consumers
    for (size_t u = 0; u < nodes.size(); ++u) {
      const Node& nd = nodes[u];
      switch (nd.op) {
        case Op::add:
        case Op::sub:
        case Op::mul:
          feeds[static_cast<size_t>(nd.a)].push_back(static_cast<int>(u));
          feeds[static_cast<size_t>(nd.b)].push_back(static_cast<int>(u));
          break;
        case Op::div:
        case Op::neg:
        case Op::sin:
        case Op::cos:
        case Op::tan:
        case Op::log:
        case Op::sqrt: feeds[static_cast<size_t>(nd.a)].push_back(static_cast<int>(u)); break;
        case Op::pow:
          if (nd.c > 0.0) feeds[static_cast<size_t>(nd.a)].push_back(static_cast<int>(u));
          break;
        default: break;
      }
    }
    for (size_t v = nodes.size(); v-- > 0;) {
      bool by_consumer = false;
      for (int u : feeds[v]) by_consumer |= covered[static_cast<size_t>(u)] != 0;
      covered[v] = 1;
      check[v] = by_consumer ? 0 : 1;
    }
    return check;
  }

  // slab holding an address: node offset and component; -1 if none
  long slab_of(const Addr& a, Index& node, Index& comp) const {
    for (size_t s = 0; s < nlp_.slabs.size(); ++s) {
      const Slab& sl = nlp_.slabs[s];
      if (a.base < sl.base || a.base >= sl.base + sl.dim * sl.nodes) continue;
      if (a.stride != 0 && a.stride != sl.dim) continue;
      node = (a.base - sl.base) / sl.dim;
      comp = (a.base - sl.base) % sl.dim;
      return static_cast<long>(s);
    }
    return -1;
  }

  // slot expression of an input at grid index `idx`
  std::string idx_slot(const Addr& a, const std::string& idx, bool /*clamp*/) {
    Index node = 0, comp = 0;
    const long s = slab_of(a, node, comp);
    if (s < 0) return a.stride == 0 ? i64(a.base) : "(" + i64(a.base) + " + " + i64(a.stride) + " * " + idx + ")";
    const Slab& sl = nlp_.slabs[static_cast<size_t>(s)];
    const std::string base = P("slab" + std::to_string(s) + ".base", sl.base);
    if (a.stride == 0) {
      // absolute slot: first node, last node (grid-dependent) or a free variable
      const bool last = sl.nodes > 1 && node == sl.nodes - 1;
      const std::string nd = last ? P("N", nlp_.N) : i64(node);
      return "(" + base + " + " + nd + " * " + i64(sl.dim) + " + " + i64(comp) + ")";
    }
    return "(" + base + " + " + i64(node * sl.dim + comp) + " + " + i64(sl.dim) + " * " + idx + ")";
  }
  // Nodes whose value does not depend on the grid index: constants, absolute
  // (stride-0) inputs such as a free final time, and operations on those.
  // Their forward values and partials are hoisted out of the tile loop.
  static std::vector<char> invariant_nodes(const Graph& gr) {
    const auto& nodes = gr.nodes();
    std::vector<char> inv(nodes.size(), 0);
    for (size_t k = 0; k < nodes.size(); ++k) {
      const Node& nd = nodes[k];
      if (nd.op == Op::cnst)
        inv[k] = 1;
      else if (nd.op == Op::input)
        inv[k] = gr.inputs()[static_cast<size_t>(nd.a)].stride == 0;
      else if (nd.op == Op::index)
        inv[k] = 0;
      else
        inv[k] = inv[static_cast<size_t>(nd.a)] && (nd.b < 0 || inv[static_cast<size_t>(nd.b)]);
    }
    return inv;
  }

  Fwd forward(Emitter& E, const Group& g, const std::string& idx, bool clamp, bool partials, int owner,
              std::vector<Check>& checks, const std::vector<char>* only = nullptr) {
    const auto& nodes = g.kernel.graph.nodes();
    const auto& ins = g.kernel.graph.inputs();
    Fwd f;
    const std::vector<char> need = value_checks(g.kernel.graph);
    f.v.resize(nodes.size());
    f.p1.assign(nodes.size(), K(0.0));
    f.p2.assign(nodes.size(), K(0.0));
    for (size_t k = 0; k < nodes.size(); ++k) {
      if (only && !(*only)[k]) continue;
      const Node& nd = nodes[k];
      V r, q1 = K(0.0), q2 = K(0.0);
      bool check_q = false;
      auto va = [&] { return f.v[static_cast<size_t>(nd.a)]; };
      auto vb = [&] { return f.v[static_cast<size_t>(nd.b)]; };
      switch (nd.op) {
        case Op::cnst: r = K(nd.c); break;
        case Op::input: {
          const Addr& ad = ins[static_cast<size_t>(nd.a)];
          const std::string staged = load_from_ ? load_from_(ad) : std::string();
          if (!staged.empty()) {
            r = E.emit("ld" + staged, staged);
          } else {
            const std::string slot = idx_slot(ad, idx, clamp);
            r = E.emit("ld" + slot, "__ldg(x + " + slot + ")");
          }
          break;
        }
        case Op::index: r = E.emit("ix" + idx + lit(nd.c), "(double)(" + idx + ") + " + lit(nd.c)); break;
        case Op::add:
          r = E.add(va(), vb());
          q1 = K(1.0);
          q2 = K(1.0);
          break;
        case Op::sub:
          r = E.sub(va(), vb());
          q1 = K(1.0);
          q2 = K(-1.0);
          break;
        case Op::mul:
          r = E.mul(va(), vb());
          q1 = vb();
          q2 = va();
          break;
        case Op::div:
          r = E.div(va(), vb());
          if (partials) {
            q1 = E.div(K(1.0), vb());
            q2 = E.div(E.neg(r), vb());
            check_q = true;
          }
          break;
        case Op::neg:
          r = E.neg(va());
          q1 = K(-1.0);
          break;
        case Op::sin:
          r = E.trig(true, va());
          if (partials) q1 = E.trig(false, va());
          break;
        case Op::cos:
          r = E.trig(false, va());
          if (partials) q1 = E.neg(E.trig(true, va()));
          break;
        case Op::tan:
          r = E.call("tan", va());
          if (partials) {
            q1 = E.add(K(1.0), E.mul(r, r));
            check_q = true;
          }
          break;
        case Op::exp:
          r = E.call("exp", va());
          q1 = r;
          break;
        case Op::log:
          r = E.call("log", va());
          if (partials) {
            q1 = E.div(K(1.0), va());
            check_q = true;
          }
          break;
        case Op::sqrt:
          r = E.call("sqrt", va());
          if (partials) {
            q1 = E.div(K(0.5), r);
            check_q = true;
          }
          break;
        case Op::pow:
          r = E.powc(va(), nd.c);
          if (partials) {
            q1 = E.mul(K(nd.c), E.powc(va(), nd.c - 1.0));
            check_q = true;
          }
          break;
      }
      f.v[k] = r;
      f.p1[k] = q1;
      f.p2[k] = q2;
      if (only) continue;  // hoisting pass: the group's own pass emits the checks
      if (!r.is_c && need[k]) checks.push_back({{owner}, r});
      if (partials && check_q) {
        if (!q1.is_c) checks.push_back({{owner}, q1});
        if (!q2.is_c) checks.push_back({{owner}, q2});
      }
    }
    return f;
  }

  // reverse sweep for one output row (evaluator.cpp:96-112); returns the dense
  // stencil gradient over input ordinals
  std::vector<V> reverse_row(Emitter& E, const Group& g, const Fwd& f, int root) {
    const auto& nodes = g.kernel.graph.nodes();
    std::vector<V> adj(nodes.size(), K(0.0));
    std::vector<V> grad(static_cast<size_t>(g.kernel.graph.n_inputs()), K(0.0));
    adj[static_cast<size_t>(root)] = K(1.0);
    for (size_t k = nodes.size(); k-- > 0;) {
      const V ak = adj[k];
      if (ak.zero()) continue;
      const Node& nd = nodes[k];
      if (nd.op == Op::input) {
        grad[static_cast<size_t>(nd.a)] = E.add(grad[static_cast<size_t>(nd.a)], ak);
      } else if (nd.a >= 0) {
        adj[static_cast<size_t>(nd.a)] = E.add(adj[static_cast<size_t>(nd.a)], E.mul(ak, f.p1[k]));
        if (nd.b >= 0) adj[static_cast<size_t>(nd.b)] = E.add(adj[static_cast<size_t>(nd.b)], E.mul(ak, f.p2[k]));
      }
    }
    return grad;
  }

  // Jacobian entries of all rows in pattern order (evaluator.cpp:114-130)
  std::vector<V> jacobian(Emitter& E, const Group& g, const Fwd& f) {
    std::vector<V> out(g.pattern.jac.size());
    size_t e = 0;
    for (int r = 0; r < g.out_dim(); ++r) {
      const size_t lo = e;
      while (e < g.pattern.jac.size() && g.pattern.jac[e].first == r) ++e;
      if (lo == e) continue;
      std::vector<V> grad = reverse_row(E, g, f, g.kernel.roots[static_cast<size_t>(r)]);
      for (size_t q = lo; q < e; ++q) out[q] = grad[static_cast<size_t>(g.pattern.jac[q].second)];
    }
    return out;
  }

  // weighted Hessian stencil (evaluator.cpp:145-233)
  std::vector<V> hessian(Emitter& E, const Group& g, const Fwd& f, const std::vector<V>& w) {
    const auto& nodes = g.kernel.graph.nodes();
    const int ni = g.kernel.graph.n_inputs();
    std::vector<int> input_node(static_cast<size_t>(ni), -1);
    for (size_t k = 0; k < nodes.size(); ++k)
      if (nodes[k].op == Op::input) input_node[static_cast<size_t>(nodes[k].a)] = static_cast<int>(k);
    std::vector<V> seeds(nodes.size(), K(0.0));
    for (int r = 0; r < g.out_dim(); ++r) {
      auto& s = seeds[static_cast<size_t>(g.kernel.roots[static_cast<size_t>(r)])];
      s = E.add(s, w[static_cast<size_t>(r)]);
    }
    std::vector<V> out(g.pattern.hess.size(), K(0.0));
    for (int j = 0; j < ni; ++j) {
      const int lo = g.pattern.dir_ptr[static_cast<size_t>(j)], hi = g.pattern.dir_ptr[static_cast<size_t>(j) + 1];
      if (lo == hi) continue;
      // forward dual sweep seeded on input j
      std::vector<V> dv(nodes.size(), K(0.0));
      for (size_t k = 0; k < nodes.size(); ++k) {
        const Node& nd = nodes[k];
        switch (nd.op) {
          case Op::cnst:
          case Op::index: dv[k] = K(0.0); break;
          case Op::input: dv[k] = K(nd.a == j ? 1.0 : 0.0); break;
          default: {
            const V t1 = E.mul(f.p1[k], dv[static_cast<size_t>(nd.a)]);
            const V t2 = nd.b >= 0 ? E.mul(f.p2[k], dv[static_cast<size_t>(nd.b)]) : K(0.0);
            dv[k] = E.add(t1, t2);
          }
        }
      }
      // reverse sweep of adjoints and adjoint duals
      std::vector<V> a = seeds, ad(nodes.size(), K(0.0));
      for (size_t k = nodes.size(); k-- > 0;) {
        const V ak = a[k], adk = ad[k];
        if (ak.zero() && adk.zero()) continue;
        const Node& nd = nodes[k];
        if (nd.a < 0 || nd.op == Op::input) continue;
        const size_t ia = static_cast<size_t>(nd.a);
        V p1d = K(0.0), p2d = K(0.0);
        switch (nd.op) {
          case Op::mul:
            p1d = dv[static_cast<size_t>(nd.b)];
            p2d = dv[ia];
            break;
          case Op::div:
            p1d = E.mul(E.mul(E.neg(f.p1[k]), f.p1[k]), dv[static_cast<size_t>(nd.b)]);
            p2d = E.neg(E.add(E.mul(dv[k], f.p1[k]), E.mul(f.v[k], p1d)));
            break;
          case Op::sin:
          case Op::cos: p1d = E.mul(E.neg(f.v[k]), dv[ia]); break;
          case Op::tan: p1d = E.mul(E.mul(K(2.0), f.v[k]), dv[k]); break;
          case Op::exp: p1d = dv[k]; break;
          case Op::log: p1d = E.mul(E.mul(E.neg(f.p1[k]), f.p1[k]), dv[ia]); break;
          case Op::sqrt:
            if (!dv[k].zero()) {
              const V num = E.mul(E.neg(f.p1[k]), dv[k]);
              const V vk = f.v[k];
              p1d = E.emit("sq" + E.s(num) + E.s(vk),
                           "(" + E.s(vk) + " != 0.0) ? " + E.s(num) + " / " + E.s(vk) + " : 0.0");
            }
            break;
          case Op::pow: {
            const V s = E.mul(K(nd.c * (nd.c - 1.0)), E.powc(f.v[ia], nd.c - 2.0));
            p1d = E.mul(s, dv[ia]);
            if (!ak.zero() && !s.is_c) {
              const std::string acc = acc_next();
              E.line(acc + " = (fin(" + E.s(s) + ") | (" + E.s(ak) + " == 0.0)) ? " + acc +
                     " : __longlong_as_double(0x7ff8000000000000LL);");
            }
            break;
          }
          default: break;
        }
        a[ia] = E.add(a[ia], E.mul(ak, f.p1[k]));
        ad[ia] = E.add(ad[ia], E.add(E.mul(adk, f.p1[k]), E.mul(ak, p1d)));
        if (nd.b >= 0) {
          const size_t ib = static_cast<size_t>(nd.b);
          a[ib] = E.add(a[ib], E.mul(ak, f.p2[k]));
          ad[ib] = E.add(ad[ib], E.add(E.mul(adk, f.p2[k]), E.mul(ak, p2d)));
        }
      }
      for (int e = lo; e < hi; ++e) {
        const int node = input_node[static_cast<size_t>(g.pattern.hess[static_cast<size_t>(e)].first)];
        out[static_cast<size_t>(e)] = node >= 0 ? ad[static_cast<size_t>(node)] : K(0.0);
      }
    }
    return out;
  }

  // finiteness: one DFMA per checked value (v*0 is NaN iff v is not finite)
  void check_inline(Emitter& E, V v) {
    if (!v.is_c) {
      const std::string a = acc_next();
      E.line(a + " = __fma_rn(" + E.s(v) + ", 0.0, " + a + ");");
    }
  }

  // integer literal of the kernel's index type (OIX: int when every array
  // index fits 32 bits, else long long)
  std::string i64(Index v) const { return std::to_string(v) + (opt_.idx32 ? "" : "LL"); }

  // AD + stores for one group instance; k is the range ordinal expression.
  void group_body(Emitter& E, Mode m, bool objective, int gi, const Fwd& f, const std::string& k) {
    const Group& g = objective ? nlp_.objs[static_cast<size_t>(gi)] : nlp_.cons[static_cast<size_t>(gi)];
    const size_t gs = static_cast<size_t>(gi);
    const Parts p = parts(m, objective, g);
    const int od = g.out_dim();
    const std::string rb = objective ? std::string() : G(false, gi, "row_base", g.row_base);
    auto row_expr = [&](int r) { return "(" + rb + " + " + k + " * " + i64(od) + " + " + i64(r) + ")"; };
    std::vector<V> rsv(static_cast<size_t>(od));
    auto rowscale = [&](int r) {
      V& v = rsv[static_cast<size_t>(r)];
      if (v.id < 0) {
        const std::string st = row_from_ ? row_from_(0, r) : std::string();
        v = st.empty() ? E.emit("rs" + row_expr(r), "__ldg(rs + " + row_expr(r) + ")") : E.emit("ld" + st, st);
      }
      return v;
    };
    // store target: staged shared memory when the kernel stages, else global
    auto lv = [&](int kind, Index e, const std::string& global) {
      const std::string s = store_to_ ? store_to_(kind, e) : std::string();
      if (!s.empty() && store_hook_) store_hook_(kind);
      if (s.empty() && !store_pred_.empty()) return "if (" + store_pred_ + ") " + global;
      return s.empty() ? global : s;
    };
    if (p.values) {
      for (int r = 0; r < od; ++r) {
        const V c = E.mul(rowscale(r), f.v[static_cast<size_t>(g.kernel.roots[static_cast<size_t>(r)])]);
        E.line(lv(0, r, "cout[" + row_expr(r) + "]") + " = " + E.s(c) + ";");
      }
    }
    if (p.jac) {
      const std::vector<V> jv = jacobian(E, g, f);
      const Index nnz = static_cast<Index>(g.pattern.jac.size());
      const std::string base = G(false, gi, "jac_off", lay_.jac_off[gs]) + " + " + k + " * " + i64(nnz);
      for (size_t e = 0; e < jv.size(); ++e) {
        check_inline(E, jv[e]);
        const V sv = E.mul(jv[e], rowscale(g.pattern.jac[e].first));
        E.line(lv(1, static_cast<Index>(e), "jac[" + base + " + " + i64(static_cast<Index>(e)) + "]") + " = " +
               E.s(sv) + ";");
      }
    }
    if (p.grad) {
      const std::vector<V> jv = jacobian(E, g, f);
      const V w = E.emit("ow" + std::to_string(gi), "__ldg(objw + " + std::to_string(gi) + ")");
      const Index nnz = static_cast<Index>(g.pattern.jac.size());
      const std::string base = G(true, gi, "grad_off", lay_.grad_off[gs]) + " + " + k + " * " + i64(nnz);
      for (size_t e = 0; e < jv.size(); ++e) {
        check_inline(E, jv[e]);
        E.line(lv(2, static_cast<Index>(e), "gout[" + base + " + " + i64(static_cast<Index>(e)) + "]") + " = " +
               E.s(E.mul(jv[e], w)) + ";");
      }
    }
    if (p.objv) {
      const V v = f.v[static_cast<size_t>(g.kernel.roots[0])];
      E.line(lv(3, 0, "objv[" + G(true, gi, "objv_off", lay_.objv_off[gs]) + " + " + k + "]") + " = " + E.s(v) + ";");
    }
    if (p.hess) {
      std::vector<V> w(static_cast<size_t>(od));
      if (objective) {
        w[0] = E.emit("ow" + std::to_string(gi), "__ldg(objw + " + std::to_string(gi) + ")");
      } else {
        for (int r = 0; r < od; ++r) {
          const std::string st = row_from_ ? row_from_(1, r) : std::string();
          const V lam = st.empty() ? E.emit("lam" + row_expr(r), "__ldg(lam + " + row_expr(r) + ")")
                                   : E.emit("ld" + st, st);
          w[static_cast<size_t>(r)] = E.mul(lam, rowscale(r));
        }
      }
      const std::vector<V> hv = hessian(E, g, f, w);
      const Index nnz = static_cast<Index>(g.pattern.hess.size());
      const std::string off = objective ? G(true, gi, "hess_off", lay_.hess_off_obj[gs])
                                        : G(false, gi, "hess_off", lay_.hess_off_con[gs]);
      const std::string base = off + " + " + k + " * " + i64(nnz);
      for (size_t e = 0; e < hv.size(); ++e) {
        check_inline(E, hv[e]);
        E.line(lv(4, static_cast<Index>(e), "hess[" + base + " + " + i64(static_cast<Index>(e)) + "]") + " = " +
               E.s(hv[e]) + ";");
      }
    }
  }

  // One kernel of a mode: persistent, warp-synchronous. Every warp walks its
  // own tiles of 32 grid indices (one per lane) with no block barriers:
  //   (1) the node slabs the grid-indexed groups read are staged into the
  //       warp's shared-memory rows with coalesced loads (x read once);
  //   (2) the groups run one after another — the whole warp executes one
  //       group's straight-line code at a time, keeping the instruction working
  //       set to one group — each lane writing its COO entries into its
  //       shared-memory row;
  //   (3) after __syncwarp the warp writes the group's contiguous COO segment
  //       (32 x nnz doubles) back with fully coalesced stores.
  // Endpoint and single-index (boundary/Mayer) instances run after the loop on
  // the last block, one thread each, straight to global memory.
  std::string kernel(Mode m, const char* name, const char* params, int& slices, int& tail) {
    struct Inst {
      bool objective;
      int gi;
      Index k;
    };
    std::vector<Inst> members, tails;
    auto scan = [&](bool objective, const std::vector<Group>& gs) {
      for (size_t g = 0; g < gs.size(); ++g) {
        if (!parts(m, objective, gs[g]).any()) continue;
        const Range& r = gs[g].range;
        if (!r.endpoints && gs[g].kind != Group::Kind::boundary)
          members.push_back({objective, static_cast<int>(g), 0});
        else
          for (Index k = 0; k < r.count(); ++k) tails.push_back({objective, static_cast<int>(g), k});
      }
    };
    scan(false, nlp_.cons);
    scan(true, nlp_.objs);
    constexpr Index W = 32;  // grid indices per warp tile
    // One-warp blocks (block == 32): every tile-level quantity derives from
    // blockIdx and the parameters, so it is warp-uniform by construction; the
    // tile's inputs then come in by TMA bulk copies on an mbarrier, double-
    // buffered (tile t+1's copies are in flight while tile t computes), and
    // one lane issues the tile's bulk copies out from uniform registers.
    if (opt_.tma && opt_.block != 32) throw std::runtime_error("TMA tiles need one-warp blocks (block = 32)");
    const bool tma = opt_.tma;
    const bool distinct = tma || opt_.distinct_regions;
    const bool split = !tma && opt_.split_kinds;
    const bool pf = !tma && opt_.prefetch && distinct && !split;
    // one-warp blocks: tile-level values are uniform, lane 0 issues the
    // tile's bulk copies out straight-line from uniform registers
    const bool uni = opt_.block == 32;
    const Index slack = tma ? 4 : 0;  // per staged input region: alignment lead, shift, tail

    // node slabs read by any member group: nodes [ib, ib + W + max_off)
    struct Use {
      Index soff = 0, max_off = 0;
    };
    std::map<size_t, Use> uses;
    for (const Inst& mb : members) {
      const Group& g = mb.objective ? nlp_.objs[static_cast<size_t>(mb.gi)] : nlp_.cons[static_cast<size_t>(mb.gi)];
      for (const Addr& a : g.kernel.graph.inputs()) {
        if (a.stride == 0) continue;
        Index node = 0, comp = 0;
        const long s = slab_of(a, node, comp);
        if (s >= 0) uses[static_cast<size_t>(s)].max_off = std::max(uses[static_cast<size_t>(s)].max_off, node);
      }
    }
    Index cur = 0;
    for (auto& [s, u] : uses) {
      u.soff = cur;
      cur += (W + u.max_off) * nlp_.slabs[s].dim + slack;
    }
    // row inputs of the member groups (row_scale, lambda): the warp's 32
    // instances read one contiguous segment of rows per group, staged with the
    // node slabs so that a tile waits for global memory once
    struct Rows {
      Index rs = -1, lam = -1;  // shared-memory offsets, -1 = not read
    };
    std::vector<Rows> rows(members.size());
    for (size_t q = 0; q < members.size(); ++q) {
      const Inst& mb = members[q];
      if (mb.objective) continue;
      const Group& g = nlp_.cons[static_cast<size_t>(mb.gi)];
      const Parts p = parts(m, false, g);
      const Index od = g.out_dim();
      if (p.values || p.jac || p.hess) {
        rows[q].rs = cur;
        cur += W * od + slack;
      }
      if (p.hess) {
        rows[q].lam = cur;
        cur += W * od + slack;
      }
    }
    // TMA tiles: two input buffers of IN doubles after the two mbarriers, the
    // output regions after them
    const Index IN = cur + (cur & 1);
    if (tma) cur = 0;
    if (pf) cur = 2 * IN;  // prefetch: two input buffers, then the outputs
    // output rows: one region reused by every group (warp-synchronous)
    struct Out {
      int kind;
      Index per_k, pitch, soff;
      std::string dst;
    };
    std::vector<std::vector<Out>> outs(members.size());
    Index region = 0;
    Index running = cur;  // distinct regions: every group's outputs at their own offsets
    for (size_t q = 0; q < members.size(); ++q) {
      const Inst& mb = members[q];
      const Group& g = mb.objective ? nlp_.objs[static_cast<size_t>(mb.gi)] : nlp_.cons[static_cast<size_t>(mb.gi)];
      const Parts p = parts(m, mb.objective, g);
      const size_t gi = static_cast<size_t>(mb.gi);
      Index off = distinct ? running : cur;
      auto add_out = [&](int kind, Index per_k, const std::string& dst) {
        // one value per instance: the lanes' stores to global memory are
        // already coalesced (8 bytes per lane, consecutive), so they go there
        // directly instead of through a staged region and a bulk copy
        if (per_k <= 1) return;
        const Index pitch = per_k;  // unpadded: the copy-out is one linear bulk copy
        outs[q].push_back({kind, per_k, pitch, off, dst});
        // + slack for the 16-byte alignment shift; split mode: every output
        // kind reuses one region, flushed before the next kind is staged
        if (split)
          region = std::max(region, W * pitch + 2);
        else
          off += W * pitch + 2;
      };
      if (p.values) add_out(0, g.out_dim(), "cout + " + G(false, mb.gi, "row_base", g.row_base));
      if (p.jac)
        add_out(1, static_cast<Index>(g.pattern.jac.size()), "jac + " + G(false, mb.gi, "jac_off", lay_.jac_off[gi]));
      if (p.grad)
        add_out(2, static_cast<Index>(g.pattern.jac.size()), "gout + " + G(true, mb.gi, "grad_off", lay_.grad_off[gi]));
      if (p.objv) add_out(3, 1, "objv + " + G(true, mb.gi, "objv_off", lay_.objv_off[gi]));
      if (p.hess)
        add_out(4, static_cast<Index>(g.pattern.hess.size()),
                "hess + " + (mb.objective ? G(true, mb.gi, "hess_off", lay_.hess_off_obj[gi])
                                          : G(false, mb.gi, "hess_off", lay_.hess_off_con[gi])));
      region = std::max(region, off - cur);
      running = off;
    }
    Index per_warp = cur + region;  // doubles of shared memory per warp
    per_warp += per_warp & 1;       // keep every warp's base 16-byte aligned (bulk copies)
    const Index out_base = tma ? 2 + 2 * IN : 0;
    if (tma) per_warp += out_base;

    Emitter E;
    E.depth = 0;
    // register budget: OCG_MINB_<name> resident blocks per SM, defined per
    // compilation (each kernel is compiled as its own module)
    E.line("extern \"C\" __global__ void __launch_bounds__(OCG_BLOCK, OCG_MINB_" + std::string(name) + ") " +
           std::string(name) +
           "(const OcgParams prm, " + params + ", long long i0_, long long n_main_, long long n_spec, const OcgBatch bt) {");
    E.depth = 1;
    {
      static const char* const roles[] = {"x", "lam", "rs", "objw", "cout", "jac", "hess", "objv", "gout", "flag"};
      std::set<std::string> names;  // last token of every parameter declaration
      std::stringstream ps(params);
      for (std::string decl; std::getline(ps, decl, ',');) names.insert(decl.substr(decl.find_last_of(" *") + 1));
      std::string adv;
      for (int r = 0; r < 10; ++r)
        if (names.count(roles[r])) adv += std::string(" ") + roles[r] + " += bz * bt.s[" + std::to_string(r) + "];";
      E.line("if (bt.ids) { const long long bz = bt.ids[blockIdx.z];" + adv + " }");
    }
    E.line("const OIX i0 = (OIX)i0_, n_main = (OIX)n_main_;");
    E.line("extern __shared__ __align__(16) double smem_all[];");
    E.line("const int lane = threadIdx.x & 31;");
    if (tma) {
      E.line("unsigned long long* const ocg_bar = reinterpret_cast<unsigned long long*>(smem_all);");
      E.line("double* const sin0 = smem_all + 2;");
      E.line("double* __restrict__ smem = smem_all + " + i64(out_base) + ";");
      E.line("if (lane == 0) { ocg_mbar_init(ocg_bar); ocg_mbar_init(ocg_bar + 1); }");
      E.line("__syncwarp();");
    } else {
      E.line(uni ? std::string("double* __restrict__ smem = smem_all;")
                 : "double* __restrict__ smem = smem_all + (threadIdx.x >> 5) * " + i64(per_warp) + ";");
    }
    E.line("double okacc = 0.0;  // fma(v, 0, acc) turns NaN iff some checked v is not finite");
    E.line("bool ok = true;");
    E.line("const OIX ntiles = (n_main + 31) / 32;");
    E.line("const OIX wpb = OCG_BLOCK / 32;");
    // loop invariants (free variables such as tf and everything computed from
    // them alone) once per thread, before the tile loop; emitted after the
    // first tile's copies are issued so that both loads are in flight together
    auto emit_invariants = [&]() {
      std::vector<Check> none;
      for (const Inst& mb : members) {
        const Group& g = mb.objective ? nlp_.objs[static_cast<size_t>(mb.gi)] : nlp_.cons[static_cast<size_t>(mb.gi)];
        const std::vector<char> inv = invariant_nodes(g.kernel.graph);
        forward(E, g, "idx", false, parts(m, mb.objective, g).partials, 0, none, &inv);
      }
    };
    // Distinct regions: the tile's outputs of every group leave together after
    // the last group, one bulk copy per lane; each lane's copy (destination
    // base, row length, shared-memory offset, range slice) is set up once here
    const bool batched = distinct && !split;
    struct Copy {
      std::string dst;
      Index S, soff;
      int R;
    };
    std::vector<Copy> copies;
    if (batched) {
      std::map<std::string, int> rid;
      // (TMA tiles: lane 0 issues every copy; no per-lane descriptors)
      for (size_t q = 0; q < members.size(); ++q) {
        const Inst& mb = members[q];
        const Group& g = mb.objective ? nlp_.objs[static_cast<size_t>(mb.gi)] : nlp_.cons[static_cast<size_t>(mb.gi)];
        const std::string key = range_param(g.range, true) + "," + range_param(g.range, false);
        if (!rid.count(key)) {
          const int r = static_cast<int>(rid.size());
          rid[key] = r;
        }
        for (const Out& o : outs[q]) copies.push_back({o.dst, o.per_k, o.soff, rid.at(key)});
      }
      for (size_t c0 = 0; c0 < copies.size() && !uni; c0 += 32) {
        const std::string C = std::to_string(c0 / 32);
        E.line("double* cd" + C + "_dst = nullptr; OIX cd" + C + "_S = 0, cd" + C + "_soff = 0; int cd" + C +
               "_R = -1;");
        for (size_t j = c0; j < std::min(copies.size(), c0 + 32); ++j)
          E.line("if (lane == " + std::to_string(j - c0) + ") { cd" + C + "_dst = " + copies[j].dst + "; cd" + C +
                 "_S = " + i64(copies[j].S) + "; cd" + C + "_soff = " + i64(copies[j].soff) + "; cd" + C +
                 "_R = " + std::to_string(copies[j].R) + "; }");
      }
    }
    // the tile's slice of every distinct group range (tile base `ib` in scope)
    auto emit_slices = [&]() {
      slices_.clear();
      for (const Inst& mb : members) {
        const Group& g = mb.objective ? nlp_.objs[static_cast<size_t>(mb.gi)] : nlp_.cons[static_cast<size_t>(mb.gi)];
        const std::string key = range_param(g.range, true) + "," + range_param(g.range, false);
        if (slices_.count(key)) continue;
        const std::string R = std::to_string(slices_.size());
        slices_[key] = R;
        const std::string lo = range_param(g.range, true), hi = range_param(g.range, false);
        E.line("const OIX kb" + R + " = ib - " + lo + ";");
        E.line("const OIX k0" + R + " = kb" + R + " > 0 ? kb" + R + " : 0;");
        E.line("OIX k1" + R + " = kb" + R + " + 32; if (k1" + R + " > " + hi + " - " + lo + ") k1" + R + " = " +
               hi + " - " + lo + "; if (k1" + R + " > i0 + n_main - " + lo + ") k1" + R + " = i0 + n_main - " + lo + ";");
        E.line("const int nk" + R + " = k1" + R + " > k0" + R + " ? (int)(k1" + R + " - k0" + R + ") : 0, r0" + R +
               " = (int)(k0" + R + " - kb" + R + ");");
      }
    };
    // global source and shared-memory region start of a staged row segment
    auto row_src = [&](size_t q, int what) {
      const Group& g = nlp_.cons[static_cast<size_t>(members[q].gi)];
      const std::string R = slice_of(g.range), od = i64(g.out_dim());
      return std::string(what == 0 ? "rs" : "lam") + " + " + G(false, members[q].gi, "row_base", g.row_base) + " + k0" + R +
             " * " + od;
    };
    auto row_pos = [&](size_t q, int what, const std::string& buf) {
      const Group& g = nlp_.cons[static_cast<size_t>(members[q].gi)];
      const std::string R = slice_of(g.range), od = i64(g.out_dim());
      return buf + " + " + i64((what == 0 ? rows[q].rs : rows[q].lam) + 1) + " + r0" + R + " * " + od;
    };
    auto slab_src = [&](size_t s) {
      const Slab& sl = nlp_.slabs[s];
      return "x + " + P("slab" + std::to_string(s) + ".base", sl.base) + " + ib * " + i64(sl.dim);
    };
    // LDGSTS staging of a tile's inputs into buffer `buf` (tile base `ib` and
    // its slices in scope); returns whether anything is staged
    auto emit_ldgsts = [&](const std::string& buf) {
      bool any = false;
      for (auto& [s, u] : uses) {
        const Slab& sl = nlp_.slabs[s];
        const Index n = (W + u.max_off) * sl.dim;
        const std::string sb = P("slab" + std::to_string(s) + ".base", sl.base);
        const std::string se = P("slab" + std::to_string(s) + ".end", sl.base + sl.nodes * sl.dim);
        // the copy count is bounded at generation time: straight-line
        // predicated copies, no loop control
        E.line("{ const OIX gb = " + sb + " + ib * " + i64(sl.dim) + "; OIX nv = " + se +
               " - gb; if (nv > " + i64(n) + ") nv = " + i64(n) + "; const int nvi = (int)nv;");
        for (Index j0 = 0; j0 < n; j0 += 32)
          E.line("  if (lane + " + std::to_string(j0) + " < nvi) ocg_cp8(" + buf + " + " + i64(u.soff + j0) +
                 " + lane, x + gb + " + std::to_string(j0) + " + lane);");
        E.line("}");
        any = true;
      }
      for (size_t q = 0; q < members.size(); ++q) {
        if (rows[q].rs < 0 && rows[q].lam < 0) continue;
        const Inst& mb = members[q];
        const Group& g = nlp_.cons[static_cast<size_t>(mb.gi)];
        const std::string rb = G(false, mb.gi, "row_base", g.row_base);
        const std::string od = i64(g.out_dim());
        const std::string R = slice_of(g.range);
        E.open("");
        E.line("const int nr = nk" + R + " * (int)" + od + ", so = r0" + R + " * (int)" + od + ";");
        E.line("const OIX g0 = " + rb + " + k0" + R + " * " + od + ";");
        const Index nmax = W * g.out_dim();
        for (Index j0 = 0; j0 < nmax; j0 += 32) {
          const std::string j = std::to_string(j0) + " + lane";
          if (rows[q].rs >= 0)
            E.line("if (" + j + " < nr) ocg_cp8(" + buf + " + " + i64(rows[q].rs) + " + so + " + j + ", rs + g0 + " + j +
                   ");");
          if (rows[q].lam >= 0)
            E.line("if (" + j + " < nr) ocg_cp8(" + buf + " + " + i64(rows[q].lam) + " + so + " + j + ", lam + g0 + " + j +
                   ");");
        }
        E.close();
        any = true;
      }
      return any;
    };
    if (pf) {
      // double-buffered LDGSTS staging: tile t+1's copies are issued before
      // tile t computes (one cp.async group per tile, wait_group 1)
      E.open("auto ocg_stage = [&](const OIX t, double* const sb)");
      E.line("const OIX ib = i0 + t * 32;");
      emit_slices();
      emit_ldgsts("sb");
      E.close(";");
      E.line("if (blockIdx.x * wpb + (threadIdx.x >> 5) < ntiles) ocg_stage(blockIdx.x * wpb + (threadIdx.x >> 5), smem);");
      E.line("ocg_cp_commit();");
      E.line("OIX it = 0;");
    }
    if (tma) {
      // tile t's inputs into buffer buf: one bulk copy per node slab and per
      // row segment, each landing where shared memory agrees with global
      // memory modulo 16 bytes (a shift of 0 or 1 double inside its region)
      E.open("auto ocg_stage = [&](const OIX t, const int buf)");
      E.line("double* const sb = sin0 + buf * " + i64(IN) + ";");
      E.line("unsigned long long* const bar = ocg_bar + buf;");
      E.line("const OIX ib = i0 + t * 32;");
      emit_slices();
      for (auto& [s, u] : uses) {
        const Slab& sl = nlp_.slabs[s];
        const Index n = (W + u.max_off) * sl.dim;
        const std::string se = P("slab" + std::to_string(s) + ".end", sl.base + sl.nodes * sl.dim);
        E.line("{ const double* const g = " + slab_src(s) + "; OIX nv = (OIX)((x + " + se + ") - g); if (nv > " + i64(n) +
               ") nv = " + i64(n) + "; double* const r = sb + " + i64(u.soff + 1) +
               "; if (nv > 0) ocg_bulk_load(r + ocg_shift(g, r), g, nv, bar); }");
      }
      for (size_t q = 0; q < members.size(); ++q) {
        if (rows[q].rs < 0 && rows[q].lam < 0) continue;
        const Group& g = nlp_.cons[static_cast<size_t>(members[q].gi)];
        const std::string R = slice_of(g.range), od = i64(g.out_dim());
        E.open("if (nk" + R + " > 0)");
        for (int what = 0; what < 2; ++what) {
          if ((what == 0 ? rows[q].rs : rows[q].lam) < 0) continue;
          E.line("{ const double* const g = " + row_src(q, what) + "; double* const r = " + row_pos(q, what, "sb") +
                 "; ocg_bulk_load(r + ocg_shift(g, r), g, (OIX)nk" + R + " * " + od + ", bar); }");
        }
        E.close();
      }
      E.line("ocg_mbar_arrive(bar);");
      E.close(";");
      E.line("if (lane == 0 && (OIX)blockIdx.x < ntiles) ocg_stage(blockIdx.x, 0);");
      E.line("OIX it = 0;");
      emit_invariants();
      E.open("for (OIX tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it)");
      E.line("const int buf = (int)(it & 1);");
      E.line("if (lane == 0 && tile + gridDim.x < ntiles) { ocg_fence_async(); ocg_stage(tile + gridDim.x, buf ^ 1); }");
    } else {
      emit_invariants();
      E.open(std::string(uni ? "for (OIX tile = blockIdx.x; tile < ntiles; tile += gridDim.x"
                             : "for (OIX tile = blockIdx.x * wpb + (threadIdx.x >> 5); tile < ntiles; tile += gridDim.x * wpb") +
             std::string(pf ? ", ++it)" : ")"));
    }
    E.line("const OIX ib = i0 + tile * 32;");
    E.line("const OIX idx = ib + lane;");
    E.line("const bool in = idx < i0 + n_main;");
    emit_slices();
    first_store_of_tile_ = true;
    if (tma) {
      // wait for this tile's copies; per-region pointers with this tile's shifts
      E.line("ocg_mbar_wait(ocg_bar + buf, (unsigned)((it >> 1) & 1));");
      E.line("__syncwarp();");
      E.line("double* const sin = sin0 + buf * " + i64(IN) + ";");
      for (auto& [s, u] : uses) {
        const std::string S = std::to_string(s);
        E.line("const double* const xs" + S + " = sin + " + i64(u.soff + 1) + " + ocg_shift(" + slab_src(s) + ", sin + " +
               i64(u.soff + 1) + ");");
      }
      for (size_t q = 0; q < members.size(); ++q) {
        for (int what = 0; what < 2; ++what) {
          if ((what == 0 ? rows[q].rs : rows[q].lam) < 0) continue;
          E.line("const double* const rq" + std::to_string(q) + "_" + std::to_string(what) + " = sin + " +
                 i64((what == 0 ? rows[q].rs : rows[q].lam) + 1) + " + ocg_shift(" + row_src(q, what) + ", " +
                 row_pos(q, what, "sin") + ");");
        }
      }
    }
    if (!tma && !pf) {
      // stage every global input of the tile with asynchronous copies, then wait once
      if (emit_ldgsts("smem")) {
        E.line("ocg_cp_wait();");
        E.line("__syncwarp();");
      }
    } else if (pf) {
      // this tile's copies (the only group in flight) and the previous tile's
      // bulk copy-out reads are complete before the next tile's copies go
      // out: ptxas tracks LDGSTS and the bulk copies on one scoreboard, so a
      // read wait later in the tile would also wait for the prefetch
      E.line("double* const sin = smem + (it & 1) * " + i64(IN) + ";");
      E.line("ocg_cp_wait();");
      E.line("ocg_bulk_wait_read();");
      E.line("__syncwarp();");
      E.line("if (tile + gridDim.x * wpb < ntiles) ocg_stage(tile + gridDim.x * wpb, smem + ((it + 1) & 1) * " + i64(IN) +
             ");");
      E.line("ocg_cp_commit();");
      first_store_of_tile_ = false;
    }
    load_from_ = [&](const Addr& a) -> std::string {
      if (a.stride == 0) return "";
      Index node = 0, comp = 0;
      const long s = slab_of(a, node, comp);
      if (s < 0) return "";
      const Index dim = nlp_.slabs[static_cast<size_t>(s)].dim;
      if (tma) return "xs" + std::to_string(s) + "[" + i64(node * dim + comp) + " + lane * " + i64(dim) + "]";
      return std::string(pf ? "sin[" : "smem[") + i64(uses.at(static_cast<size_t>(s)).soff + node * dim + comp) + " + lane * " + i64(dim) + "]";
    };
    for (size_t q = 0; q < members.size(); ++q) {
      const Inst& mb = members[q];
      const Group& g = mb.objective ? nlp_.objs[static_cast<size_t>(mb.gi)] : nlp_.cons[static_cast<size_t>(mb.gi)];
      const Parts p = parts(m, mb.objective, g);
      const std::string lo = range_param(g.range, true);
      const std::string hi = range_param(g.range, false);
      // this tile's slice of the group (shared by every group of the same
      // range): instances [k0, k1), lanes r0..r0+nk-1; each output kind's rows
      // start at a shift of 0 or 1 double so that the shared-memory source and
      // the global destination agree modulo 16 bytes
      const std::string qn = std::to_string(q);
      const std::string R = slice_of(g.range);
      if (!outs[q].empty()) {
        for (size_t oi = 0; oi < outs[q].size(); ++oi) {
          const Out& o = outs[q][oi];
          const std::string S = i64(o.per_k);
          E.line("const int sh" + qn + "_" + std::to_string(oi) + " = ocg_shift(" + o.dst + " + k0" + R + " * " + S +
                 ", smem + " + i64(o.soff) + " + r0" + R + " * " + S + ");");
        }
      }
      // staged copy-out of output kind oi of this group
      auto flush = [&, qn, R](size_t oi) {
        const Out& o = outs[q][oi];
        const std::string S = i64(o.per_k);
        E.line("ocg_fence_async(); __syncwarp();");
        E.line("if (lane == 0 && nk" + R + " > 0) { ocg_bulk_store(" + o.dst + " + k0" + R + " * " + S + ", smem + " +
               i64(o.soff) + " + sh" + qn + "_" + std::to_string(oi) + " + r0" + R + " * " + S + ", nk" + R +
               " * (int)" + S + "); ocg_bulk_commit(); }");
      };
      int cur_kind = -2;  // -2: nothing stored yet in this group
      store_hook_ = [&](int kind) {
        if (kind == cur_kind) return;
        if (split && cur_kind >= 0) {
          for (size_t oi = 0; oi < outs[q].size(); ++oi)
            if (outs[q][oi].kind == cur_kind) flush(oi);
        }
        // region free again? (distinct regions: only the tile's first store
        // waits, for the previous tile's copy-out)
        if ((cur_kind == -2 && (!distinct || first_store_of_tile_)) || split)
          E.line("ocg_bulk_wait_read(); __syncwarp();");
        first_store_of_tile_ = false;
        cur_kind = kind;
      };
      store_to_ = [&](int kind, Index e) -> std::string {
        for (size_t oi = 0; oi < outs[q].size(); ++oi) {
          const Out& o = outs[q][oi];
          if (o.kind == kind)
            return "smem[" + i64(o.soff + e) + " + sh" + qn + "_" + std::to_string(oi) + " + lane * " + i64(o.pitch) +
                   "]";
        }
        return "";
      };
      row_from_ = [&](int what, int r) -> std::string {
        const Index off = what == 0 ? rows[q].rs : rows[q].lam;
        if (off < 0) return "";
        if (tma)
          return "rq" + std::to_string(q) + "_" + std::to_string(what) + "[" + i64(r) + " + lane * " + i64(g.out_dim()) +
                 "]";
        return std::string(pf ? "sin[" : "smem[") + i64(off + r) + " + lane * " + i64(g.out_dim()) + "]";
      };
      // Every lane evaluates every member group in one scope (so common
      // subexpressions are shared across groups) and stores its rows to
      // shared memory unconditionally; lanes outside the group's range write
      // rows the copy-out skips, and only the finiteness verdict is predicated.
      const std::string qs = std::to_string(q);
      E.line("// ---- " + std::string(mb.objective ? "objective" : "constraint") + " group " +
             std::to_string(mb.gi) + ": " + g.label);
      E.line("const bool p" + qs + " = in && idx >= " + lo + " && idx < " + hi + ";");
      store_pred_ = "p" + qs;
      {
        std::string decl = "double okg" + qs + "_0 = 0.0";
        for (int a = 1; a < kAccChains; ++a) decl += ", okg" + qs + "_" + std::to_string(a) + " = 0.0";
        E.line(decl + ";");
      }
      acc_ = "okg" + qs;
      acc_chains_ = kAccChains;
      acc_rr_ = 0;
      std::vector<Check> sc;
      Fwd f = forward(E, g, "idx", false, p.partials, 0, sc);
      for (const auto& c : sc) check_inline(E, c.v);
      group_body(E, m, mb.objective, mb.gi, f, "(idx - " + lo + ")");
      {
        std::string sum = "okg" + qs + "_0";
        for (int a = 1; a < kAccChains; ++a) sum = "(" + sum + " + okg" + qs + "_" + std::to_string(a) + ")";
        E.line("if (p" + qs + ") okacc += " + sum + ";");
      }
      acc_ = "okacc";
      acc_chains_ = 1;
      store_to_ = nullptr;
      store_pred_.clear();
      row_from_ = nullptr;
      store_hook_ = nullptr;
      if (outs[q].empty() || batched) continue;
      // rows are unpadded (pitch == per_k): the tile's segment of each output
      // is contiguous in shared memory and in the COO array -> one bulk copy
      if (split) {
        for (size_t oi = 0; oi < outs[q].size(); ++oi)
          if (outs[q][oi].kind == cur_kind) flush(oi);
      } else {
        // one output kind per lane: lanes 0..K-1 select their copy's
        // arguments (no divergent branches) and issue the bulk copies together
        E.line("ocg_fence_async(); __syncwarp();");
        E.open("");
        std::string dsel = "nullptr", ssel = "nullptr", nsel = "0";
        for (size_t oi = outs[q].size(); oi-- > 0;) {
          const Out& o = outs[q][oi];
          const std::string S = i64(o.per_k);
          const std::string cond = "lane == " + std::to_string(oi);
          dsel = "(" + cond + " ? " + o.dst + " + k0" + R + " * " + S + " : " + dsel + ")";
          ssel = "(" + cond + " ? smem + " + i64(o.soff) + " + sh" + qn + "_" + std::to_string(oi) + " + r0" + R +
                 " * " + S + " : " + ssel + ")";
          nsel = "(" + cond + " ? nk" + R + " * (int)" + S + " : " + nsel + ")";
        }
        E.line("double* const bd = " + dsel + ";");
        E.line("const double* const bs = " + ssel + ";");
        E.line("const int bn = " + nsel + ";");
        E.line("if (lane < " + std::to_string(outs[q].size()) + " && bn > 0) { ocg_bulk_store(bd, bs, bn); ocg_bulk_commit(); }");
        E.close();
      }
    }
    if (uni && batched && !copies.empty()) {
      // every output of the tile: lane 0 issues the copies (uniform operands)
      E.line("ocg_fence_async(); __syncwarp();");
      E.open("if (lane == 0)");
      for (size_t q = 0; q < members.size(); ++q) {
        const Inst& mb = members[q];
        const Group& g = mb.objective ? nlp_.objs[static_cast<size_t>(mb.gi)] : nlp_.cons[static_cast<size_t>(mb.gi)];
        const std::string R = slice_of(g.range);
        for (const Out& o : outs[q]) {
          const std::string S = i64(o.per_k);
          E.line("if (nk" + R + " > 0) { double* const g = " + o.dst + " + k0" + R + " * " + S +
                 "; const double* const sb = smem + " + i64(o.soff) + " + r0" + R + " * " + S +
                 "; ocg_bulk_store(g, sb + ocg_shift(g, sb), nk" + R + " * (int)" + S + "); }");
        }
      }
      E.line("ocg_bulk_commit();");
      E.close();
    } else if (tma) {
      E.line("__syncwarp();");
    }
    if (batched && !copies.empty() && !uni) {
      // every output of the tile, one bulk copy per lane (chunks of 32)
      E.line("ocg_fence_async(); __syncwarp();");
      const int nslice = static_cast<int>(slices_.size());
      auto sel = [&](const std::string& C, const char* what) {
        std::string e = what + std::to_string(nslice - 1);
        for (int r = nslice - 2; r >= 0; --r)
          e = "(cd" + C + "_R == " + std::to_string(r) + " ? " + what + std::to_string(r) + " : " + e + ")";
        return e;
      };
      for (size_t c0 = 0; c0 < copies.size(); c0 += 32) {
        const std::string C = std::to_string(c0 / 32);
        E.open("if (cd" + C + "_R >= 0)");
        E.line("const OIX k0s = " + sel(C, "k0") + ";");
        E.line("const int r0s = " + sel(C, "r0") + ", nks = " + sel(C, "nk") + ";");
        E.open("if (nks > 0)");
        E.line("double* const g = cd" + C + "_dst + k0s * cd" + C + "_S;");
        E.line("const double* const sb = smem + cd" + C + "_soff + r0s * cd" + C + "_S;");
        E.line("ocg_bulk_store(g, sb + ocg_shift(g, sb), nks * (int)cd" + C + "_S);");
        E.line("ocg_bulk_commit();");
        E.close();
        E.close();
      }
    }
    load_from_ = nullptr;
    // every lane is done reading this tile's staged inputs before any lane
    // stages the next tile's (a kernel whose outputs all go straight to
    // global memory has no copy-out barrier)
    E.line("__syncwarp();");
    E.close();  // tile loop
    // the block's shared memory must outlive the bulk copies' reads; their
    // global writes complete with the grid (as a TMA-store epilogue's
    // wait_group.read 0 before exit)
    E.line("ocg_bulk_wait_read();");

    if (!tails.empty()) {
      E.open("if (blockIdx.x == gridDim.x - 1)");
      E.open("for (int s = threadIdx.x; s < (int)n_spec; s += OCG_BLOCK)");
      E.line("switch (s) {");
      for (size_t s = 0; s < tails.size(); ++s) {
        const Inst& in = tails[s];
        const Group& g = in.objective ? nlp_.objs[static_cast<size_t>(in.gi)] : nlp_.cons[static_cast<size_t>(in.gi)];
        const Parts p = parts(m, in.objective, g);
        E.open("case " + std::to_string(s) + ":");
        const std::string idx = in.k == 0 ? G(in.objective, in.gi, "lo", g.range.lo)
                                          : G(in.objective, in.gi, "hi", g.range.hi);
        E.line("const OIX sidx = " + idx + ";");
        std::vector<Check> sc;
        Fwd f = forward(E, g, "sidx", false, p.partials, 0, sc);
        for (const auto& c : sc) check_inline(E, c.v);
        group_body(E, m, in.objective, in.gi, f, i64(in.k));
        E.line("break;");
        E.close();
      }
      E.line("default: break;");
      E.line("}");
      E.close();
      E.close();
    }
    E.line("if (!ok || !fin(okacc)) *flag = 1;");
    E.depth = 0;
    E.line("}");
    E.line("");
    slices = 1;
    tail = static_cast<int>(tails.size());
    smem_out_ = per_warp * 8 * (opt_.block / 32);
    return E.out;
  }
};

}  // namespace

Generated generate(const Nlp& nlp, const Layout& lay, const GenOptions& opt) {
  Generator gen(nlp, lay, opt);
  return gen.module();
}

}  // namespace ocg

