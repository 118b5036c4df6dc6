// Direct transcription on a uniform grid into generator groups.
//
// Follows /root/reference/proj/src/transcribe/transcribe.cpp:180-409: slab
// layout in declaration order (node-major, base + node*dim + comp), one 1-row
// dynamics group per state component over steps [0, N), boundary groups at a
// single index, path groups over nodes [0, N] (euler control-only: [0, N)),
// trapezoid/left-rectangle Lagrange quadrature plus the Mayer term, row
// numbering, bounds, clip boxes and the start point. Node creation order is
// kept equal to the reference build (g++), which fixes each graph's node ids
// and therefore the accumulation order of every reverse sweep.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <sstream>

#include "model.hpp"

namespace ocg {

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

Index slab_slot(const std::vector<Slab>& slabs, int decl, int comp, Index node) {
  const Slab& s = slabs[static_cast<size_t>(decl)];
  return s.base + node * s.dim + comp;
}

class Lowering {
 public:
  Lowering(const Problem& p, const std::vector<Slab>& slabs, Index N) : p_(p), slabs_(slabs), N_(N) {}

  int endpoint(Graph& g, double cval, int var, const char* fallback) const {
    if (var < 0) return g.cnst(cval);
    const std::string& nm = p_.decls[static_cast<size_t>(var)].name;
    return g.input({slab_slot(slabs_, var, 0, 0), 0}, nm.empty() ? fallback : nm);
  }

  // h = (tf - t0) / N
  int step(Graph& g) const {
    const int t0 = endpoint(g, p_.t0, p_.t0_var, "t0");
    const int tf = endpoint(g, p_.tf, p_.tf_var, "tf");
    const int n = g.cnst(static_cast<double>(N_));
    const int span = g.sub(tf, t0);
    return g.div(span, n);
  }

  int lower(Graph& g, const Expr& e, int comp, int offset) const {
    switch (e.k) {
      case Expr::K::number: return g.cnst(e.value);
      case Expr::K::time: {
        const int t0 = endpoint(g, p_.t0, p_.t0_var, "t0");
        const int h = step(g);
        const int i = g.index(static_cast<double>(offset));
        return g.add(t0, g.mul(i, h));
      }
      case Expr::K::ref: return lower_ref(g, e, comp, offset);
      case Expr::K::unary: {
        const int a = lower(g, *e.a, comp, offset);
        switch (e.uop) {
          case Un::neg: return g.neg(a);
          case Un::sin: return g.unary(Op::sin, a);
          case Un::cos: return g.unary(Op::cos, a);
          case Un::tan: return g.unary(Op::tan, a);
          case Un::exp: return g.unary(Op::exp, a);
          case Un::log: return g.unary(Op::log, a);
          case Un::sqrt: return g.unary(Op::sqrt, a);
        }
        return a;
      }
      case Expr::K::binary: {
        if (e.bop == Bin::pow) {
          if (!e.b->is_num()) throw std::runtime_error("non-constant exponents are not supported");
          return g.pow(lower(g, *e.a, comp, offset), e.b->value);
        }
        const int a = lower(g, *e.a, comp, offset);
        const int b = lower(g, *e.b, comp, offset);
        switch (e.bop) {
          case Bin::add: return g.add(a, b);
          case Bin::sub: return g.sub(a, b);
          case Bin::mul: return g.mul(a, b);
          case Bin::div: return g.div(a, b);
          default: return a;
        }
      }
      case Expr::K::vec: return lower(g, *e.elems[static_cast<size_t>(comp)], 0, offset);
      case Expr::K::integral: throw std::runtime_error("integral(...) must be handled by the cost lowering");
    }
    return g.cnst(0.0);
  }

 private:
  int lower_ref(Graph& g, const Expr& e, int comp, int offset) const {
    const int c = e.comp >= 0 ? e.comp : comp;
    const VarDecl& d = p_.decls[static_cast<size_t>(e.decl)];
    const std::string label = p_.comp_name(e.decl, d.dim == 1 ? -1 : c);
    if (d.kind == VarKind::variable) return g.input({slab_slot(slabs_, e.decl, c, 0), 0}, label);
    switch (e.when) {
      case When::initial: return g.input({slab_slot(slabs_, e.decl, c, 0), 0}, label + "@0");
      case When::final: return g.input({slab_slot(slabs_, e.decl, c, N_), 0}, label + "@N");
      case When::symbolic: {
        const Slab& s = slabs_[static_cast<size_t>(e.decl)];
        return g.input({s.base + static_cast<Index>(offset) * s.dim + c, s.dim},
                       label + (offset == 0 ? "@i" : "@i+1"));
      }
    }
    return g.cnst(0.0);
  }

  const Problem& p_;
  const std::vector<Slab>& slabs_;
  Index N_;
};

bool controls_only(const Problem& p, const Expr& e) {
  switch (e.k) {
    case Expr::K::number: return true;
    case Expr::K::time: return false;
    case Expr::K::ref: return p.decls[static_cast<size_t>(e.decl)].kind == VarKind::control;
    case Expr::K::unary:
    case Expr::K::integral: return controls_only(p, *e.a);
    case Expr::K::binary: return controls_only(p, *e.a) && controls_only(p, *e.b);
    case Expr::K::vec:
      for (const auto& el : e.elems)
        if (!controls_only(p, *el)) return false;
      return true;
  }
  return false;
}

int width(const Problem& p, const Expr& e) {
  switch (e.k) {
    case Expr::K::number:
    case Expr::K::time: return 1;
    case Expr::K::ref: return e.comp >= 0 ? 1 : p.decls[static_cast<size_t>(e.decl)].dim;
    case Expr::K::unary:
    case Expr::K::integral: return width(p, *e.a);
    case Expr::K::binary: return std::max(width(p, *e.a), width(p, *e.b));
    case Expr::K::vec: return static_cast<int>(e.elems.size());
  }
  return 1;
}

Group finish_group(Kernel k, Range r, Group::Kind kind, std::string label) {
  Group g;
  g.kind = kind;
  g.pattern = sparsity_of(k);
  g.kernel = std::move(k);
  g.range = r;
  g.label = std::move(label);
  return g;
}

void tighten(std::vector<double>& lo, std::vector<double>& hi, size_t slot, double l, double u) {
  lo[slot] = std::max(lo[slot], l);
  hi[slot] = std::min(hi[slot], u);
}

}  // namespace

Nlp transcribe(const Problem& p, Scheme scheme, Index N, bool boxes_as_bounds) {
  if (N < 1) throw std::invalid_argument("grid size N must be >= 1");
  Nlp nlp;
  nlp.scheme = scheme;
  nlp.N = N;
  nlp.maximize = p.maximize;

  Index base = 0;
  for (const auto& d : p.decls) {
    Slab s;
    s.kind = d.kind;
    s.dim = d.dim;
    s.base = base;
    s.nodes = d.kind == VarKind::variable ? 1 : N + 1;
    base += s.dim * s.nodes;
    nlp.slabs.push_back(s);
  }
  nlp.nvar = base;
  const auto nv = static_cast<size_t>(nlp.nvar);
  nlp.lvar.assign(nv, -kInf);
  nlp.uvar.assign(nv, kInf);

  Lowering low(p, nlp.slabs, N);

  for (const auto& dy : p.dynamics) {
    Kernel k;
    Graph& g = k.graph;
    const Slab& s = nlp.slabs[static_cast<size_t>(dy.decl)];
    const std::string nm = p.comp_name(dy.decl, p.decls[static_cast<size_t>(dy.decl)].dim == 1 ? -1 : dy.comp);
    const int xi = g.input({s.base + dy.comp, s.dim}, nm + "@i");
    const int xn = g.input({s.base + s.dim + dy.comp, s.dim}, nm + "@i+1");
    const int h = low.step(g);
    int root;
    if (scheme == Scheme::euler) {
      const int f0 = low.lower(g, *dy.rhs, 0, 0);
      const int hf = g.mul(h, f0);
      const int dx = g.sub(xn, xi);
      root = g.sub(dx, hf);
    } else {
      const int f0 = low.lower(g, *dy.rhs, 0, 0);
      const int f1 = low.lower(g, *dy.rhs, 0, 1);
      const int two = g.cnst(2.0);
      const int avg = g.div(g.mul(h, g.add(f0, f1)), two);
      const int dx = g.sub(xn, xi);
      root = g.sub(dx, avg);
    }
    k.roots.push_back(root);
    Group grp = finish_group(std::move(k), {0, N, false}, Group::Kind::dynamics, "dynamics " + nm);
    grp.lower = {0.0};
    grp.upper = {0.0};
    nlp.cons.push_back(std::move(grp));
  }

  for (const auto& c : p.cons) {
    const int dim = width(p, *c.expr);
    if (c.k == Con::K::box_variable) {
      const auto slot = static_cast<size_t>(slab_slot(nlp.slabs, c.expr->decl, std::max(c.expr->comp, 0), 0));
      tighten(nlp.lvar, nlp.uvar, slot, c.lo[0], c.hi[0]);
      if (nlp.lvar[slot] > nlp.uvar[slot])
        throw std::runtime_error("contradictory bounds on variable at line " + std::to_string(c.line));
      continue;
    }
    const bool single_slot = c.expr->k == Expr::K::ref &&
                             (c.expr->comp >= 0 || p.decls[static_cast<size_t>(c.expr->decl)].dim == 1);
    if (boxes_as_bounds && c.k == Con::K::path && single_slot) {
      const int comp = std::max(c.expr->comp, 0);
      for (Index node = 0; node <= N; ++node)
        tighten(nlp.lvar, nlp.uvar, static_cast<size_t>(slab_slot(nlp.slabs, c.expr->decl, comp, node)), c.lo[0],
                c.hi[0]);
      continue;
    }
    Kernel k;
    for (int comp = 0; comp < dim; ++comp) k.roots.push_back(low.lower(k.graph, *c.expr, comp, 0));
    Group grp;
    if (c.k == Con::K::boundary) {
      grp = finish_group(std::move(k), {0, 1, false}, Group::Kind::boundary, "boundary line " + std::to_string(c.line));
    } else {
      const Index hi = (scheme == Scheme::euler && controls_only(p, *c.expr)) ? N : N + 1;
      grp = finish_group(std::move(k), {0, hi, false}, Group::Kind::path, "path line " + std::to_string(c.line));
    }
    grp.lower = c.lo;
    grp.upper = c.hi;
    nlp.cons.push_back(std::move(grp));
  }

  // start-value clip boxes: slot bounds tightened by single-slot path rows
  nlp.clip_lo = nlp.lvar;
  nlp.clip_hi = nlp.uvar;
  for (const auto& c : p.cons) {
    if (c.k != Con::K::path || c.expr->k != Expr::K::ref) continue;
    if (c.expr->comp < 0 && p.decls[static_cast<size_t>(c.expr->decl)].dim != 1) continue;
    const int comp = std::max(c.expr->comp, 0);
    for (Index node = 0; node <= N; ++node)
      tighten(nlp.clip_lo, nlp.clip_hi, static_cast<size_t>(slab_slot(nlp.slabs, c.expr->decl, comp, node)),
              c.lo[0], c.hi[0]);
  }

  nlp.m_con = 0;
  for (auto& grp : nlp.cons) {
    grp.row_base = nlp.m_con;
    nlp.m_con += grp.rows();
  }
  nlp.lcon.resize(static_cast<size_t>(nlp.m_con));
  nlp.ucon.resize(static_cast<size_t>(nlp.m_con));
  for (const auto& grp : nlp.cons)
    for (Index k = 0; k < grp.range.count(); ++k)
      for (int r = 0; r < grp.out_dim(); ++r) {
        const auto row = static_cast<size_t>(grp.row_base + k * grp.out_dim() + r);
        nlp.lcon[row] = grp.lower[static_cast<size_t>(r)];
        nlp.ucon[row] = grp.upper[static_cast<size_t>(r)];
      }

  // objective: scheme-matched Lagrange quadrature, then the Mayer term
  auto running = [&](Range r, double w, const char* label) {
    Kernel k;
    const int h = low.step(k.graph);
    const int body = low.lower(k.graph, *p.lagrange, 0, 0);
    k.roots.push_back(k.graph.mul(h, body));
    Group grp = finish_group(std::move(k), r, Group::Kind::path, label);
    grp.weight = w;
    nlp.objs.push_back(std::move(grp));
  };
  if (p.lagrange) {
    if (scheme == Scheme::euler) {
      running({0, N, false}, 1.0, "lagrange (left rectangle)");
    } else {
      running({0, N, true}, 0.5, "lagrange (trapezoid endpoints)");
      if (N >= 2) running({1, N, false}, 1.0, "lagrange (trapezoid interior)");
    }
  }
  if (p.mayer) {
    Kernel k;
    k.roots.push_back(low.lower(k.graph, *p.mayer, 0, 0));
    Group grp = finish_group(std::move(k), {0, 1, false}, Group::Kind::boundary, "mayer");
    nlp.objs.push_back(std::move(grp));
  }

  // start point: 0.1 per slot, clipped into the clip box
  nlp.x_start.assign(nv, 0.1);
  for (size_t i = 0; i < nv; ++i) nlp.x_start[i] = std::clamp(nlp.x_start[i], nlp.clip_lo[i], nlp.clip_hi[i]);

  if (scheme == Scheme::euler) {  // U_N is referenced by nothing: pin it
    for (const auto& s : nlp.slabs) {
      if (s.kind != VarKind::control) continue;
      for (int c = 0; c < s.dim; ++c) {
        const auto slot = static_cast<size_t>(s.base + N * s.dim + c);
        nlp.lvar[slot] = nlp.uvar[slot] = nlp.x_start[slot];
        nlp.clip_lo[slot] = nlp.clip_hi[slot] = nlp.x_start[slot];
      }
    }
  }

  std::vector<char> used(nv, 0);
  auto mark = [&](const Group& grp) {
    for (const auto& a : grp.kernel.graph.inputs()) {
      if (a.stride == 0)
        used[static_cast<size_t>(a.base)] = 1;
      else
        for (Index k = 0; k < grp.range.count(); ++k) used[static_cast<size_t>(a.slot(grp.range.at(k)))] = 1;
    }
  };
  for (const auto& grp : nlp.cons) mark(grp);
  for (const auto& grp : nlp.objs) mark(grp);
  for (size_t s = 0; s < nv; ++s)
    if (!used[s] && !std::isfinite(nlp.lvar[s]) && !std::isfinite(nlp.uvar[s]))
      throw std::runtime_error("decision slot " + std::to_string(s) +
                               " is referenced by no constraint, objective, or bound");
  return nlp;
}

// ---- structure dump (same schema as oracle/ref_harness.cpp ref_model_json) ----

namespace {
void put_num(std::ostringstream& os, double v) {
  if (std::isnan(v)) {
    os << "NaN";
  } else if (std::isinf(v)) {
    os << (v > 0 ? "Infinity" : "-Infinity");
  } else {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    os << buf;
  }
}
void put_str(std::ostringstream& os, const std::string& s) {
  os << '"';
  for (char c : s) {
    if (c == '"' || c == '\\') os << '\\';
    os << c;
  }
  os << '"';
}
void put_vec(std::ostringstream& os, const std::vector<double>& v) {
  os << '[';
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) os << ',';
    put_num(os, v[i]);
  }
  os << ']';
}
void put_group(std::ostringstream& os, const Group& g, bool constraint) {
  const Graph& gr = g.kernel.graph;
  os << "{\"nodes\":[";
  for (size_t i = 0; i < gr.nodes().size(); ++i) {
    const Node& n = gr.nodes()[i];
    if (i) os << ',';
    os << '[' << static_cast<int>(n.op) << ',' << n.a << ',' << n.b << ',';
    put_num(os, n.c);
    os << ']';
  }
  os << "],\"roots\":[";
  for (size_t i = 0; i < g.kernel.roots.size(); ++i) os << (i ? "," : "") << g.kernel.roots[i];
  os << "],\"inputs\":[";
  for (size_t i = 0; i < gr.inputs().size(); ++i) {
    os << (i ? "," : "") << '[' << gr.inputs()[i].base << ',' << gr.inputs()[i].stride << ',';
    put_str(os, gr.labels()[i]);
    os << ']';
  }
  os << "],\"jac\":[";
  for (size_t i = 0; i < g.pattern.jac.size(); ++i)
    os << (i ? "," : "") << '[' << g.pattern.jac[i].first << ',' << g.pattern.jac[i].second << ']';
  os << "],\"hess\":[";
  for (size_t i = 0; i < g.pattern.hess.size(); ++i)
    os << (i ? "," : "") << '[' << g.pattern.hess[i].first << ',' << g.pattern.hess[i].second << ']';
  os << "],\"label\":";
  put_str(os, g.label);
  os << ",\"range\":[" << g.range.lo << ',' << g.range.hi << ',' << (g.range.endpoints ? "true" : "false") << ']';
  if (constraint) {
    os << ",\"kind\":" << static_cast<int>(g.kind) << ",\"out_dim\":" << g.out_dim()
       << ",\"row_base\":" << g.row_base << ",\"lower\":";
    put_vec(os, g.lower);
    os << ",\"upper\":";
    put_vec(os, g.upper);
  } else {
    os << ",\"weight\":";
    put_num(os, g.weight);
  }
  os << '}';
}
}  // namespace

std::string Nlp::structure_json() const {
  std::ostringstream os;
  os << "{\"N\":" << N << ",\"nvar\":" << nvar << ",\"m_con\":" << m_con
     << ",\"maximize\":" << (maximize ? "true" : "false") << ",\"scheme\":\""
     << (scheme == Scheme::euler ? "euler" : "trapezoid") << "\",\"layout\":[";
  for (size_t i = 0; i < slabs.size(); ++i)
    os << (i ? "," : "") << '[' << static_cast<int>(slabs[i].kind) << ',' << slabs[i].dim << ',' << slabs[i].base
       << ',' << slabs[i].nodes << ']';
  os << "],\"con_groups\":[";
  for (size_t i = 0; i < cons.size(); ++i) {
    if (i) os << ',';
    put_group(os, cons[i], true);
  }
  os << "],\"obj_groups\":[";
  for (size_t i = 0; i < objs.size(); ++i) {
    if (i) os << ',';
    put_group(os, objs[i], false);
  }
  os << "]}";
  return os.str();
}

}  // namespace ocg
