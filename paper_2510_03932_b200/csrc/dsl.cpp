// Line-oriented OCP model language (grammar: /root/reference/proj/docs/grammar.md).
//
// Semantics follow the reference front end so that the same model text
// produces the same problem: tokenisation (proj/src/dsl/lexer.cpp:39-135),
// constant folding and alias expansion in the expression constructors
// (proj/src/dsl/ast.cpp:75-93), line dispatch and declaration/constraint/cost
// handling (proj/src/dsl/parser.cpp:160-498), and the final validation
// (parser.cpp:708-728). The front end runs once per problem and is not on the
// device path.
#include <cctype>
#include <charconv>
#include <cmath>
#include <limits>
#include <unordered_map>

#include "model.hpp"

namespace ocg {

namespace {
constexpr double kInf = std::numeric_limits<double>::infinity();

ExprP make(Expr e) { return std::make_shared<const Expr>(std::move(e)); }

double fold_unary(Un op, double x) {
  switch (op) {
    case Un::neg: return -x;
    case Un::sin: return std::sin(x);
    case Un::cos: return std::cos(x);
    case Un::tan: return std::tan(x);
    case Un::exp: return std::exp(x);
    case Un::log: return std::log(x);
    case Un::sqrt: return std::sqrt(x);
  }
  return 0.0;
}

double fold_binary(Bin op, double x, double y) {
  switch (op) {
    case Bin::add: return x + y;
    case Bin::sub: return x - y;
    case Bin::mul: return x * y;
    case Bin::div: return x / y;
    case Bin::pow: return std::pow(x, y);
  }
  return 0.0;
}
}  // namespace

ExprP num(double v) {
  Expr e;
  e.k = Expr::K::number;
  e.value = v;
  return make(std::move(e));
}
ExprP time_expr() {
  Expr e;
  e.k = Expr::K::time;
  return make(std::move(e));
}
ExprP ref(int decl, int comp, When w) {
  Expr e;
  e.k = Expr::K::ref;
  e.decl = decl;
  e.comp = comp;
  e.when = w;
  return make(std::move(e));
}
ExprP unary(Un op, ExprP a) {
  if (a->is_num()) return num(fold_unary(op, a->value));
  if (op == Un::neg && a->k == Expr::K::unary && a->uop == Un::neg) return a->a;
  Expr e;
  e.k = Expr::K::unary;
  e.uop = op;
  e.a = std::move(a);
  return make(std::move(e));
}
ExprP binary(Bin op, ExprP a, ExprP b) {
  if (a->is_num() && b->is_num()) return num(fold_binary(op, a->value, b->value));
  Expr e;
  e.k = Expr::K::binary;
  e.bop = op;
  e.a = std::move(a);
  e.b = std::move(b);
  return make(std::move(e));
}
ExprP vec(std::vector<ExprP> elems) {
  Expr e;
  e.k = Expr::K::vec;
  e.elems = std::move(elems);
  return make(std::move(e));
}
ExprP integral(ExprP a) {
  Expr e;
  e.k = Expr::K::integral;
  e.a = std::move(a);
  return make(std::move(e));
}

std::string Problem::comp_name(int d, int comp) const {
  const VarDecl& v = decls.at(static_cast<size_t>(d));
  if (comp < 0 || v.dim == 1) return v.name;
  if (!v.aliases.empty()) return v.aliases.at(static_cast<size_t>(comp));
  return v.name + std::to_string(comp + 1);
}

namespace {

// ---- tokens -----------------------------------------------------------------

enum class T { ident, keyword, integer, real, op, comma, lpar, rpar, lbr, rbr, eol, end };

struct Tok {
  T t;
  std::string s;
  int line;
  double v = 0.0;
};

bool is_keyword(const std::string& s) {
  return s == "in" || s == "time" || s == "state" || s == "control" || s == "variable" || s == "min" ||
         s == "max";
}

std::vector<Tok> lex(const std::string& src) {
  std::vector<Tok> out;
  int line = 1;
  size_t i = 0;
  const size_t n = src.size();
  auto alpha = [](char c) { return std::isalpha(static_cast<unsigned char>(c)) || c == '_'; };
  auto alnum = [](char c) { return std::isalnum(static_cast<unsigned char>(c)) || c == '_'; };
  auto digit = [](char c) { return std::isdigit(static_cast<unsigned char>(c)) != 0; };
  while (i < n) {
    const char c = src[i];
    if (c == '\n') {
      out.push_back({T::eol, "\n", line});
      ++line;
      ++i;
      continue;
    }
    if (c == ' ' || c == '\t' || c == '\r') {
      ++i;
      continue;
    }
    if (c == '#') {
      while (i < n && src[i] != '\n') ++i;
      continue;
    }
    if (alpha(c)) {
      size_t j = i;
      while (j < n && alnum(src[j])) ++j;
      std::string w = src.substr(i, j - i);
      out.push_back({is_keyword(w) ? T::keyword : T::ident, w, line});
      i = j;
      continue;
    }
    if (digit(c) || (c == '.' && i + 1 < n && digit(src[i + 1]))) {
      size_t j = i;
      bool real = false;
      while (j < n && digit(src[j])) ++j;
      if (j < n && src[j] == '.' && j + 1 < n && digit(src[j + 1])) {
        real = true;
        ++j;
        while (j < n && digit(src[j])) ++j;
      } else if (j < n && src[j] == '.' && !(j + 1 < n && alpha(src[j + 1]))) {
        real = true;  // "1."
        ++j;
      }
      if (j < n && (src[j] == 'e' || src[j] == 'E')) {  // exponent only with digits
        size_t k = j + 1;
        if (k < n && (src[k] == '+' || src[k] == '-')) ++k;
        if (k < n && digit(src[k])) {
          real = true;
          while (k < n && digit(src[k])) ++k;
          j = k;
        }
      }
      std::string w = src.substr(i, j - i);
      double v = 0.0;
      auto res = std::from_chars(w.data(), w.data() + w.size(), v);
      if (res.ec != std::errc()) throw ParseError(line, "malformed number '" + w + "'");
      out.push_back({real ? T::real : T::integer, w, line, v});
      i = j;
      continue;
    }
    if (i + 1 < n) {
      const std::string two = src.substr(i, 2);
      if (two == "<=" || two == ">=" || two == "==" || two == "=>") {
        out.push_back({T::op, two, line});
        i += 2;
        continue;
      }
    }
    switch (c) {
      case '+': case '-': case '*': case '/': case '^': case '<': case '>': case '=':
        out.push_back({T::op, std::string(1, c), line});
        break;
      case ',': out.push_back({T::comma, ",", line}); break;
      case '(': out.push_back({T::lpar, "(", line}); break;
      case ')': out.push_back({T::rpar, ")", line}); break;
      case '[': out.push_back({T::lbr, "[", line}); break;
      case ']': out.push_back({T::rbr, "]", line}); break;
      default: throw ParseError(line, std::string("illegal character '") + c + "'");
    }
    ++i;
  }
  out.push_back({T::end, "", line});
  return out;
}

// ---- parser -------------------------------------------------------------------

struct Flags {
  bool symbolic = false, instant = false, decl_ref = false, var_ref = false, integral = false;
};

class Parser {
 public:
  explicit Parser(const std::string& src) : toks_(lex(src)) {
    for (char ch : src) n_lines_ += ch == '\n';
    n_lines_ += 1;
  }

  Problem run() {
    while (!is(T::end)) {
      if (is(T::eol)) {
        ++pos_;
        continue;
      }
      statement();
      if (!is(T::eol) && !is(T::end)) fail("unexpected trailing '" + cur().s + "'");
    }
    validate();
    return std::move(p_);
  }

 private:
  struct Sym {
    enum class K { constant, alias, decl, comp } k;
    double value = 0.0;
    ExprP alias;
    int decl = -1, comp = -1;
  };

  std::vector<Tok> toks_;
  size_t pos_ = 0;
  int n_lines_ = 0;
  Problem p_;
  std::unordered_map<std::string, Sym> syms_;
  bool have_time_ = false, have_cost_ = false;

  const Tok& cur(size_t ahead = 0) const {
    const size_t i = pos_ + ahead;
    return i < toks_.size() ? toks_[i] : toks_.back();
  }
  bool is(T t, size_t ahead = 0) const { return cur(ahead).t == t; }
  bool is_op(const char* s, size_t ahead = 0) const { return is(T::op, ahead) && cur(ahead).s == s; }
  bool is_kw(const char* s) const { return is(T::keyword) && cur().s == s; }
  const Tok& take() { return toks_[pos_ < toks_.size() - 1 ? pos_++ : pos_]; }
  int line() const { return is(T::end) ? n_lines_ : cur().line; }
  [[noreturn]] void fail(const std::string& m) const { throw ParseError(line(), m); }
  [[noreturn]] void fail_at(int l, const std::string& m) const { throw ParseError(l, m); }
  void want(T t, const char* what) {
    if (!is(t)) fail(std::string("expected ") + what + ", got '" + cur().s + "'");
    ++pos_;
  }
  void want_op(const char* s) {
    if (!is_op(s)) fail(std::string("expected '") + s + "', got '" + cur().s + "'");
    ++pos_;
  }

  void define(const std::string& name, Sym s, int l) {
    if (syms_.count(name) || (have_time_ && name == p_.time_name)) fail_at(l, "duplicate identifier '" + name + "'");
    syms_.emplace(name, std::move(s));
  }
  const Sym* find(const std::string& name) const {
    auto it = syms_.find(name);
    return it == syms_.end() ? nullptr : &it->second;
  }
  // "x2" -> component 1 of declaration x (exact symbol names win)
  bool indexed(const std::string& name, int& decl, int& comp) const {
    size_t i = name.size();
    while (i > 0 && std::isdigit(static_cast<unsigned char>(name[i - 1]))) --i;
    if (i == 0 || i == name.size()) return false;
    const Sym* base = find(name.substr(0, i));
    if (!base || base->k != Sym::K::decl) return false;
    const int c = std::stoi(name.substr(i));
    if (c < 1 || c > p_.decls[static_cast<size_t>(base->decl)].dim) return false;
    decl = base->decl;
    comp = c - 1;
    return true;
  }

  void statement() {
    size_t end = pos_;
    while (toks_[end].t != T::eol && toks_[end].t != T::end) ++end;
    const Tok& last = toks_[end - 1];
    bool has_cost = false;
    for (size_t i = pos_; i < end; ++i) has_cost |= toks_[i].t == T::op && toks_[i].s == "=>";
    if (last.t == T::keyword && (last.s == "state" || last.s == "control" || last.s == "variable"))
      var_decl();
    else if (last.t == T::keyword && last.s == "time")
      time_decl();
    else if (has_cost)
      cost();
    else if (is(T::ident) && cur().s == "derivative")
      dynamics();
    else if (is(T::ident) && is_op("=", 1))
      definition();
    else
      constraint();
  }

  void var_decl() {
    const int l = line();
    if (!is(T::ident)) fail("expected identifier");
    VarDecl d;
    d.name = take().s;
    d.line = l;
    if (is_op("=")) {
      ++pos_;
      want(T::lpar, "'('");
      for (;;) {
        if (!is(T::ident)) fail("expected component name");
        d.aliases.push_back(take().s);
        if (!is(T::comma)) break;
        ++pos_;
      }
      want(T::rpar, "')'");
    }
    if (!is_kw("in")) fail("expected 'in'");
    ++pos_;
    if (!(is(T::ident) && cur().s == "R")) fail("expected 'R' or 'R^k'");
    ++pos_;
    if (is_op("^")) {
      ++pos_;
      if (!is(T::integer)) fail("expected integer dimension");
      d.dim = static_cast<int>(take().v);
      if (d.dim < 1) fail_at(l, "dimension must be >= 1");
    }
    want(T::comma, "','");
    if (!is(T::keyword)) fail("expected state/control/variable");
    const std::string kw = take().s;
    d.kind = kw == "state" ? VarKind::state : kw == "control" ? VarKind::control : VarKind::variable;
    if (!d.aliases.empty() && static_cast<int>(d.aliases.size()) != d.dim)
      fail_at(l, "component alias list has " + std::to_string(d.aliases.size()) + " names but dimension is " +
                     std::to_string(d.dim));
    const int idx = static_cast<int>(p_.decls.size());
    define(d.name, {Sym::K::decl, 0.0, nullptr, idx, -1}, l);
    for (size_t c = 0; c < d.aliases.size(); ++c)
      define(d.aliases[c], {Sym::K::comp, 0.0, nullptr, idx, static_cast<int>(c)}, l);
    p_.decls.push_back(std::move(d));
  }

  void time_bound(const ExprP& e, double& cval, int& var, int l) {
    if (e->is_num()) {
      cval = e->value;
      var = -1;
      return;
    }
    if (e->k == Expr::K::ref) {
      const VarDecl& d = p_.decls[static_cast<size_t>(e->decl)];
      if (d.kind == VarKind::variable && d.dim == 1) {
        var = e->decl;
        return;
      }
    }
    fail_at(l, "time bounds must be constants or a scalar decision variable");
  }

  void time_decl() {
    const int l = line();
    if (have_time_) fail_at(l, "duplicate time declaration");
    if (!is(T::ident)) fail("expected time identifier");
    const std::string name = take().s;
    if (syms_.count(name)) fail_at(l, "duplicate identifier '" + name + "'");
    if (!is_kw("in")) fail("expected 'in'");
    ++pos_;
    want(T::lbr, "'['");
    time_bound(expr(), p_.t0, p_.t0_var, l);
    want(T::comma, "','");
    time_bound(expr(), p_.tf, p_.tf_var, l);
    want(T::rbr, "']'");
    want(T::comma, "','");
    if (!is_kw("time")) fail("expected 'time'");
    ++pos_;
    p_.time_name = name;
    have_time_ = true;
  }

  void definition() {
    const int l = line();
    const std::string name = take().s;
    want_op("=");
    ExprP e = expr();
    if (e->k == Expr::K::vec) fail_at(l, "vector constants are not supported in definitions");
    if (e->is_num())
      define(name, {Sym::K::constant, e->value, nullptr, -1, -1}, l);
    else
      define(name, {Sym::K::alias, 0.0, e, -1, -1}, l);
  }

  void dynamics() {
    const int l = line();
    ++pos_;  // derivative
    want(T::lpar, "'('");
    if (!is(T::ident)) fail("expected state component");
    const std::string name = take().s;
    want(T::rpar, "')'");
    int decl = -1, comp = -1;
    if (const Sym* s = find(name)) {
      if (s->k == Sym::K::comp || s->k == Sym::K::decl) {
        decl = s->decl;
        comp = s->comp;
      }
    }
    if (decl < 0 && !indexed(name, decl, comp)) fail_at(l, "unknown state component '" + name + "'");
    const VarDecl& d = p_.decls[static_cast<size_t>(decl)];
    if (d.kind != VarKind::state) fail_at(l, "derivative of non-state '" + name + "'");
    if (comp < 0) {
      if (d.dim != 1) fail_at(l, "vector-form dynamics are not supported; write one equation per component");
      comp = 0;
    }
    want(T::lpar, "'('");
    if (!(is(T::ident) && have_time_ && cur().s == p_.time_name))
      fail("expected the time symbol '" + (have_time_ ? p_.time_name : std::string("t")) + "'");
    ++pos_;
    want(T::rpar, "')'");
    want_op("==");
    ExprP rhs = expr();
    const Flags f = flags(*rhs);
    if (f.instant) fail_at(l, "dynamics must not reference boundary instants");
    if (f.integral) fail_at(l, "integral(...) is only allowed in the cost");
    if (dim_of(*rhs, l) != 1) fail_at(l, "dynamics right-hand side must be scalar");
    for (const auto& dy : p_.dynamics)
      if (dy.decl == decl && dy.comp == comp)
        fail_at(l, "duplicate dynamics for state component '" + p_.comp_name(decl, comp) + "'");
    p_.dynamics.push_back({decl, comp, std::move(rhs), l});
  }

  std::vector<double> bounds_of(const ExprP& e, int dim, int l) const {
    if (e->is_num()) return std::vector<double>(static_cast<size_t>(dim), e->value);
    if (e->k == Expr::K::vec) {
      if (static_cast<int>(e->elems.size()) != dim)
        fail_at(l, "wrong bound dimension (expected " + std::to_string(dim) + ", got " +
                       std::to_string(e->elems.size()) + ")");
      std::vector<double> out;
      for (const auto& el : e->elems) {
        if (!el->is_num()) fail_at(l, "constraint bounds must be constant");
        out.push_back(el->value);
      }
      return out;
    }
    fail_at(l, "constraint bounds must be constant");
  }

  void constraint() {
    const int l = line();
    ExprP first = expr();
    std::vector<std::pair<std::string, ExprP>> rel;
    while (is_op("<=") || is_op(">=") || is_op("==")) {
      std::string op = take().s;
      rel.emplace_back(op, expr());
    }
    if (rel.empty()) fail_at(l, "expected a constraint, declaration, or cost");
    if (is_op("<") || is_op(">")) fail("strict inequalities are not supported");
    auto constant = [](const ExprP& e) { return e->k == Expr::K::number || e->k == Expr::K::vec; };

    Con c;
    c.line = l;
    if (rel.size() == 2) {
      if (rel[0].first != rel[1].first || rel[0].first == "==")
        fail_at(l, "chained constraints must use a single direction of <= or >=");
      if (!constant(first) || !constant(rel[1].second)) fail_at(l, "chained constraint bounds must be constant");
      c.expr = rel[0].second;
      const int dim = dim_of(*c.expr, l);
      std::vector<double> outer = bounds_of(first, dim, l), inner = bounds_of(rel[1].second, dim, l);
      if (rel[0].first == "<=") {
        c.lo = outer;
        c.hi = inner;
      } else {
        c.lo = inner;
        c.hi = outer;
      }
    } else if (rel.size() == 1) {
      const std::string& op = rel[0].first;
      const ExprP& lhs = first;
      const ExprP& rhs = rel[0].second;
      const bool lc = constant(lhs), rc = constant(rhs);
      if (lc && rc) fail_at(l, "constraint has no unknowns");
      if (!lc && !rc) {
        c.expr = binary(Bin::sub, lhs, rhs);
        const size_t dim = static_cast<size_t>(dim_of(*c.expr, l));
        c.lo.assign(dim, op == "<=" ? -kInf : 0.0);
        c.hi.assign(dim, op == ">=" ? kInf : 0.0);
      } else {
        c.expr = lc ? rhs : lhs;
        const int dim = dim_of(*c.expr, l);
        std::vector<double> bnd = bounds_of(lc ? lhs : rhs, dim, l);
        const bool bound_is_upper = (op == "<=" && !lc) || (op == ">=" && lc);
        if (op == "==") {
          c.lo = bnd;
          c.hi = bnd;
        } else if (bound_is_upper) {
          c.lo.assign(static_cast<size_t>(dim), -kInf);
          c.hi = bnd;
        } else {
          c.lo = bnd;
          c.hi.assign(static_cast<size_t>(dim), kInf);
        }
      }
    } else {
      fail_at(l, "too many relations in one constraint");
    }
    for (size_t i = 0; i < c.lo.size(); ++i)
      if (!(c.lo[i] <= c.hi[i])) fail_at(l, "empty constraint interval (lower > upper)");
    const Flags f = flags(*c.expr);
    if (f.integral) fail_at(l, "integral(...) is only allowed in the cost");
    if (f.symbolic && f.instant) fail_at(l, "cannot mix boundary instants and symbolic time in one constraint");
    if (f.symbolic)
      c.k = Con::K::path;
    else if (f.instant || f.decl_ref)
      c.k = Con::K::boundary;
    else if (f.var_ref)
      c.k = c.expr->k == Expr::K::ref ? Con::K::box_variable : Con::K::boundary;
    else
      fail_at(l, "constraint has no unknowns");
    p_.cons.push_back(std::move(c));
  }

  void add_term(ExprP& slot, ExprP term, bool negate) {
    if (negate) term = unary(Un::neg, std::move(term));
    slot = slot ? binary(Bin::add, slot, std::move(term)) : std::move(term);
  }

  // top-level sums split into integral (Lagrange) and endpoint (Mayer) terms
  void split(const ExprP& e, bool negate, int l) {
    if (e->k == Expr::K::binary && (e->bop == Bin::add || e->bop == Bin::sub)) {
      split(e->a, negate, l);
      split(e->b, e->bop == Bin::sub ? !negate : negate, l);
      return;
    }
    if (e->k == Expr::K::unary && e->uop == Un::neg) return split(e->a, !negate, l);
    if (e->k == Expr::K::integral) return add_term(p_.lagrange, e->a, negate);
    if (e->k == Expr::K::binary && e->bop == Bin::mul) {
      if (e->a->is_num() && e->b->k == Expr::K::integral)
        return add_term(p_.lagrange, binary(Bin::mul, e->a, e->b->a), negate);
      if (e->b->is_num() && e->a->k == Expr::K::integral)
        return add_term(p_.lagrange, binary(Bin::mul, e->b, e->a->a), negate);
    }
    if (e->k == Expr::K::binary && e->bop == Bin::div && e->a->k == Expr::K::integral && e->b->is_num())
      return add_term(p_.lagrange, binary(Bin::div, e->a->a, e->b), negate);
    if (flags(*e).integral) fail_at(l, "integral(...) must appear linearly in the cost");
    add_term(p_.mayer, e, negate);
  }

  void cost() {
    const int l = line();
    if (have_cost_) fail_at(l, "duplicate cost declaration");
    ExprP e = expr();
    want_op("=>");
    if (!is(T::keyword) || (cur().s != "min" && cur().s != "max")) fail("expected 'min' or 'max'");
    const bool is_max = take().s == "max";
    split(e, false, l);
    if (!p_.mayer && !p_.lagrange) fail_at(l, "cost is constant");
    if (p_.mayer) {
      if (flags(*p_.mayer).symbolic) fail_at(l, "endpoint cost terms must use t0/tf instants, not symbolic time");
      if (dim_of(*p_.mayer, l) != 1) fail_at(l, "cost must be scalar");
    }
    if (p_.lagrange) {
      if (flags(*p_.lagrange).instant) fail_at(l, "boundary instants are not allowed inside integral(...)");
      if (dim_of(*p_.lagrange, l) != 1) fail_at(l, "cost must be scalar");
    }
    if (is_max) {
      if (p_.mayer) p_.mayer = unary(Un::neg, p_.mayer);
      if (p_.lagrange) p_.lagrange = unary(Un::neg, p_.lagrange);
      p_.maximize = true;
    }
    have_cost_ = true;
  }

  // ---- expressions ----
  ExprP expr() {
    ExprP e = term();
    while (is_op("+") || is_op("-")) {
      const Bin op = take().s == "+" ? Bin::add : Bin::sub;
      e = binary(op, e, term());
    }
    return e;
  }
  ExprP term() {
    ExprP e = signed_factor();
    while (is_op("*") || is_op("/")) {
      const Bin op = take().s == "*" ? Bin::mul : Bin::div;
      e = binary(op, e, signed_factor());
    }
    return e;
  }
  ExprP signed_factor() {
    if (is_op("-")) {
      ++pos_;
      return unary(Un::neg, signed_factor());
    }
    if (is_op("+")) {
      ++pos_;
      return signed_factor();
    }
    return factor();
  }
  ExprP factor() {
    const bool numeric = is(T::integer) || is(T::real);
    ExprP e = atom();
    if (numeric && (is(T::ident) || is(T::lpar))) return binary(Bin::mul, e, factor());  // 2pi, 0.5u(t)^2
    while (is_op("^")) {
      ++pos_;
      e = binary(Bin::pow, e, signed_factor());
    }
    return e;
  }
  ExprP atom() {
    if (is(T::integer) || is(T::real)) return num(take().v);
    if (is(T::lpar)) {
      ++pos_;
      ExprP e = expr();
      want(T::rpar, "')'");
      return e;
    }
    if (is(T::lbr)) {
      ++pos_;
      std::vector<ExprP> el;
      if (!is(T::rbr)) {
        el.push_back(expr());
        while (is(T::comma)) {
          ++pos_;
          el.push_back(expr());
        }
      }
      want(T::rbr, "']'");
      return vec(std::move(el));
    }
    if (is(T::ident)) return name_ref();
    fail("expected an expression, got '" + cur().s + "'");
  }

  ExprP call_arg() {
    want(T::lpar, "'('");
    ExprP a = expr();
    want(T::rpar, "')'");
    return a;
  }

  ExprP name_ref() {
    const int l = line();
    const std::string name = take().s;
    static const std::unordered_map<std::string, Un> funcs = {{"sin", Un::sin}, {"cos", Un::cos},
                                                              {"tan", Un::tan}, {"exp", Un::exp},
                                                              {"log", Un::log}, {"sqrt", Un::sqrt}};
    if (auto it = funcs.find(name); it != funcs.end()) return unary(it->second, call_arg());
    if (name == "integral") return integral(call_arg());
    if (name == "zeros") {
      want(T::lpar, "'('");
      if (!is(T::integer)) fail("expected integer in zeros(n)");
      const int n = static_cast<int>(take().v);
      want(T::rpar, "')'");
      return vec(std::vector<ExprP>(static_cast<size_t>(n), num(0.0)));
    }
    if (name == "pi") return num(M_PI);
    if (name == "derivative") fail_at(l, "derivative(...) may only start a dynamics line");
    if (have_time_ && name == p_.time_name) return time_expr();
    if (const Sym* s = find(name)) {
      switch (s->k) {
        case Sym::K::constant: return num(s->value);
        case Sym::K::alias: return s->alias;
        case Sym::K::decl: return ref_tail(s->decl, -1, name, l);
        case Sym::K::comp: return ref_tail(s->decl, s->comp, name, l);
      }
    }
    int decl = -1, comp = -1;
    if (indexed(name, decl, comp)) return ref_tail(decl, comp, name, l);
    fail_at(l, "unknown identifier '" + name + "'");
  }

  ExprP ref_tail(int decl, int comp, const std::string& name, int l) {
    const VarDecl& d = p_.decls[static_cast<size_t>(decl)];
    if (is(T::lpar)) {
      ++pos_;
      const When w = time_arg(l);
      want(T::rpar, "')'");
      if (d.kind == VarKind::variable) fail_at(l, "free variable '" + name + "' takes no time argument");
      return ref(decl, comp, w);
    }
    if (d.kind != VarKind::variable)
      fail_at(l, std::string(d.kind == VarKind::state ? "state '" : "control '") + name +
                     "' requires a time argument");
    return ref(decl, comp, When::symbolic);
  }

  When time_arg(int l) {
    ExprP e = expr();
    if (e->k == Expr::K::time) return When::symbolic;
    if (e->k == Expr::K::ref) {
      if (p_.t0_var >= 0 && e->decl == p_.t0_var) return When::initial;
      if (p_.tf_var >= 0 && e->decl == p_.tf_var) return When::final;
      fail_at(l, "time argument must be the time symbol, t0, or tf");
    }
    if (e->is_num()) {
      if (!have_time_) fail_at(l, "time must be declared before boundary references");
      if (p_.t0_var < 0 && e->value == p_.t0) return When::initial;
      if (p_.tf_var < 0 && e->value == p_.tf) return When::final;
      fail_at(l, "time instant must be t0 or tf; interior instants are not supported");
    }
    fail_at(l, "malformed time argument");
  }

  Flags flags(const Expr& e) const {
    Flags f;
    auto merge = [&f](const Flags& g) {
      f.symbolic |= g.symbolic;
      f.instant |= g.instant;
      f.decl_ref |= g.decl_ref;
      f.var_ref |= g.var_ref;
      f.integral |= g.integral;
    };
    switch (e.k) {
      case Expr::K::number: break;
      case Expr::K::time: f.symbolic = true; break;
      case Expr::K::ref:
        if (p_.decls[static_cast<size_t>(e.decl)].kind == VarKind::variable) {
          f.var_ref = true;
        } else {
          f.decl_ref = true;
          (e.when == When::symbolic ? f.symbolic : f.instant) = true;
        }
        break;
      case Expr::K::unary: merge(flags(*e.a)); break;
      case Expr::K::integral:
        merge(flags(*e.a));
        f.integral = true;
        break;
      case Expr::K::binary:
        merge(flags(*e.a));
        merge(flags(*e.b));
        break;
      case Expr::K::vec:
        for (const auto& el : e.elems) merge(flags(*el));
        break;
    }
    return f;
  }

  int dim_of(const Expr& e, int l) const {
    switch (e.k) {
      case Expr::K::number:
      case Expr::K::time: return 1;
      case Expr::K::ref: return e.comp >= 0 ? 1 : p_.decls[static_cast<size_t>(e.decl)].dim;
      case Expr::K::unary:
      case Expr::K::integral: return dim_of(*e.a, l);
      case Expr::K::binary: {
        const int da = dim_of(*e.a, l), db = dim_of(*e.b, l);
        if (da == db || db == 1) return da;
        if (da == 1) return db;
        fail_at(l, "wrong bound dimension: operands have dimensions " + std::to_string(da) + " and " +
                       std::to_string(db));
      }
      case Expr::K::vec: return static_cast<int>(e.elems.size());
    }
    return 1;
  }

  void validate() {
    if (!have_time_) throw ParseError(1, "missing time declaration");
    if (!have_cost_) throw ParseError(n_lines_, "missing cost declaration");
    for (size_t di = 0; di < p_.decls.size(); ++di) {
      const VarDecl& d = p_.decls[di];
      if (d.kind != VarKind::state) continue;
      for (int c = 0; c < d.dim; ++c) {
        bool found = false;
        for (const auto& dy : p_.dynamics) found |= dy.decl == static_cast<int>(di) && dy.comp == c;
        if (!found)
          throw ParseError(d.line,
                           "missing dynamics for state component '" + p_.comp_name(static_cast<int>(di), c) + "'");
      }
    }
    if (p_.dynamics.empty()) throw ParseError(1, "problem declares no state dynamics");
  }
};

}  // namespace

Problem parse_problem(const std::string& source) { return Parser(source).run(); }

}  // namespace ocg
