// Host-side model of a direct-transcription OCP: DSL front end, hash-consed
// scalar graphs with structural sparsity, and the generator-structured NLP
// (the reference's StructuredNlp). This is setup code that runs once per
// problem; it produces the exact graphs, patterns, ranges and offsets the
// device evaluation plan is generated from.
//
// Reference interfaces mirrored (same semantics, bit-identical structure):
//   kernel::Graph / Node / Op / InputAddress / Pattern / detect_pattern
//       /root/reference/proj/include/octrans/kernel/graph.hpp:35-133
//   transcribe::Slab / VariableLayout / IndexRange / ConstraintGroup /
//       ObjectiveGroup / StructuredNlp
//       /root/reference/proj/include/octrans/transcribe/nlp.hpp:36-117
//   dsl::parse_ocp   /root/reference/proj/include/octrans/dsl/parser.hpp:33
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

namespace ocg {

using Index = std::int64_t;

// ---------------------------------------------------------------------------
// Scalar expression graph (one kernel = one graph + one root per output row)
// ---------------------------------------------------------------------------

// Numbering equals the reference enum (graph.hpp:43-59) so structure dumps
// compare directly.
enum class Op : std::uint8_t { cnst, input, index, add, sub, mul, div, neg, sin, cos, tan, exp, log, sqrt, pow };

struct Node {
  Op op = Op::cnst;
  std::int32_t a = -1;
  std::int32_t b = -1;
  double c = 0.0;
};

// slot(i) = base + stride * i (stride 0: absolute slot).
struct Addr {
  Index base = 0;
  Index stride = 0;
  Index slot(Index i) const { return base + stride * i; }
  bool operator==(const Addr& o) const { return base == o.base && stride == o.stride; }
};

class Graph {
 public:
  int cnst(double v);
  int input(Addr addr, const std::string& label = "");
  int index(double offset);
  int add(int a, int b);
  int sub(int a, int b);
  int mul(int a, int b);
  int div(int a, int b);
  int neg(int a);
  int pow(int a, double c);
  int unary(Op op, int a);
  // A graph handed over node for node by another front end (the reference's
  // StructuredNlp through ocg_model_create_from_nlp): no folding, no interning.
  // (nodes are still registered for hash-consing, so derivative graphs built
  // on top fold exactly like the reference's)
  void append_raw(const Node& n);
  void append_raw_input(Addr a, const std::string& label) {
    addrs_.push_back(a);
    labels_.push_back(label);
  }

  const std::vector<Node>& nodes() const { return nodes_; }
  const Node& at(int i) const { return nodes_[static_cast<size_t>(i)]; }
  int n_inputs() const { return static_cast<int>(addrs_.size()); }
  const std::vector<Addr>& inputs() const { return addrs_; }
  const std::vector<std::string>& labels() const { return labels_; }
  bool is_const(int n) const { return at(n).op == Op::cnst; }
  bool is_value(int n, double v) const { return at(n).op == Op::cnst && at(n).c == v; }

 private:
  int make(Node n);
  std::vector<Node> nodes_;
  std::vector<Addr> addrs_;
  std::vector<std::string> labels_;
  std::map<std::tuple<int, int, int, std::uint64_t>, int> interned_;
};

struct Kernel {
  Graph graph;
  std::vector<int> roots;
  int out_dim() const { return static_cast<int>(roots.size()); }
};

// jac: (row, input) sorted; hess: (i, j) with i >= j sorted by (j, i);
// dir_ptr[j]..dir_ptr[j+1] delimits direction j.
struct Pattern {
  int out_dim = 0;
  int n_inputs = 0;
  std::vector<std::pair<int, int>> jac;
  std::vector<std::pair<int, int>> hess;
  std::vector<int> dir_ptr;
};

Pattern sparsity_of(const Kernel& k);

// ---------------------------------------------------------------------------
// DSL abstract syntax
// ---------------------------------------------------------------------------

enum class VarKind { state, control, variable };
enum class When { symbolic, initial, final };
enum class Un { neg, sin, cos, tan, exp, log, sqrt };
enum class Bin { add, sub, mul, div, pow };

struct Expr;
using ExprP = std::shared_ptr<const Expr>;

struct Expr {
  enum class K { number, time, ref, unary, binary, vec, integral } k = K::number;
  double value = 0.0;
  int decl = -1, comp = -1;
  When when = When::symbolic;
  Un uop = Un::neg;
  Bin bop = Bin::add;
  ExprP a, b;
  std::vector<ExprP> elems;
  bool is_num() const { return k == K::number; }
};

ExprP num(double v);
ExprP time_expr();
ExprP ref(int decl, int comp, When w);
ExprP unary(Un op, ExprP a);
ExprP binary(Bin op, ExprP a, ExprP b);
ExprP vec(std::vector<ExprP> elems);
ExprP integral(ExprP a);

struct VarDecl {
  std::string name;
  VarKind kind = VarKind::state;
  int dim = 1;
  std::vector<std::string> aliases;
  int line = 0;
};

struct Dyn {
  int decl = -1, comp = 0;
  ExprP rhs;
  int line = 0;
};

struct Con {
  enum class K { boundary, path, box_variable } k = K::path;
  ExprP expr;
  std::vector<double> lo, hi;
  int line = 0;
};

struct Problem {
  std::string time_name;
  double t0 = 0.0, tf = 0.0;
  int t0_var = -1, tf_var = -1;
  std::vector<VarDecl> decls;
  std::vector<Dyn> dynamics;
  std::vector<Con> cons;
  ExprP mayer, lagrange;
  bool maximize = false;

  std::string comp_name(int decl, int comp) const;
};

class ParseError : public std::runtime_error {
 public:
  ParseError(int line, const std::string& msg)
      : std::runtime_error("line " + std::to_string(line) + ": " + msg), line_(line) {}
  int line() const { return line_; }

 private:
  int line_;
};

Problem parse_problem(const std::string& source);

// ---------------------------------------------------------------------------
// Transcribed NLP
// ---------------------------------------------------------------------------

enum class Scheme { euler = 0, trapezoid = 1 };

struct Slab {
  VarKind kind = VarKind::state;
  int dim = 1;
  Index base = 0;
  Index nodes = 1;
};

struct Range {
  Index lo = 0, hi = 0;
  bool endpoints = false;
  Index count() const { return endpoints ? (lo == hi ? 1 : 2) : hi - lo; }
  Index at(Index k) const { return endpoints ? (k == 0 ? lo : hi) : lo + k; }
};

struct Group {
  enum class Kind { dynamics = 0, path = 1, boundary = 2 } kind = Kind::path;
  Kernel kernel;
  Pattern pattern;
  Range range;
  std::vector<double> lower, upper;  // constraint groups only
  Index row_base = 0;                // constraint groups only
  double weight = 1.0;               // objective groups only
  std::string label;
  int out_dim() const { return kernel.out_dim(); }
  Index rows() const { return range.count() * out_dim(); }
};

struct Nlp {
  Scheme scheme = Scheme::trapezoid;
  Index N = 0;
  std::vector<Slab> slabs;
  Index nvar = 0;
  std::vector<Group> cons;  // constraint groups
  std::vector<Group> objs;  // objective groups (single root)
  std::vector<double> lvar, uvar, x_start, clip_lo, clip_hi, lcon, ucon;
  Index m_con = 0;
  bool maximize = false;

  std::string structure_json() const;
};

Nlp transcribe(const Problem& p, Scheme scheme, Index N, bool boxes_as_bounds = false);

}  // namespace ocg
