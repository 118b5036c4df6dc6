// Host side of the reference-order LDL^T (refldl.hpp): the ordering, the
// symbolic analysis and the device plan. O(nnz(L)) after the ordering.
#include "refldl.hpp"

#include <algorithm>
#include <cmath>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>

namespace ocg::rl {

std::vector<int64_t> min_degree_order(int64_t n, const std::vector<int64_t>& Fp, const std::vector<int64_t>& Fi) {
  std::vector<int64_t> order;
  order.reserve(static_cast<size_t>(n));
  if (n <= 0) return order;
  // elimination graph: sorted live neighbour lists
  std::vector<std::vector<int64_t>> nb(static_cast<size_t>(n));
  for (int64_t v = 0; v < n; ++v) {
    auto& a = nb[static_cast<size_t>(v)];
    a.assign(Fi.begin() + Fp[static_cast<size_t>(v)], Fi.begin() + Fp[static_cast<size_t>(v) + 1]);
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
    a.erase(std::remove(a.begin(), a.end(), v), a.end());
  }
  // AMD's dense-row rule (amd_l_defaults: dense = 10): vertices of degree
  // above max(16, 10 sqrt(n)) leave the graph and are ordered last
  std::vector<char> out(static_cast<size_t>(n), 0);
  const double dense_deg = std::max(16.0, 10.0 * std::sqrt(static_cast<double>(n)));
  std::vector<int64_t> dense;
  for (int64_t v = 0; v < n; ++v)
    if (static_cast<double>(nb[static_cast<size_t>(v)].size()) > dense_deg) {
      dense.push_back(v);
      out[static_cast<size_t>(v)] = 1;
    }
  if (!dense.empty())
    for (auto& a : nb) a.erase(std::remove_if(a.begin(), a.end(), [&](int64_t u) { return out[static_cast<size_t>(u)] != 0; }), a.end());

  // live vertices keyed (current degree, index): the next pivot is the minimum
  std::set<std::pair<int64_t, int64_t>> live;
  for (int64_t v = 0; v < n; ++v)
    if (!out[static_cast<size_t>(v)]) live.emplace(static_cast<int64_t>(nb[static_cast<size_t>(v)].size()), v);
  std::vector<int64_t> merged;
  while (!live.empty()) {
    const int64_t v = live.begin()->second;
    live.erase(live.begin());
    order.push_back(v);
    out[static_cast<size_t>(v)] = 1;
    std::vector<int64_t> clique = std::move(nb[static_cast<size_t>(v)]);
    nb[static_cast<size_t>(v)].clear();
    for (int64_t u : clique) {
      auto& a = nb[static_cast<size_t>(u)];
      live.erase({static_cast<int64_t>(a.size()), u});
      merged.clear();
      std::set_union(a.begin(), a.end(), clique.begin(), clique.end(), std::back_inserter(merged));
      a.clear();
      for (int64_t w : merged)
        if (w != u && w != v) a.push_back(w);
      live.emplace(static_cast<int64_t>(a.size()), u);
    }
  }
  for (int64_t v : dense) order.push_back(v);
  return order;
}

Symbolic analyze(int64_t dim, const int64_t* colp, const int64_t* rowi, int64_t n_free, int64_t ntot) {
  Symbolic S;
  S.dim = dim;
  S.ntot = ntot;
  const size_t n = static_cast<size_t>(dim);
  const int64_t nnz = dim > 0 ? colp[dim] : 0;

  // full adjacency, both triangles, diagonal stripped (ldl.cpp:31-52)
  std::vector<int64_t> Fp(n + 1, 0), Fi;
  {
    std::vector<int64_t> cnt(n, 0);
    for (int64_t j = 0; j < dim; ++j)
      for (int64_t p = colp[j]; p < colp[j + 1]; ++p)
        if (rowi[p] != j) {
          ++cnt[static_cast<size_t>(rowi[p])];
          ++cnt[static_cast<size_t>(j)];
        }
    for (size_t j = 0; j < n; ++j) Fp[j + 1] = Fp[j] + cnt[j];
    Fi.resize(static_cast<size_t>(Fp[n]));
    std::vector<int64_t> nx(Fp.begin(), Fp.end() - 1);
    for (int64_t j = 0; j < dim; ++j)
      for (int64_t p = colp[j]; p < colp[j + 1]; ++p)
        if (rowi[p] != j) {
          Fi[static_cast<size_t>(nx[static_cast<size_t>(j)]++)] = rowi[p];
          Fi[static_cast<size_t>(nx[static_cast<size_t>(rowi[p])]++)] = j;
        }
  }
  std::vector<int64_t> perm = min_degree_order(dim, Fp, Fi);

  // pivot_after_ (eval.cpp:409-426): a kept equality row (a dual without a
  // slack entry) whose Jacobian has exactly one free primal column. Lower CSC
  // with row >= col: the dual rows' entries sit in the primal columns.
  std::vector<int64_t> one_col(n, -1);
  std::vector<int> ncols(n, 0);
  std::vector<char> has_slack(n, 0);
  for (int64_t c = 0; c < std::min(ntot, dim); ++c)
    for (int64_t p = colp[c]; p < colp[c + 1]; ++p) {
      const int64_t r = rowi[p];
      if (r < ntot) continue;
      if (c >= n_free) {
        has_slack[static_cast<size_t>(r)] = 1;
      } else if (ncols[static_cast<size_t>(r)] == 0 || one_col[static_cast<size_t>(r)] != c) {
        ++ncols[static_cast<size_t>(r)];
        one_col[static_cast<size_t>(r)] = c;
      }
    }
  // symbolic() (eval.cpp:445-465): duals are chained per column in pivot_after_
  // order (dual ordinal ascending) and emitted last-in first after the column
  std::vector<int64_t> head(n, -1), next(n, -1);
  std::vector<char> deferred(n, 0);
  for (int64_t r = ntot; r < dim; ++r)
    if (!has_slack[static_cast<size_t>(r)] && ncols[static_cast<size_t>(r)] == 1) {
      const int64_t c = one_col[static_cast<size_t>(r)];
      next[static_cast<size_t>(r)] = head[static_cast<size_t>(c)];
      head[static_cast<size_t>(c)] = r;
      deferred[static_cast<size_t>(r)] = 1;
    }
  S.perm.reserve(n);
  for (int64_t v : perm) {
    if (deferred[static_cast<size_t>(v)]) continue;
    S.perm.push_back(v);
    for (int64_t t = head[static_cast<size_t>(v)]; t >= 0; t = next[static_cast<size_t>(t)]) S.perm.push_back(t);
  }
  if (static_cast<int64_t>(S.perm.size()) != dim) throw std::runtime_error("refldl: ordering lost indices");
  S.iperm.assign(n, 0);
  for (size_t k = 0; k < n; ++k) S.iperm[static_cast<size_t>(S.perm[k])] = static_cast<int64_t>(k);

  // permuted upper pattern by column (analyze_ordered, ldl.cpp:85-104)
  std::vector<int64_t> Up(n + 1, 0), Ui(static_cast<size_t>(nnz));
  {
    std::vector<int64_t> cnt(n, 0);
    for (int64_t j = 0; j < dim; ++j)
      for (int64_t p = colp[j]; p < colp[j + 1]; ++p)
        ++cnt[static_cast<size_t>(std::max(S.iperm[static_cast<size_t>(rowi[p])], S.iperm[static_cast<size_t>(j)]))];
    for (size_t j = 0; j < n; ++j) Up[j + 1] = Up[j] + cnt[j];
    std::vector<int64_t> nx(Up.begin(), Up.end() - 1);
    for (int64_t j = 0; j < dim; ++j)
      for (int64_t p = colp[j]; p < colp[j + 1]; ++p) {
        const int64_t a = S.iperm[static_cast<size_t>(rowi[p])], b = S.iperm[static_cast<size_t>(j)];
        Ui[static_cast<size_t>(nx[static_cast<size_t>(std::max(a, b))]++)] = std::min(a, b);
      }
  }
  // elimination tree and pattern of L: row k of L is the union of the etree
  // paths from the entries of column k of the upper pattern up to k; each
  // row index is appended to its columns in increasing k (ascending rows)
  S.parent.assign(n, -1);
  std::vector<int64_t> flag(n, -1), cnt(n, 0);
  for (int pass = 0; pass < 2; ++pass) {
    std::fill(flag.begin(), flag.end(), -1);
    std::vector<int64_t> fill;
    if (pass == 1) {
      S.Lp.assign(n + 1, 0);
      for (size_t j = 0; j < n; ++j) S.Lp[j + 1] = S.Lp[j] + cnt[j];
      S.Li.resize(static_cast<size_t>(S.Lp[n]));
      fill.assign(S.Lp.begin(), S.Lp.end() - 1);
    }
    for (int64_t k = 0; k < dim; ++k) {
      flag[static_cast<size_t>(k)] = k;
      for (int64_t p = Up[static_cast<size_t>(k)]; p < Up[static_cast<size_t>(k) + 1]; ++p)
        for (int64_t i = Ui[static_cast<size_t>(p)]; flag[static_cast<size_t>(i)] != k; i = S.parent[static_cast<size_t>(i)]) {
          if (pass == 0) {
            if (S.parent[static_cast<size_t>(i)] < 0) S.parent[static_cast<size_t>(i)] = k;
            ++cnt[static_cast<size_t>(i)];
          } else {
            S.Li[static_cast<size_t>(fill[static_cast<size_t>(i)]++)] = k;
          }
          flag[static_cast<size_t>(i)] = k;
        }
    }
  }
  return S;
}

HostPlan build_plan(const Symbolic& S, const int64_t* colp, const int64_t* rowi) {
  HostPlan H;
  const int64_t dim = S.dim;
  const size_t n = static_cast<size_t>(dim);
  H.dim = dim;
  H.nnz = dim > 0 ? colp[dim] : 0;
  H.lnz = static_cast<int64_t>(S.Li.size());
  auto cc = [&](int64_t k) { return S.Lp[static_cast<size_t>(k) + 1] - S.Lp[static_cast<size_t>(k)]; };

  std::vector<char> has_child(n, 0);
  for (size_t k = 0; k < n; ++k)
    if (S.parent[k] >= 0) has_child[static_cast<size_t>(S.parent[k])] = 1;
  std::vector<int64_t> jidx(n, -1), lidx(n, -1);
  for (int64_t k = 0; k < dim; ++k) {
    const int64_t f = 1 + cc(k);
    if (f > kMaxFront)
      throw std::runtime_error("reference-order LDL: front of " + std::to_string(f) + " rows exceeds " +
                               std::to_string(kMaxFront));
    H.fmax = std::max<int>(H.fmax, static_cast<int>(f));
    if (has_child[static_cast<size_t>(k)]) {
      jidx[static_cast<size_t>(k)] = static_cast<int64_t>(H.nl_pos.size());
      H.nl_pos.push_back(k);
      H.nl_lp.push_back(S.Lp[static_cast<size_t>(k)]);
      H.nl_f.push_back(static_cast<int32_t>(f));
    } else {
      lidx[static_cast<size_t>(k)] = static_cast<int64_t>(H.lf_pos.size());
      H.lf_pos.push_back(k);
      H.lf_f.push_back(static_cast<int32_t>(f));
    }
  }
  const int64_t nnl = static_cast<int64_t>(H.nl_pos.size());

  // rel: where each row of column k sits in its parent's front [p, struct(p)]
  H.rel.assign(static_cast<size_t>(H.lnz), 0);
  for (int64_t k = 0; k < dim; ++k) {
    const int64_t p = S.parent[static_cast<size_t>(k)];
    if (p < 0) continue;
    int64_t q = S.Lp[static_cast<size_t>(p)];
    const int64_t qe = S.Lp[static_cast<size_t>(p) + 1];
    for (int64_t t = S.Lp[static_cast<size_t>(k)]; t < S.Lp[static_cast<size_t>(k) + 1]; ++t) {
      const int64_t r = S.Li[static_cast<size_t>(t)];
      if (r == p) {
        H.rel[static_cast<size_t>(t)] = 0;
        continue;
      }
      while (q < qe && S.Li[static_cast<size_t>(q)] < r) ++q;
      if (q == qe || S.Li[static_cast<size_t>(q)] != r) throw std::runtime_error("refldl: column pattern not nested in its parent's");
      H.rel[static_cast<size_t>(t)] = static_cast<int32_t>(1 + q - S.Lp[static_cast<size_t>(p)]);
    }
  }

  // W = [chain fronts (packed lower f(f+1)/2, then f diagonal maxima) | leaf A columns (f)]
  H.nl_foff.resize(static_cast<size_t>(nnl));
  H.nl_voff.resize(static_cast<size_t>(nnl));
  H.nl_soff.resize(static_cast<size_t>(nnl));
  int64_t w = 0, v = 0, st = 0;
  for (int64_t j = 0; j < nnl; ++j) {
    const int64_t f = H.nl_f[static_cast<size_t>(j)];
    H.nl_foff[static_cast<size_t>(j)] = w;
    const int64_t sz = f * (f + 1) / 2 + f;
    w += sz + (sz & 1);  // fronts start on 16 bytes: chunks of them stream by bulk copies
    H.nl_voff[static_cast<size_t>(j)] = v;
    v += f;
    const int64_t p = S.parent[static_cast<size_t>(H.nl_pos[static_cast<size_t>(j)])];
    if (p < 0) {
      H.nl_soff[static_cast<size_t>(j)] = kRoot;
    } else if (j + 1 < nnl && H.nl_pos[static_cast<size_t>(j) + 1] == p) {
      H.nl_soff[static_cast<size_t>(j)] = kChain;
    } else {
      H.nl_soff[static_cast<size_t>(j)] = st;
      st += (f - 1) * f / 2 + (f - 1);
    }
  }
  H.fronts_len = w;
  H.lf_aoff.resize(H.lf_pos.size());
  for (size_t i = 0; i < H.lf_pos.size(); ++i) {
    H.lf_aoff[i] = w;
    w += H.lf_f[i];
  }
  H.w_len = std::max<int64_t>(w, 1);
  H.v_len = std::max<int64_t>(v, 1);
  H.stash_len = std::max<int64_t>(st, 1);

  // stashed children of every chain column (chain indices ascending)
  {
    std::vector<std::vector<int32_t>> kids(static_cast<size_t>(nnl));
    for (int64_t j = 0; j < nnl; ++j)
      if (H.nl_soff[static_cast<size_t>(j)] >= 0)
        kids[static_cast<size_t>(jidx[static_cast<size_t>(S.parent[static_cast<size_t>(H.nl_pos[static_cast<size_t>(j)])])])]
            .push_back(static_cast<int32_t>(j));
    H.sc_ptr.assign(static_cast<size_t>(nnl) + 1, 0);
    for (int64_t j = 0; j < nnl; ++j) {
      H.sc_ptr[static_cast<size_t>(j) + 1] = H.sc_ptr[static_cast<size_t>(j)] + static_cast<int64_t>(kids[static_cast<size_t>(j)].size());
      H.sc_child.insert(H.sc_child.end(), kids[static_cast<size_t>(j)].begin(), kids[static_cast<size_t>(j)].end());
    }
  }
  // leaf update matrices pre-assembled into their parents (leaves ascending)
  {
    std::vector<std::vector<int32_t>> kids(static_cast<size_t>(nnl));
    for (size_t i = 0; i < H.lf_pos.size(); ++i) {
      const int64_t p = S.parent[static_cast<size_t>(H.lf_pos[i])];
      if (p >= 0) kids[static_cast<size_t>(jidx[static_cast<size_t>(p)])].push_back(static_cast<int32_t>(i));
    }
    H.pa_ptr.push_back(0);
    for (int64_t j = 0; j < nnl; ++j) {
      if (kids[static_cast<size_t>(j)].empty()) continue;
      H.pa_j.push_back(static_cast<int32_t>(j));
      H.pa_leaf.insert(H.pa_leaf.end(), kids[static_cast<size_t>(j)].begin(), kids[static_cast<size_t>(j)].end());
      H.pa_ptr.push_back(static_cast<int64_t>(H.pa_leaf.size()));
    }
  }
  // forward solve: leaf terms of every chain row, leaf columns ascending
  {
    std::vector<std::vector<std::pair<int64_t, int64_t>>> terms(static_cast<size_t>(nnl));
    for (size_t i = 0; i < H.lf_pos.size(); ++i) {
      const int64_t c = H.lf_pos[i];
      for (int64_t t = S.Lp[static_cast<size_t>(c)]; t < S.Lp[static_cast<size_t>(c) + 1]; ++t)
        terms[static_cast<size_t>(jidx[static_cast<size_t>(S.Li[static_cast<size_t>(t)])])].emplace_back(t, c);
    }
    H.fl_ptr.push_back(0);
    H.fl_all_ptr.assign(static_cast<size_t>(nnl) + 1, 0);
    for (int64_t j = 0; j < nnl; ++j) {
      H.fl_all_ptr[static_cast<size_t>(j) + 1] =
          H.fl_all_ptr[static_cast<size_t>(j)] + static_cast<int64_t>(terms[static_cast<size_t>(j)].size());
      if (static_cast<int64_t>(terms[static_cast<size_t>(j)].size()) > kPreLong) H.pre_long.push_back(static_cast<int32_t>(j));
      if (terms[static_cast<size_t>(j)].empty()) continue;
      H.fl_j.push_back(static_cast<int32_t>(j));
      for (const auto& [t, c] : terms[static_cast<size_t>(j)]) {
        H.fl_lx.push_back(t);
        H.fl_col.push_back(c);
      }
      H.fl_ptr.push_back(static_cast<int64_t>(H.fl_lx.size()));
    }
  }
  // K entry -> W
  H.sc_dst.resize(static_cast<size_t>(H.nnz));
  H.sc_dpos.assign(static_cast<size_t>(H.nnz), -1);
  H.sc_ms.assign(static_cast<size_t>(H.nnz), -1);
  for (int64_t col = 0; col < dim; ++col)
    for (int64_t p = colp[col]; p < colp[col + 1]; ++p) {
      const int64_t a = S.iperm[static_cast<size_t>(rowi[p])], b = S.iperm[static_cast<size_t>(col)];
      const int64_t lo = std::min(a, b), hi = std::max(a, b);
      int64_t r = 0;
      if (hi != lo) {
        const auto beg = S.Li.begin() + S.Lp[static_cast<size_t>(lo)], end = S.Li.begin() + S.Lp[static_cast<size_t>(lo) + 1];
        const auto it = std::lower_bound(beg, end, hi);
        if (it == end || *it != hi) throw std::runtime_error("refldl: entry outside the pattern of L");
        r = 1 + (it - beg);
      } else {
        H.sc_dpos[static_cast<size_t>(p)] = lo;
      }
      const int64_t j = jidx[static_cast<size_t>(lo)];
      if (j >= 0) {
        const int64_t fo = H.nl_foff[static_cast<size_t>(j)], f = H.nl_f[static_cast<size_t>(j)];
        H.sc_dst[static_cast<size_t>(p)] = fo + r * (r + 1) / 2;
        if (hi == lo) H.sc_ms[static_cast<size_t>(p)] = fo + f * (f + 1) / 2;
      } else {
        H.sc_dst[static_cast<size_t>(p)] = H.lf_aoff[static_cast<size_t>(lidx[static_cast<size_t>(lo)])] + r;
      }
    }
  // packed per-column records of the warp walks (32-bit fields)
  if (H.lnz >= (int64_t{1} << 31) || dim >= (int64_t{1} << 31) || H.stash_len >= (int64_t{1} << 31))
    throw std::runtime_error("reference-order LDL: factor too large for the 32-bit column records");
  H.rec.resize(static_cast<size_t>(nnl));
  for (int64_t j = 0; j < nnl; ++j) {
    ColRec& r = H.rec[static_cast<size_t>(j)];
    r.foff = H.nl_foff[static_cast<size_t>(j)];
    r.lp = static_cast<int>(H.nl_lp[static_cast<size_t>(j)]);
    r.pos = static_cast<int>(H.nl_pos[static_cast<size_t>(j)]);
    r.f = static_cast<short>(H.nl_f[static_cast<size_t>(j)]);
    r.flags = 0;
    r.soff = static_cast<int>(H.nl_soff[static_cast<size_t>(j)]);
    r.sc0 = static_cast<int>(H.sc_ptr[static_cast<size_t>(j)]);
    r.sc1 = static_cast<int>(H.sc_ptr[static_cast<size_t>(j) + 1]);
    r.inv8 = 0;
    r.rel8 = 0;
    if (r.f <= 8)
      for (int a = 1; a < r.f; ++a)
        r.rel8 |= static_cast<unsigned long long>(H.rel[static_cast<size_t>(r.lp + a - 1)]) << (8 * (a - 1));
    if (r.soff == kChain && r.f <= 8 && H.nl_f[static_cast<size_t>(j) + 1] <= 8)
      for (int a = 1; a < r.f; ++a) {
        const int dst = H.rel[static_cast<size_t>(r.lp + a - 1)];
        r.inv8 |= static_cast<unsigned long long>(a) << (8 * dst);
      }
    if (r.soff == kChain && r.inv8 != 0 && H.sc_ptr[static_cast<size_t>(j) + 1] == H.sc_ptr[static_cast<size_t>(j) + 2])
      r.flags |= 1;
  }
  for (int64_t j = 0; j < nnl; j += 16) H.chunk_foff.push_back(H.nl_foff[static_cast<size_t>(j)]);
  H.chunk_foff.push_back(H.fronts_len);
  H.primal.resize(n);
  for (size_t k = 0; k < n; ++k) H.primal[k] = S.perm[k] < S.ntot ? 1 : 0;
  return H;
}

}  // namespace ocg::rl
