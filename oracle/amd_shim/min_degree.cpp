// Test infrastructure only (oracle build). Clean-room exact minimum-degree
// ordering behind the amd_l_* entry points declared in amd.h. See amd.h for
// why it exists. Eliminating a vertex turns its live neighbourhood into a
// clique; the next pivot is the live vertex of smallest current degree,
// ties broken by smallest index (a lazy min-heap keyed on (degree, index)).
// As in AMD, rows denser than max(16, control[AMD_DENSE] * sqrt(n)) (a free
// final time coupled to every time step) are left out of the elimination
// graph and ordered last, in index order; control[AMD_DENSE] < 0 keeps them.
#include "amd.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <queue>
#include <vector>

extern "C" void amd_l_defaults(double control[]) {
  for (int i = 0; i < AMD_CONTROL; ++i) control[i] = 0.0;
  control[AMD_DENSE] = 10.0;
  control[AMD_AGGRESSIVE] = 1.0;
}

extern "C" SuiteSparse_long amd_l_order(SuiteSparse_long n, const SuiteSparse_long Ap[],
                                        const SuiteSparse_long Ai[], SuiteSparse_long P[], double* control,
                                        double info[]) {
  using I = std::int64_t;
  if (n < 0) return AMD_INVALID;
  std::vector<std::vector<I>> adj(static_cast<size_t>(n));
  for (I j = 0; j < n; ++j) {
    auto& a = adj[static_cast<size_t>(j)];
    for (I p = Ap[j]; p < Ap[j + 1]; ++p)
      if (Ai[p] != j) a.push_back(Ai[p]);
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
  }
  std::vector<char> dead(static_cast<size_t>(n), 0);
  // dense rows: out of the graph, ordered last
  const double dens = control ? control[AMD_DENSE] : 10.0;
  std::vector<I> dense;
  if (dens >= 0) {
    const double thresh = std::max(16.0, dens * std::sqrt(static_cast<double>(n)));
    std::vector<I> deg(static_cast<size_t>(n), 0);
    for (I j = 0; j < n; ++j)
      for (I u : adj[static_cast<size_t>(j)]) {
        ++deg[static_cast<size_t>(u)];
      }
    for (I v = 0; v < n; ++v)
      if (static_cast<double>(deg[static_cast<size_t>(v)]) > thresh) {
        dense.push_back(v);
        dead[static_cast<size_t>(v)] = 1;
      }
    if (!dense.empty())
      for (I j = 0; j < n; ++j) {
        auto& a = adj[static_cast<size_t>(j)];
        a.erase(std::remove_if(a.begin(), a.end(), [&](I u) { return dead[static_cast<size_t>(u)] != 0; }), a.end());
      }
  }
  using Key = std::pair<I, I>;  // (degree, vertex)
  std::priority_queue<Key, std::vector<Key>, std::greater<Key>> heap;
  for (I v = 0; v < n; ++v)
    if (!dead[static_cast<size_t>(v)]) heap.emplace(static_cast<I>(adj[static_cast<size_t>(v)].size()), v);

  std::vector<I> clique, merged;
  I k = 0;
  while (!heap.empty()) {
    auto [deg, v] = heap.top();
    heap.pop();
    if (dead[static_cast<size_t>(v)] || deg != static_cast<I>(adj[static_cast<size_t>(v)].size())) continue;
    P[k++] = v;
    dead[static_cast<size_t>(v)] = 1;
    clique.clear();
    for (I u : adj[static_cast<size_t>(v)])
      if (!dead[static_cast<size_t>(u)]) clique.push_back(u);
    for (I u : clique) {
      auto& au = adj[static_cast<size_t>(u)];
      merged.clear();
      merged.reserve(au.size() + clique.size());
      std::set_union(au.begin(), au.end(), clique.begin(), clique.end(), std::back_inserter(merged));
      au.clear();
      for (I w : merged)
        if (w != u && w != v && !dead[static_cast<size_t>(w)]) au.push_back(w);
      heap.emplace(static_cast<I>(au.size()), u);
    }
    adj[static_cast<size_t>(v)].clear();
    adj[static_cast<size_t>(v)].shrink_to_fit();
  }
  for (I v : dense) P[k++] = v;
  if (info) info[0] = AMD_OK;
  return AMD_OK;
}
