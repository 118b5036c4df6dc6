// Node-range shards over several GPUs: the shard plan, the communicator
// (NCCL loaded at run time, or host callbacks) and the C ABI of shard.hpp.
#include "shard.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>

#include "handles.hpp"

namespace ocg {

namespace {

// slab of a slot, node within it
struct SlotLoc {
  int slab = -1;
  Index node = 0;
};
SlotLoc locate(const Nlp& nlp, Index slot) {
  for (size_t s = 0; s < nlp.slabs.size(); ++s) {
    const Slab& sl = nlp.slabs[s];
    if (slot >= sl.base && slot < sl.base + sl.dim * sl.nodes) return {static_cast<int>(s), (slot - sl.base) / sl.dim};
  }
  return {};
}

// main grid range of rank q: boundaries on the objective's chunk grid (the
// first node-indexed objective group's first index + multiples of 512)
Index chunk_origin(const Nlp& nlp, const Layout& L) {
  for (const Group& g : nlp.objs)
    if (!g.range.endpoints && g.range.lo >= L.idx_lo && g.range.lo < L.idx_hi) return g.range.lo;
  return L.idx_lo;
}
std::pair<Index, Index> rank_range(const Layout& L, Index origin, int q, int world) {
  const Index n = L.idx_hi - L.idx_lo;
  const Index per = ((n + world - 1) / world + 511) / 512 * 512;
  auto cut = [&](int k) {  // boundary k of world+1, clamped into the grid
    if (k <= 0) return L.idx_lo;
    if (k >= world) return L.idx_hi;
    return std::clamp(origin + per * k, L.idx_lo, L.idx_hi);
  };
  return {cut(q), cut(q + 1)};
}

}  // namespace

ShardPlan make_shard_plan(const Nlp& nlp, const Layout& L, int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world) throw std::runtime_error("shard plan: bad rank / world");
  ShardPlan P;
  P.rank = rank;
  P.world = world;
  const Index origin = chunk_origin(nlp, L);
  auto rank_range = [&](const Layout& LL, int q, int w) { return ocg::rank_range(LL, origin, q, w); };
  std::tie(P.lo, P.hi) = rank_range(L, rank, world);
  P.specials = rank == 0;
  // node n of a time slab is owned by the rank whose index range holds n
  // (nodes before the grid by rank 0, after it by the last rank)
  auto own = [&](int q, Index nodes) {
    auto [a, b] = rank_range(L, q, world);
    if (q == 0) a = 0;
    if (q == world - 1) b = nodes;
    return std::pair<Index, Index>{std::max<Index>(0, a), std::min(nodes, std::max(a, b))};
  };
  auto owner = [&](Index n, Index nodes) {
    for (int q = 0; q < world; ++q) {
      const auto [a, b] = own(q, nodes);
      if (n >= a && n < b) return q;
    }
    return world - 1;
  };
  // what each rank reads: per time slab a contiguous run of nodes (its main
  // instances; the ends of each input's run bound it) plus isolated nodes
  // (endpoint instances on rank 0)
  const size_t ns = nlp.slabs.size();
  struct Need {
    std::vector<std::pair<Index, Index>> run;  // [lo, hi] per slab, lo > hi = none
    std::set<std::pair<int, Index>> iso;
  };
  std::vector<Need> need(static_cast<size_t>(world));
  for (int q = 0; q < world; ++q) {
    const auto [lo, hi] = rank_range(L, q, world);
    Need& nd = need[static_cast<size_t>(q)];
    nd.run.assign(ns, {1, 0});
    auto slot_of = [&](Index slot) {
      const SlotLoc p = locate(nlp, slot);
      if (p.slab < 0) throw std::runtime_error("shard plan: an input outside the variable slabs");
      return p;
    };
    for (const auto* gs : {&nlp.cons, &nlp.objs})
      for (const Group& g : *gs) {
        if (g.range.endpoints) {
          if (q != 0) continue;
          for (Index k = 0; k < g.range.count(); ++k)
            for (const Addr& ad : g.kernel.graph.inputs()) {
              const SlotLoc p = slot_of(ad.slot(g.range.at(k)));
              if (nlp.slabs[static_cast<size_t>(p.slab)].nodes > 1) nd.iso.emplace(p.slab, p.node);
            }
          continue;
        }
        const Index a = std::max(lo, g.range.lo), b = std::min(hi, g.range.hi);
        if (a >= b) continue;
        for (const Addr& ad : g.kernel.graph.inputs()) {
          const SlotLoc p0 = slot_of(ad.slot(a)), p1 = slot_of(ad.slot(b - 1));
          if (nlp.slabs[static_cast<size_t>(p0.slab)].nodes == 1) continue;
          if (ad.stride == 0) {  // an absolute node (e.g. x(N) in a path group): isolated
            nd.iso.emplace(p0.slab, p0.node);
            continue;
          }
          auto& r = nd.run[static_cast<size_t>(p0.slab)];
          const Index n0 = std::min(p0.node, p1.node), n1 = std::max(p0.node, p1.node);
          r = r.first > r.second ? std::pair<Index, Index>{n0, n1}
                                 : std::pair<Index, Index>{std::min(r.first, n0), std::max(r.second, n1)};
        }
      }
  }
  // uploads: the owned nodes of every time slab and the free variables
  for (size_t s = 0; s < ns; ++s) {
    const Slab& sl = nlp.slabs[s];
    if (sl.nodes == 1) {
      P.x_own.push_back({sl.base, sl.dim});
      continue;
    }
    const auto [a, b] = own(rank, sl.nodes);
    if (a < b) P.x_own.push_back({sl.base + a * sl.dim, (b - a) * sl.dim});
  }
  // exchange: the nodes a rank reads but does not own, from their owners, in
  // (slab, node) order on both sides
  P.send_to.assign(static_cast<size_t>(world), {});
  P.recv_from.assign(static_cast<size_t>(world), {});
  for (int q = 0; q < world; ++q) {
    std::set<std::pair<int, Index>> foreign;
    const Need& nd = need[static_cast<size_t>(q)];
    for (size_t s = 0; s < ns; ++s) {
      const Index nodes = nlp.slabs[s].nodes;
      if (nodes == 1) continue;
      const auto [r0, r1] = nd.run[s];
      if (r0 > r1) continue;
      const auto [a, b] = own(q, nodes);
      for (Index n = r0; n <= r1 && n < a; ++n) foreign.emplace(static_cast<int>(s), n);
      for (Index n = std::max(r0, b); n <= r1; ++n) foreign.emplace(static_cast<int>(s), n);
    }
    for (const auto& [s, n] : nd.iso) {
      const auto [a, b] = own(q, nlp.slabs[static_cast<size_t>(s)].nodes);
      if (n < a || n >= b) foreign.emplace(s, n);
    }
    for (const auto& [s, n] : foreign) {
      const Slab& sl = nlp.slabs[static_cast<size_t>(s)];
      const int o = owner(n, sl.nodes);
      const Run r{sl.base + n * sl.dim, sl.dim};
      if (q == rank) {
        P.recv_from[static_cast<size_t>(o)].push_back(r);
        P.halo_doubles += r.len;
      }
      if (o == rank) P.send_to[static_cast<size_t>(q)].push_back(r);
    }
  }
  // constraint rows of this rank's instances (lambda, row_scale)
  for (const Group& g : nlp.cons) {
    const Index od = g.out_dim();
    if (g.range.endpoints) {
      if (P.specials && g.rows() > 0) P.rows.push_back({g.row_base, g.rows()});
      continue;
    }
    const Index a = std::max(P.lo, g.range.lo), b = std::min(P.hi, g.range.hi);
    if (a < b) P.rows.push_back({g.row_base + (a - g.range.lo) * od, (b - a) * od});
  }
  // objective chunks (512 instances of a group, reference par_reduce order)
  for (const Group& g : nlp.objs) {
    const Index cnt = g.range.count();
    for (Index c = 0; c * 512 < cnt; ++c) {
      if (g.range.endpoints) {
        P.chunk_owned.push_back(P.specials ? 1 : 0);
        continue;
      }
      const Index a = g.range.lo + 512 * c, b = std::min(g.range.hi, a + 512);
      const bool inside = a >= P.lo && b <= P.hi;
      if (!inside && std::max(a, P.lo) < std::min(b, P.hi)) P.objective_exact = false;  // straddles two ranks
      P.chunk_owned.push_back(inside ? 1 : 0);
    }
  }
  return P;
}

}  // namespace ocg

// ---------------------------------------------------------------------------
// NCCL, loaded at run time (torch's copy when it is already in the process)
// ---------------------------------------------------------------------------

namespace {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static std::once_flag once;
  static Nccl n;
  static std::string why;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (n.h) break;
    }
    if (!n.h) {
      why = dlerror() ? dlerror() : "libnccl.so.2 not found";
      return;
    }
    auto sym = [](const char* s) {
      void* p = dlsym(n.h, s);
      if (!p) throw std::runtime_error(std::string("NCCL symbol missing: ") + s);
      return p;
    };
    try {
      n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
      n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
      n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
      n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
      n.Send = reinterpret_cast<decltype(n.Send)>(sym("ncclSend"));
      n.Recv = reinterpret_cast<decltype(n.Recv)>(sym("ncclRecv"));
      n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
      n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
      n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
    } catch (const std::exception& ex) {
      why = ex.what();
      n.h = nullptr;
    }
  });
  if (!n.h) throw std::runtime_error("NCCL unavailable: " + why);
  return n;
}

void ckn(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + nccl().GetErrorString(r));
}
void ckc(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw ocg::hd::CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
void ckh(int rc, const char* what) {
  if (rc != 0) throw std::runtime_error(std::string("communicator callback failed: ") + what);
}
cudaStream_t st(ocg_stream s) { return static_cast<cudaStream_t>(s); }

int fail(int code, const std::string& msg) { return ocg::hd::set_error(code, msg); }

// exchange the plan's node runs into x_dev (device)
void exchange(ocg_comm* c, const ocg::ShardPlan& P, double* x, cudaStream_t s) {
  const int W = P.world, q = P.rank;
  if (W == 1) return;
  if (c->nccl) {
    const Nccl& n = nccl();
    auto comm = static_cast<ncclComm_t>(c->nccl);
    ckn(n.GroupStart(), "ncclGroupStart");
    for (int p = 0; p < W; ++p) {
      if (p == q) continue;
      for (const ocg::Run& r : P.send_to[static_cast<size_t>(p)])
        ckn(n.Send(x + r.off, static_cast<size_t>(r.len), ncclFloat64, p, comm, s), "ncclSend");
      for (const ocg::Run& r : P.recv_from[static_cast<size_t>(p)])
        ckn(n.Recv(x + r.off, static_cast<size_t>(r.len), ncclFloat64, p, comm, s), "ncclRecv");
    }
    ckn(n.GroupEnd(), "ncclGroupEnd");
    return;
  }
  // host callbacks: round d sends to q+d and receives from q-d (both sides agree)
  for (int d = 1; d < W; ++d) {
    const int to = (q + d) % W, from = (q - d + W) % W;
    const auto& sr = P.send_to[static_cast<size_t>(to)];
    const auto& rr = P.recv_from[static_cast<size_t>(from)];
    Index ns = 0, nr = 0;
    for (const auto& r : sr) ns += r.len;
    for (const auto& r : rr) nr += r.len;
    if (ns == 0 && nr == 0) continue;
    c->hbuf_send.resize(static_cast<size_t>(ns));
    c->hbuf_recv.resize(static_cast<size_t>(nr));
    Index o = 0;
    for (const auto& r : sr) {
      ckc(cudaMemcpyAsync(c->hbuf_send.data() + o, x + r.off, static_cast<size_t>(r.len) * sizeof(double),
                          cudaMemcpyDeviceToHost, s),
          "halo d2h");
      o += r.len;
    }
    ckc(cudaStreamSynchronize(s), "sync");
    ckh(c->fns.sendrecv_f64(c->fns.ctx, c->hbuf_send.data(), ns, to, c->hbuf_recv.data(), nr, from), "sendrecv");
    o = 0;
    for (const auto& r : rr) {
      ckc(cudaMemcpyAsync(x + r.off, c->hbuf_recv.data() + o, static_cast<size_t>(r.len) * sizeof(double),
                          cudaMemcpyHostToDevice, s),
          "halo h2d");
      o += r.len;
    }
    ckc(cudaStreamSynchronize(s), "sync");  // hbuf_recv is reused
  }
}

}  // namespace

extern "C" {

int ocg_comm_nccl_unique_id(unsigned char id[128]) {
  if (!id) return fail(OCG_ERR_ARG, "null argument");
  try {
    ncclUniqueId u;
    ckn(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    static_assert(sizeof(u.internal) == 128, "ncclUniqueId");
    std::memcpy(id, u.internal, 128);
    return OCG_OK;
  } catch (const std::exception& ex) {
    return fail(OCG_ERR_CUDA, ex.what());
  }
}

int ocg_comm_create_nccl(const unsigned char id[128], int rank, int world, int device, ocg_comm** out) {
  if (!id || !out || world < 1 || rank < 0 || rank >= world) return fail(OCG_ERR_ARG, "ocg_comm_create_nccl: bad arguments");
  try {
    ocg::mem::DeviceScope ds(device);
    ckc(cudaSetDevice(device), "cudaSetDevice");
    ncclUniqueId u;
    std::memcpy(u.internal, id, 128);
    ncclComm_t comm = nullptr;
    ckn(nccl().CommInitRank(&comm, world, u, rank), "ncclCommInitRank");
    auto c = std::make_unique<ocg_comm>();
    c->rank = rank;
    c->world = world;
    c->device = device;
    c->nccl = comm;
    *out = c.release();
    return OCG_OK;
  } catch (const std::exception& ex) {
    return fail(OCG_ERR_CUDA, ex.what());
  }
}

int ocg_comm_create_host(const ocg_comm_host_fns* fns, int rank, int world, int device, ocg_comm** out) {
  if (!fns || !out || world < 1 || rank < 0 || rank >= world || !fns->allreduce_sum_f64 || !fns->allreduce_max_i32 ||
      !fns->sendrecv_f64)
    return fail(OCG_ERR_ARG, "ocg_comm_create_host: bad arguments");
  auto c = std::make_unique<ocg_comm>();
  c->rank = rank;
  c->world = world;
  c->device = device;
  c->fns = *fns;
  *out = c.release();
  return OCG_OK;
}

void ocg_comm_destroy(ocg_comm* c) {
  if (!c) return;
  if (c->nccl) {
    try {
      nccl().CommDestroy(static_cast<ncclComm_t>(c->nccl));
    } catch (...) {
    }
  }
  delete c;
}

int ocg_eval_create_sharded(const ocg_model* m, const ocg_eval_options* opts, ocg_comm* comm, ocg_eval** out) {
  if (!m || !comm || !out) return fail(OCG_ERR_ARG, "ocg_eval_create_sharded: null argument");
  try {
    const ocg::Layout L = ocg::make_layout(m->nlp);
    auto plan = std::make_shared<ocg::ShardPlan>(ocg::make_shard_plan(m->nlp, L, comm->rank, comm->world));
    ocg_eval_options o;
    ocg_eval_default_options(&o);
    if (opts) o = *opts;
    o.device = comm->device;
    o.idx_lo = plan->lo;
    o.idx_hi = plan->hi;
    o.specials = plan->specials ? 1 : 0;
    ocg_eval* e = nullptr;
    const int rc = ocg_eval_create(m, &o, &e);
    if (rc != OCG_OK) return rc;
    e->comm = comm;
    e->shard = plan;
    *out = e;
    return OCG_OK;
  } catch (const std::exception& ex) {
    return fail(OCG_ERR_ARG, std::string("ocg_eval_create_sharded: ") + ex.what());
  }
}

int ocg_eval_shard(const ocg_eval* e, int64_t* out) {
  if (!e || !out) return fail(OCG_ERR_ARG, "null argument");
  if (!e->shard) {
    out[0] = e->i0;
    out[1] = e->i0 + e->n_main;
    out[2] = e->specials ? 1 : 0;
    out[3] = 0;
    out[4] = 1;
    out[5] = 0;
    return OCG_OK;
  }
  const auto& P = *e->shard;
  out[0] = P.lo;
  out[1] = P.hi;
  out[2] = P.specials ? 1 : 0;
  out[3] = P.rank;
  out[4] = P.world;
  out[5] = P.halo_doubles;
  return OCG_OK;
}

int ocg_eval_halo_exchange(ocg_eval* e, double* x_dev, ocg_stream s) {
  if (!e || !x_dev) return fail(OCG_ERR_ARG, "null argument");
  if (!e->shard) return OCG_OK;
  try {
    ocg::mem::DeviceScope ds(e->device);
    exchange(e->comm, *e->shard, x_dev, st(s));
    return OCG_OK;
  } catch (const ocg::hd::CudaError& ex) {
    return fail(OCG_ERR_CUDA, ex.what());
  } catch (const std::exception& ex) {
    return fail(OCG_ERR_CUDA, ex.what());
  }
}

int ocg_eval_scatter_x(ocg_eval* e, const double* x_host, double* x_dev, int64_t* h2d_bytes, ocg_stream s) {
  if (!e || !x_host || !x_dev) return fail(OCG_ERR_ARG, "null argument");
  try {
    ocg::mem::DeviceScope ds(e->device);
    int64_t bytes = 0;
    if (!e->shard) {
      const size_t n = static_cast<size_t>(e->model->nlp.nvar);
      ckc(cudaMemcpyAsync(x_dev, x_host, n * sizeof(double), cudaMemcpyHostToDevice, st(s)), "x h2d");
      bytes = static_cast<int64_t>(n * sizeof(double));
    } else {
      for (const ocg::Run& r : e->shard->x_own) {
        ckc(cudaMemcpyAsync(x_dev + r.off, x_host + r.off, static_cast<size_t>(r.len) * sizeof(double),
                            cudaMemcpyHostToDevice, st(s)),
            "x h2d");
        bytes += r.len * static_cast<int64_t>(sizeof(double));
      }
      exchange(e->comm, *e->shard, x_dev, st(s));
    }
    if (h2d_bytes) *h2d_bytes = bytes;
    return OCG_OK;
  } catch (const std::exception& ex) {
    return fail(OCG_ERR_CUDA, ex.what());
  }
}

int ocg_eval_scatter_rows(ocg_eval* e, const double* lam_host, double* lam_dev, int64_t* h2d_bytes, ocg_stream s) {
  if (!e || !lam_host || !lam_dev) return fail(OCG_ERR_ARG, "null argument");
  try {
    ocg::mem::DeviceScope ds(e->device);
    int64_t bytes = 0;
    std::vector<ocg::Run> all{{0, e->model->nlp.m_con}};
    for (const ocg::Run& r : e->shard ? e->shard->rows : all) {
      if (r.len <= 0) continue;
      ckc(cudaMemcpyAsync(lam_dev + r.off, lam_host + r.off, static_cast<size_t>(r.len) * sizeof(double),
                          cudaMemcpyHostToDevice, st(s)),
          "rows h2d");
      bytes += r.len * static_cast<int64_t>(sizeof(double));
    }
    if (h2d_bytes) *h2d_bytes = bytes;
    return OCG_OK;
  } catch (const std::exception& ex) {
    return fail(OCG_ERR_CUDA, ex.what());
  }
}

int ocg_eval_status_all(ocg_eval* e, ocg_stream s) {
  if (!e) return fail(OCG_ERR_ARG, "null eval");
  if (!e->shard || e->shard->world == 1) return ocg_eval_status(e, s);
  try {
    ocg::mem::DeviceScope ds(e->device);
    int32_t h = 0;
    if (e->comm->nccl) {
      ckn(nccl().AllReduce(e->flag.p, e->flag.p, 1, ncclInt32, ncclMax, static_cast<ncclComm_t>(e->comm->nccl),
                           st(s)),
          "ncclAllReduce(flag)");
      ckc(cudaMemcpyAsync(&h, e->flag.p, sizeof(int), cudaMemcpyDeviceToHost, st(s)), "flag d2h");
      ckc(cudaStreamSynchronize(st(s)), "sync");
    } else {
      ckc(cudaMemcpyAsync(&h, e->flag.p, sizeof(int), cudaMemcpyDeviceToHost, st(s)), "flag d2h");
      ckc(cudaStreamSynchronize(st(s)), "sync");
      h = h ? 1 : 0;
      ckh(e->comm->fns.allreduce_max_i32(e->comm->fns.ctx, &h, 1), "allreduce_max_i32");
    }
    if (h) {
      ckc(cudaMemsetAsync(e->flag.p, 0, sizeof(int), st(s)), "flag reset");
      ckc(cudaStreamSynchronize(st(s)), "sync");
      return OCG_EVAL_DOMAIN;
    }
    return OCG_OK;
  } catch (const std::exception& ex) {
    return fail(OCG_ERR_CUDA, ex.what());
  }
}

int ocg_eval_objective_all(ocg_eval* e, const double* x_dev, double* f, ocg_stream s) {
  if (!e || !x_dev || !f) return fail(OCG_ERR_ARG, "null argument");
  try {
    ocg::mem::DeviceScope ds(e->device);
    const size_t nc = static_cast<size_t>(e->n_chunks);
    int rc = ocg_eval_objective_partials(e, x_dev, e->partials.p, s);
    if (rc < 0) return rc;
    if (e->shard && e->shard->world > 1) {
      if (!e->shard->objective_exact)
        return fail(OCG_ERR_STATE,
                    "ocg_eval_objective_all: an objective chunk straddles two ranks (objective groups on different "
                    "512-chunk grids)");
      std::vector<double> h(nc);
      if (nc) ckc(cudaMemcpyAsync(h.data(), e->partials.p, nc * sizeof(double), cudaMemcpyDeviceToHost, st(s)), "d2h");
      ckc(cudaStreamSynchronize(st(s)), "sync");
      for (size_t c = 0; c < nc; ++c)
        if (!e->shard->chunk_owned[c]) h[c] = 0.0;  // a SUM then has one nonzero term per chunk: exact
      if (e->comm->nccl) {
        if (nc) ckc(cudaMemcpyAsync(e->partials.p, h.data(), nc * sizeof(double), cudaMemcpyHostToDevice, st(s)), "h2d");
        ckn(nccl().AllReduce(e->partials.p, e->partials.p, nc, ncclFloat64, ncclSum,
                             static_cast<ncclComm_t>(e->comm->nccl), st(s)),
            "ncclAllReduce(partials)");
      } else {
        ckh(e->comm->fns.allreduce_sum_f64(e->comm->fns.ctx, h.data(), static_cast<int64_t>(nc)), "allreduce_sum_f64");
        if (nc) ckc(cudaMemcpyAsync(e->partials.p, h.data(), nc * sizeof(double), cudaMemcpyHostToDevice, st(s)), "h2d");
      }
      ckc(cudaStreamSynchronize(st(s)), "sync");  // h is a stack buffer
    }
    rc = ocg_eval_objective_combine(e, e->partials.p, e->scratch.p, s);
    if (rc < 0) return rc;
    ckc(cudaMemcpyAsync(f, e->scratch.p, sizeof(double), cudaMemcpyDeviceToHost, st(s)), "f d2h");
    return ocg_eval_status_all(e, s);
  } catch (const std::exception& ex) {
    return fail(OCG_ERR_CUDA, ex.what());
  }
}

char* ocg_shard_plan_json(const ocg_model* m, int rank, int world) {
  if (!m) {
    fail(OCG_ERR_ARG, "null model");
    return nullptr;
  }
  try {
    const ocg::ShardPlan P = ocg::make_shard_plan(m->nlp, ocg::make_layout(m->nlp), rank, world);
    auto runs = [](const std::vector<ocg::Run>& v) {
      std::string o = "[";
      for (size_t i = 0; i < v.size(); ++i)
        o += (i ? ", [" : "[") + std::to_string(v[i].off) + ", " + std::to_string(v[i].len) + "]";
      return o + "]";
    };
    auto peers = [&](const std::vector<std::vector<ocg::Run>>& v) {
      std::string o = "[";
      for (size_t i = 0; i < v.size(); ++i) o += (i ? ", " : "") + runs(v[i]);
      return o + "]";
    };
    std::string js = "{\"lo\": " + std::to_string(P.lo) + ", \"hi\": " + std::to_string(P.hi) +
                     ", \"specials\": " + (P.specials ? "true" : "false") + ", \"x_own\": " + runs(P.x_own) +
                     ", \"send_to\": " + peers(P.send_to) + ", \"recv_from\": " + peers(P.recv_from) +
                     ", \"rows\": " + runs(P.rows) + ", \"halo_doubles\": " + std::to_string(P.halo_doubles) +
                     ", \"objective_exact\": " + (P.objective_exact ? "true" : "false") +
                     ", \"chunk_owned\": [";
    for (size_t i = 0; i < P.chunk_owned.size(); ++i) js += (i ? ", " : "") + std::to_string(int(P.chunk_owned[i]));
    js += "]}";
    char* out = static_cast<char*>(std::malloc(js.size() + 1));
    std::memcpy(out, js.c_str(), js.size() + 1);
    return out;
  } catch (const std::exception& ex) {
    fail(OCG_ERR_ARG, ex.what());
    return nullptr;
  }
}

}  // extern "C"
