// Node-range shards of one evaluation over several GPUs.
//
// Rank q of W evaluates the main grid indices [lo_q, hi_q) — contiguous,
// boundaries on the objective's 512-instance chunk grid so that no chunk of
// the reference's par_reduce (backend.cpp:119-133) straddles two ranks — and rank
// 0 also the endpoint instances. A time node n of a slab is OWNED by the rank
// whose index range holds n (node N by the last rank). Each rank uploads from
// the host only the nodes it owns (plus the free variables, e.g. tf) and the
// multiplier rows of its own instances; the nodes it reads but does not own —
// the one-node right halo, and node N for rank 0's terminal conditions — come
// from their owners over the communicator (ncclSend/ncclRecv, or host
// callbacks such as torch.distributed). The only other collectives are the
// ok flag (max) and the objective's chunk partials (sum of exactly one
// nonzero term per chunk, then the fixed-order combine: bit-identical to one
// device).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/octgpu.h"
#include "model.hpp"
#include "plan.hpp"

namespace ocg {

struct Run {
  Index off = 0, len = 0;  // [off, off + len) of x (or of the rows)
};

struct ShardPlan {
  int rank = 0, world = 1;
  Index lo = 0, hi = 0;     // main grid indices of this rank
  bool specials = true;     // endpoint instances (rank 0)
  std::vector<Run> x_own;   // slots uploaded from the host
  std::vector<std::vector<Run>> send_to, recv_from;  // [peer]: node runs exchanged
  std::vector<Run> rows;    // constraint rows (lambda / row_scale) the instances read
  std::vector<uint8_t> chunk_owned;  // objective chunks computed in full here
  bool objective_exact = true;       // no chunk straddles two ranks
  Index halo_doubles = 0;   // doubles received per exchange
};

// rank q's shard of `nlp` (main grid [L.idx_lo, L.idx_hi)) over `world` ranks
ShardPlan make_shard_plan(const Nlp& nlp, const Layout& L, int rank, int world);

}  // namespace ocg

// the communicator behind ocg_comm (shard.cpp)
struct ocg_comm {
  int rank = 0, world = 1;
  int device = 0;
  void* nccl = nullptr;  // ncclComm_t, or NULL for host callbacks
  ocg_comm_host_fns fns{};
  std::vector<double> hbuf_send, hbuf_recv;  // host staging for the callbacks
};
