// rca_table.h — Tables 3/4 of the Mycroft paper as pure functions, compiled
// for both host (C ABI known-answer entry points) and device (the RCA decide
// kernel). Same code on both sides, so the KATs exercise the device logic.
#pragma once

#include <cstdint>

#include "csg_engine.h"

namespace csg {

// Lexicographic (rdma_done, rdma_transmitted, gpu_ready) order used by
// check_min_data and the exoneration tie rule (proj/src/rca.cpp:266-268,
// :494-500).
__host__ __device__ inline bool prog_less(uint64_t d0, uint64_t t0,
                                          uint64_t r0, uint64_t d1,
                                          uint64_t t1, uint64_t r1) {
  if (d0 != d1) return d0 < d1;
  if (t0 != t1) return t0 < t1;
  return r0 < r1;
}

// check_rc_table (proj/src/rca.cpp:278-306). Returns false when the counters
// violate ready >= tx >= done (the reference throws DataError there).
__host__ __device__ inline bool rc_table(uint64_t ready, uint64_t tx,
                                         uint64_t done, bool has_peer,
                                         uint64_t p_ready, uint64_t p_tx,
                                         uint64_t p_done, int* category,
                                         int* side) {
  if (!(ready >= tx && tx >= done)) return false;
  int cat;
  if (ready == 0 && tx == 0 && done == 0)
    cat = CSG_RC_UNINITIALIZED_OR_BLOCKED;
  else if (tx > done)  // the deeper pipeline stage wins
    cat = CSG_RC_RDMA_ISSUE_OR_RECEIVER_FAILED;
  else if (ready > tx)
    cat = CSG_RC_RDMA_ISSUE_OR_RECEIVER_NOT_READY;
  else
    cat = CSG_RC_GPU_ISSUE;
  int sd = CSG_SIDE_UNDETERMINED;
  if (cat == CSG_RC_GPU_ISSUE)
    sd = CSG_SIDE_LOCAL;
  else if (has_peer && cat == CSG_RC_RDMA_ISSUE_OR_RECEIVER_FAILED &&
           ready == tx && p_ready == p_tx && p_tx == p_done)
    sd = CSG_SIDE_REMOTE;
  *category = cat;
  *side = sd;
  return true;
}

}  // namespace csg
