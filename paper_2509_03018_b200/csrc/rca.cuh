// rca.cuh — device root-cause analysis (Algorithm 2, Tables 3/4).
#pragma once

#include "objects.h"

namespace csg {

// Per (trip, rank) summary of the rank's store-order prefix at the trip time
// (the reference's per-member prefix scans, proj/src/rca.cpp:146-237).
struct RankSum {
  uint32_t cutoff;   // prefix length: first rank-local index with ts > t
  uint32_t flags;    // RS_*
  int64_t last_op;   // last_logs_of_group: op of the last prefix record
  double last_ts;
  int32_t last_chan;
  int32_t pad;
  double onset;      // stall_onset_of(rank, last_op, t)
  uint64_t ready, tx, done;  // progress_of(rank, last_op, t)
};
enum : uint32_t { RS_HAS_LAST = 1, RS_STUCK = 2, RS_PROG = 4 };

// Per (straggler trip, group): complete_iterations summary.
struct GroupIter {
  int32_t n_common;
  int32_t late;  // group_has_late_member
};

// Per (straggler trip, membership slot): flow-rule findings of one member.
struct FlowSum {
  int32_t flags;  // 1 skew, 2 incomplete
  int32_t skew_chan;
  int64_t skew_op;
  double skew_start;
  double skew_end;
  int64_t inc_op;
  int32_t inc_chan;
  int32_t pad;
};

struct Cand {
  int32_t rank;
  int32_t group;
  uint8_t cat, side, known, pad;
  int32_t pad2;
  int64_t op;
  double onset;
  uint64_t ready, tx, done;
  int64_t it_lo, it_hi;
  uint32_t ev_off, ev_n;
};

struct TripOut {
  int32_t verdict;
  int32_t n_aff;
  uint64_t scanned;
  uint32_t sus_off, n_sus, exo_off, n_exo, ev_off, n_ev;
};

// Bump-allocated device pools shared by all trips of a batch.
struct Pools {
  Cand* cand;
  unsigned long long cand_cap;
  csg_evidence* cev;
  unsigned long long cev_cap;
  csg_suspect* sus;
  unsigned long long sus_cap;
  csg_evidence* ev;
  unsigned long long ev_cap;
  unsigned long long* bits;
  unsigned long long bits_cap;
  uint32_t* u32;
  unsigned long long u32_cap;
  unsigned long long* used;  // [6] counters
};

struct RcaResult {
  std::vector<TripOut> trips;
  std::vector<csg_suspect> sus;
  std::vector<csg_evidence> ev;
  // [J * G] row j: trip j's affected groups (first trips[j].n_aff valid);
  // points into the context's pinned read-back buffer (valid until the
  // next analysis on the context)
  const int32_t* aff = nullptr;
  int32_t G = 0;
};

// Analyze J triggers (time, kind, suspect rank) over the indexed store.
void rca_batch(csg_store* s, const csg_model* m, const csg_analysis_config& cfg,
               const csg_trigger_event* trips, int32_t J, bool affected_only,
               RcaResult& out);

}  // namespace csg
