// rca.cu — Algorithm 2 (dependency-driven root-cause analysis) on the device.
//
// Every tripped tick of a detection run is analyzed in one batch. The O(N)
// work — each rank's store-order prefix at the trip time — is spread over
// one warp per (trip, rank); the reference does the same scans serially per
// group member (proj/src/rca.cpp:146-237, :327-349, :702-731). Group
// reductions, the exoneration sweep and report assembly then run as one
// thread block per trip over those compact per-rank summaries.
//
// Exact-semantics notes:
//  * prefix = rank-local records before the first ts > t in STORE order,
//    found by upper_bound on the per-rank running max (store.cu);
//  * op-DAG reachability (DepIndex::depends_on, rca.cpp:94-139) is answered
//    with candidate bitsets propagated over the periodic program DAG in
//    (iteration, level) order, restricted to [min candidate op, max]: every
//    parent edge points to a smaller global op, so nothing below the smallest
//    candidate can lead to a candidate;
//  * greedy exoneration, straggler candidate de-duplication and the
//    self-evidence filter keep the reference's sequential order.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>

#include "comm.cuh"
#include "fetch.cuh"
#include "rca.cuh"
#include "rca_table.h"

namespace csg {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kDecideThreads = 256;
constexpr int kSfBlocks = 148 * 4;  // persistent k_self_faulted grid
constexpr int kChTbl = 4096;  // max channel id + 1 (store.cu enforces)

__device__ inline double as_double(uint64_t u) {
  double d;
  memcpy(&d, &u, 8);
  return d;
}

// First index in [lo, hi) where the monotone predicate holds, else hi.
// 32-ary warp search: three probes rounds cover 32k elements.
template <typename P>
__device__ uint32_t warp_partition_point(uint32_t lo, uint32_t hi, P pred) {
  const int lane = threadIdx.x & 31;
  while (hi - lo > 32) {
    const uint32_t len = hi - lo;
    const uint32_t step = (len + 31) / 32;
    uint32_t off = (lane + 1) * step;
    if (off > len) off = len;
    const unsigned mm = __ballot_sync(FULL, pred(lo + off - 1));
    if (!mm) return hi;
    const int f = __ffs(mm) - 1;
    uint32_t offf = (f + 1) * step;
    if (offf > len) offf = len;
    const uint32_t qf = lo + offf - 1;
    if (f) {
      uint32_t offp = f * step;
      if (offp > len) offp = len;
      lo = lo + offp;
    }
    hi = qf;
  }
  const uint32_t q = lo + lane;
  const unsigned mm = __ballot_sync(FULL, q < hi && pred(q));
  return mm ? lo + __ffs(mm) - 1 : hi;
}

// First rank-major position of rank r's segment whose ts is > x (strict)
// or >= x, else the segment end; warp-collective. Binary search over the
// chunked prefix maxima (store.cu k_chunkmax_blk), then one 128-record
// chunk scan. This is the reference's store-order prefix cut-off (the first
// record with ts > t ends the prefix, rca.cpp:156 / :174 / :207 / :225).
__device__ uint32_t seg_first(const StoreView& s, int32_t r, double x, bool strict) {
  const uint32_t b = s.rank_off[r], e = s.rank_off[r + 1];
  const uint32_t nc = (e - b + kCmChunk - 1) / kCmChunk;
  const double* cm = s.cmax + (b / kCmChunk + r);
  const uint32_t c = warp_partition_point(0, nc, [&](uint32_t k) {
    const double m = cm[k];
    return strict ? m > x : m >= x;
  });
  if (c == nc) return e;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (uint32_t k = 0; k < kCmChunk / 32; ++k) {
    const uint32_t p = b + c * kCmChunk + k * 32 + lane;
    bool hit = false;
    if (p < e) {
      const double t = s.ts[p];
      hit = strict ? t > x : t >= x;
    }
    const unsigned mm = __ballot_sync(FULL, hit);
    if (mm) return b + c * kCmChunk + k * 32 + __ffs(mm) - 1;
  }
  return e;  // unreachable: the chunk's maximum satisfies the predicate
}

// Lower median sorted[(n-1)/2] of n virtual values (warp; O(n^2/32)).
template <typename V>
__device__ double warp_lower_median(int n, V val) {
  const int lane = threadIdx.x & 31;
  const int k = (n - 1) / 2;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    bool mine = false;
    double vi = 0;
    if (i < n) {
      vi = val(i);
      int less = 0, leq = 0;
      for (int q = 0; q < n; ++q) {
        const double vq = val(q);
        less += vq < vi;
        leq += vq <= vi;
      }
      mine = less <= k && k < leq;
    }
    const unsigned mm = __ballot_sync(FULL, mine);
    if (mm) return __shfl_sync(FULL, vi, __ffs(mm) - 1);
  }
  return 0;  // unreachable for n >= 1
}

// The same lower median over n <= 32 * S values held in registers, value
// s * 32 + lane in v[s] (shuffles instead of n reloads per lane).
template <int S>
__device__ double warp_lower_median_reg(int n, const double (&v)[S]) {
  const int lane = threadIdx.x & 31;
  const int k = (n - 1) / 2;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    if (s * 32 >= n) break;
    const int i = s * 32 + lane;
    const double vi = v[s];
    int less = 0, leq = 0;
#pragma unroll
    for (int t = 0; t < S; ++t) {
      if (t * 32 >= n) break;
      const int lim = min(32, n - t * 32);
      for (int l = 0; l < lim; ++l) {
        const double vq = __shfl_sync(FULL, v[t], l);
        less += vq < vi;
        leq += vq <= vi;
      }
    }
    const bool mine = i < n && less <= k && k < leq;
    const unsigned mm = __ballot_sync(FULL, mine);
    if (mm) return __shfl_sync(FULL, vi, __ffs(mm) - 1);
  }
  return 0;  // unreachable for n >= 1
}

// ---------------------------------------------------------------------------
// K1: per (trip, rank) prefix summary.
// ---------------------------------------------------------------------------
__global__ void k_rank_summary(StoreView s, int32_t J,
                               const double* __restrict__ trip_t,
                               double delta_a, RankSum* __restrict__ out,
                               unsigned long long* __restrict__ chan_key,
                               int32_t nch, int32_t r0, int32_t nr) {
  extern __shared__ uint32_t sm_tbl[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const bool active = w < static_cast<int64_t>(nr) * J;
  const int32_t r = active ? r0 + static_cast<int32_t>(w / J) : 0;
  const int32_t j = active ? static_cast<int32_t>(w % J) : 0;
  uint32_t* tbl = sm_tbl + wib * nch;
  if (!active) return;
  for (int c = lane; c < nch; c += 32) tbl[c] = 0;
  __syncwarp();
  const double t = trip_t[j];
  const double ws = t - delta_a;  // window_start, rca.cpp:405
  const uint32_t b = s.rank_off[r], e = s.rank_off[r + 1];
  const uint32_t cend = seg_first(s, r, t, true);
  const uint32_t c = cend - b;
  // A rank without prefix records leaves an all-zero summary, so summaries
  // of ranks owned by other shards combine by summation (see comm.cu).
  RankSum o;
  o.cutoff = c;
  o.flags = 0;
  o.last_op = 0;
  o.last_ts = 0;
  o.last_chan = 0;
  o.pad = 0;
  o.onset = 0;
  o.ready = o.tx = o.done = 0;
  if (c > 0) {
    o.flags |= RS_HAS_LAST;
    o.last_op = s.op[cend - 1];
    o.last_ts = s.ts[cend - 1];
    o.last_chan = s.chan[cend - 1];
    // stuck_on_incomplete (rca.cpp:216-237): the last prefix record with
    // ts >= window_start is a state whose op has no prefix completion.
    int64_t found = -1;
    // The prefix's running max bounds every timestamp in it: a rank that
    // has been silent since before the window has nothing to scan.
    const int64_t scan_from = seg_first(s, r, ws, false) < cend
                                  ? static_cast<int64_t>(cend) - 1
                                  : static_cast<int64_t>(b) - 1;
    for (int64_t top = scan_from;
         top >= static_cast<int64_t>(b) && found < 0; top -= 32) {
      const int64_t p = top - lane;
      const bool pr = p >= static_cast<int64_t>(b) && s.ts[p] >= ws;
      const unsigned mm = __ballot_sync(FULL, pr);
      if (mm) found = top - (__ffs(mm) - 1);
    }
    bool cand_stuck = false;
    int64_t stuck_op = 0;
    if (found >= 0 && ko_kind(s.ko[found]) == CSG_KIND_STATE) {
      cand_stuck = true;
      stuck_op = s.op[found];
    }
    const int64_t lop = o.last_op;
    bool comp_hit = false, onset_found = false;
    for (uint32_t base = b; base < cend; base += 32) {
      const uint32_t p = base + lane;
      const bool valid = p < cend;
      const int64_t op = valid ? s.op[p] : 0;
      const uint8_t ko = valid ? s.ko[p] : 0;
      if (cand_stuck && !comp_hit)
        comp_hit = __any_sync(FULL, valid && ko_kind(ko) == CSG_KIND_COMPLETION &&
                                        op == stuck_op);
      const unsigned mo = __ballot_sync(FULL, valid && op == lop);
      if (!onset_found && mo) {
        // stall_onset_of (rca.cpp:202-212): first prefix record of the op
        o.onset = s.ts[base + __ffs(mo) - 1];
        onset_found = true;
      }
      if (valid && op == lop && ko_kind(ko) == CSG_KIND_STATE)
        atomicMax(&tbl[s.chan[p]], p + 1);  // latest per channel
    }
    __syncwarp();
    if (cand_stuck && !comp_hit) o.flags |= RS_STUCK;
    // progress_of(rank, last_op, t) (rca.cpp:167-196): sum over channels.
    unsigned long long rd = 0, tx = 0, dn = 0;
    int any = 0;
    for (int ch = lane; ch < nch; ch += 32) {
      const uint32_t q = tbl[ch];
      if (q) {
        any = 1;
        const uint64_t a = s.pa[q - 1];
        rd += a & 0xffffffffull;
        tx += a >> 32;
        dn += s.pb[q - 1];
      }
    }
#pragma unroll
    for (int x = 16; x; x >>= 1) {
      rd += __shfl_xor_sync(FULL, rd, x);
      tx += __shfl_xor_sync(FULL, tx, x);
      dn += __shfl_xor_sync(FULL, dn, x);
      any |= __shfl_xor_sync(FULL, any, x);
    }
    if (any) {
      o.flags |= RS_PROG;
      o.ready = rd;
      o.tx = tx;
      o.done = dn;
    }
  }
  // per-channel evidence: the latest state's timestamp as an ordered key
  // (0 = no state on that channel); the op is the rank's last op.
  unsigned long long* ck = chan_key + (static_cast<uint64_t>(j) * s.R + r) * nch;
  for (int ch = lane; ch < nch; ch += 32)
    ck[ch] = tbl[ch] ? static_cast<unsigned long long>(dkey(s.ts[tbl[ch] - 1])) : 0ull;
  if (lane == 0) out[static_cast<uint64_t>(j) * s.R + r] = o;
}

// K1 (flow-index form): the same summary with every "scan the prefix for
// records of op X" replaced by a lookup in the (rank, op, channel)-ordered
// flow index: the (rank, op) entries are one contiguous range, so stall
// onset, "completion of the stuck op inside the prefix" and the per-channel
// latest state are O(log n + entries of that op), not O(prefix).
__global__ void k_rank_summary_fi(StoreView s, FlowView f, int32_t J,
                                  const double* __restrict__ trip_t,
                                  double delta_a, RankSum* __restrict__ out,
                                  unsigned long long* __restrict__ chan_key,
                                  int32_t nch, int32_t r0, int32_t nr) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint32_t sm_tbl[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= static_cast<int64_t>(nr) * J) return;
  const int32_t r = r0 + static_cast<int32_t>(w / J);
  const int32_t j = static_cast<int32_t>(w % J);
  uint32_t* tbl = sm_tbl + wib * nch;
  for (int c = lane; c < nch; c += 32) tbl[c] = 0;
  __syncwarp();
  const double t = trip_t[j];
  const double ws = t - delta_a;
  const uint32_t b = s.rank_off[r], e = s.rank_off[r + 1];
  const uint32_t cend = seg_first(s, r, t, true);
  const uint32_t c = cend - b;
  // A rank without prefix records leaves an all-zero summary, so summaries
  // of ranks owned by other shards combine by summation (see comm.cu).
  RankSum o;
  o.cutoff = c;
  o.flags = 0;
  o.last_op = 0;
  o.last_ts = 0;
  o.last_chan = 0;
  o.pad = 0;
  o.onset = 0;
  o.ready = o.tx = o.done = 0;
  if (c > 0) {
    o.flags |= RS_HAS_LAST;
    o.last_op = s.op[cend - 1];
    o.last_ts = s.ts[cend - 1];
    o.last_chan = s.chan[cend - 1];
    int64_t found = -1;
    // The prefix's running max bounds every timestamp in it: a rank that
    // has been silent since before the window has nothing to scan.
    const int64_t scan_from = seg_first(s, r, ws, false) < cend
                                  ? static_cast<int64_t>(cend) - 1
                                  : static_cast<int64_t>(b) - 1;
    for (int64_t top = scan_from;
         top >= static_cast<int64_t>(b) && found < 0; top -= 32) {
      const int64_t p = top - lane;
      const bool pr = p >= static_cast<int64_t>(b) && s.ts[p] >= ws;
      const unsigned mm = __ballot_sync(FULL, pr);
      if (mm) found = top - (__ffs(mm) - 1);
    }
    bool cand_stuck = false;
    int64_t stuck_op = 0;
    if (found >= 0 && ko_kind(s.ko[found]) == CSG_KIND_STATE) {
      cand_stuck = true;
      stuck_op = s.op[found];
    }
    const bool uns = f.unsorted[r] != 0;
    auto range_of = [&](int64_t op, uint32_t& fo, uint32_t& fe) {
      fo = warp_partition_point(b, e, [&](uint32_t i) { return s.op[f.at(uns, i)] >= op; });
      fe = warp_partition_point(fo, e, [&](uint32_t i) { return s.op[f.at(uns, i)] > op; });
    };
    uint32_t fo, fe;
    range_of(o.last_op, fo, fe);
    uint32_t first = 0xFFFFFFFFu;
    for (uint32_t i = fo + lane; i < fe; i += 32) {
      const uint32_t p = f.at(uns, i);
      if (p >= cend) continue;
      first = min(first, p);
      if (ko_kind(s.ko[p]) == CSG_KIND_STATE) atomicMax(&tbl[s.chan[p]], p + 1);
    }
#pragma unroll
    for (int x = 16; x; x >>= 1) first = min(first, __shfl_xor_sync(FULL, first, x));
    o.onset = s.ts[first];  // stall_onset_of: first prefix record of the op
    if (cand_stuck) {
      uint32_t so = fo, se = fe;
      if (stuck_op != o.last_op) range_of(stuck_op, so, se);
      bool hit = false;
      for (uint32_t i = so + lane; i < se && !hit; i += 32) {
        const uint32_t p = f.at(uns, i);
        hit = p < cend && ko_kind(s.ko[p]) == CSG_KIND_COMPLETION;
      }
      if (!__any_sync(FULL, hit)) o.flags |= RS_STUCK;
    }
    __syncwarp();
    unsigned long long rd = 0, tx = 0, dn = 0;
    int any = 0;
    for (int ch = lane; ch < nch; ch += 32) {
      const uint32_t q = tbl[ch];
      if (q) {
        any = 1;
        const uint64_t a = s.pa[q - 1];
        rd += a & 0xffffffffull;
        tx += a >> 32;
        dn += s.pb[q - 1];
      }
    }
#pragma unroll
    for (int x = 16; x; x >>= 1) {
      rd += __shfl_xor_sync(FULL, rd, x);
      tx += __shfl_xor_sync(FULL, tx, x);
      dn += __shfl_xor_sync(FULL, dn, x);
      any |= __shfl_xor_sync(FULL, any, x);
    }
    if (any) {
      o.flags |= RS_PROG;
      o.ready = rd;
      o.tx = tx;
      o.done = dn;
    }
  }
  // per-channel evidence: the latest state's timestamp as an ordered key
  // (0 = no state on that channel); the op is the rank's last op.
  unsigned long long* ck = chan_key + (static_cast<uint64_t>(j) * s.R + r) * nch;
  for (int ch = lane; ch < nch; ch += 32)
    ck[ch] = tbl[ch] ? static_cast<unsigned long long>(dkey(s.ts[tbl[ch] - 1])) : 0ull;
  if (lane == 0) out[static_cast<uint64_t>(j) * s.R + r] = o;
}

// ---------------------------------------------------------------------------
// K1b: ring-successor progress (rca.cpp:596-605). For every membership slot
// (trip, group, member s) whose ring predecessor p has a prefix: progress_of
// (s, last_op(p), t) with per-channel evidence. A suspect at ring position i
// reads the slot of position i+1. Computed by the shard owning s.
// ---------------------------------------------------------------------------
struct SuccProg {
  uint32_t known;
  uint32_t pad;
  unsigned long long ready, tx, done;
};

__global__ void k_succ_prog(StoreView s, FlowView f, ModelView m, int32_t J,
                            uint32_t M, const uint32_t* __restrict__ slot_group,
                            const RankSum* __restrict__ rs,
                            SuccProg* __restrict__ out,
                            unsigned long long* __restrict__ sp_key,
                            int32_t nch, const uint32_t* __restrict__ slots,
                            uint32_t nslots, const int32_t* __restrict__ trip_kind) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint32_t sp_tbl[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  // slots (sharded stores): only the membership slots of owned ranks
  const uint32_t E = slots ? nslots : M;
  if (w >= static_cast<int64_t>(E) * J) return;
  const int32_t j = static_cast<int32_t>(w / E);
  // only failure analysis reads the successor's progress (k_fail_cands)
  if (trip_kind[j] != CSG_TRIGGER_FAILURE) return;
  const uint32_t q = slots ? slots[w % E] : static_cast<uint32_t>(w % E);
  uint32_t* tbl = sp_tbl + wib * nch;
  for (int c = lane; c < nch; c += 32) tbl[c] = 0;
  __syncwarp();
  const int32_t g = static_cast<int32_t>(slot_group[q]);
  const uint32_t mo = m.member_off[g];
  const int32_t mm = static_cast<int32_t>(m.member_off[g + 1] - mo);
  const int32_t i = static_cast<int32_t>(q - mo);
  const int32_t sr = m.members[q];
  SuccProg o{0, 0, 0, 0, 0};
  const RankSum* rsj = rs + static_cast<uint64_t>(j) * s.R;
  bool go = mm >= 2 && sr >= 0 && sr < s.R && s.rank_off[sr + 1] > s.rank_off[sr];
  int32_t pred = -1;
  if (go) {
    pred = m.members[mo + (i + mm - 1) % mm];
    go = pred >= 0 && pred < s.R && (rsj[pred].flags & RS_HAS_LAST);
  }
  if (go) {
    const int64_t op = rsj[pred].last_op;
    const uint32_t b = s.rank_off[sr];
    const uint32_t cend = min(b + rsj[sr].cutoff, s.rank_off[sr + 1]);
    if (f.n) {
      const uint32_t e = s.rank_off[sr + 1];
      const bool uns = f.unsorted[sr] != 0;
      const uint32_t fo = warp_partition_point(
          b, e, [&](uint32_t x) { return s.op[f.at(uns, x)] >= op; });
      const uint32_t fe = warp_partition_point(
          fo, e, [&](uint32_t x) { return s.op[f.at(uns, x)] > op; });
      for (uint32_t x = fo + lane; x < fe; x += 32) {
        const uint32_t p = f.at(uns, x);
        if (p < cend && ko_kind(s.ko[p]) == CSG_KIND_STATE)
          atomicMax(&tbl[s.chan[p]], p + 1);
      }
    } else {  // no flow index: scan the prefix
      for (uint32_t p = b + lane; p < cend; p += 32)
        if (s.op[p] == op && ko_kind(s.ko[p]) == CSG_KIND_STATE)
          atomicMax(&tbl[s.chan[p]], p + 1);
    }
    __syncwarp();
    unsigned long long rd = 0, tx = 0, dn = 0;
    int any = 0;
    for (int ch = lane; ch < nch; ch += 32) {
      const uint32_t qq = tbl[ch];
      if (qq) {
        any = 1;
        const uint64_t a = s.pa[qq - 1];
        rd += a & 0xffffffffull;
        tx += a >> 32;
        dn += s.pb[qq - 1];
      }
    }
#pragma unroll
    for (int x = 16; x; x >>= 1) {
      rd += __shfl_xor_sync(FULL, rd, x);
      tx += __shfl_xor_sync(FULL, tx, x);
      dn += __shfl_xor_sync(FULL, dn, x);
      any |= __shfl_xor_sync(FULL, any, x);
    }
    o.known = any ? 1 : 0;
    o.ready = rd;
    o.tx = tx;
    o.done = dn;
  }
  unsigned long long* ck = sp_key + (static_cast<uint64_t>(j) * M + q) * nch;
  for (int ch = lane; ch < nch; ch += 32)
    ck[ch] = tbl[ch] ? static_cast<unsigned long long>(dkey(s.ts[tbl[ch] - 1])) : 0ull;
  if (lane == 0) out[static_cast<uint64_t>(j) * M + q] = o;
}

// ---------------------------------------------------------------------------
// K2: group_iterations (rca.cpp:327-349) for straggler trips: per
// (trip, member slot, iteration) min start / max end of the member's prefix
// completions with comm_id == group.
// ---------------------------------------------------------------------------
// Min / max of (start, end) keys into table cells, one atomic pair per
// distinct cell of the warp: consecutive records of a rank segment mostly
// fall into the same (slot, iteration) cell, and 32 same-address atomics
// serialise at L2. Warp-uniform call; part = this lane has a record.
__device__ __forceinline__ void warp_cell_minmax(bool part, uint64_t idx, unsigned long long ks,
                                                 unsigned long long ke,
                                                 unsigned long long* __restrict__ tbl_s,
                                                 unsigned long long* __restrict__ tbl_e) {
  const int lane = threadIdx.x & 31;
  unsigned todo = __ballot_sync(FULL, part);
  while (todo) {
    const int l = __ffs(todo) - 1;
    const uint64_t cidx = __shfl_sync(FULL, idx, l);
    const bool mine = part && idx == cidx;
    unsigned long long vmn = mine ? ks : ~0ull, vmx = mine ? ke : 0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      vmn = min(vmn, __shfl_xor_sync(FULL, vmn, o));
      vmx = max(vmx, __shfl_xor_sync(FULL, vmx, o));
    }
    if (lane == l) {
      atomicMin(&tbl_s[cidx], vmn);
      atomicMax(&tbl_e[cidx], vmx);
    }
    todo &= ~__ballot_sync(FULL, mine);
  }
}

__global__ void k_iter_tables(StoreView s, ModelView m, int32_t Js,
                              const int32_t* __restrict__ strag_trip,
                              const RankSum* __restrict__ rs, int64_t it_min,
                              int32_t n_it, uint32_t M,
                              unsigned long long* __restrict__ tbl_s,
                              unsigned long long* __restrict__ tbl_e) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= static_cast<int64_t>(s.R) * Js) return;
  const int32_t r = static_cast<int32_t>(w / Js);
  const int32_t js = static_cast<int32_t>(w % Js);
  if (r >= m.rank_space) return;
  const uint32_t g0 = m.rg_off[r], g1 = m.rg_off[r + 1];
  if (g0 == g1) return;
  const int32_t j = strag_trip[js];
  const uint32_t b = s.rank_off[r];
  // summaries are global after the shard all-reduce; only this shard's
  // segment is walked (empty for ranks owned elsewhere)
  const uint32_t cend =
      min(b + rs[static_cast<uint64_t>(j) * s.R + r].cutoff, s.rank_off[r + 1]);
  for (uint32_t pw = b; pw < cend; pw += 32) {
    const uint32_t p = pw + lane;
    uint32_t slot = kNoPos;
    if (p < cend && ko_kind(s.ko[p]) == CSG_KIND_COMPLETION) {
      const int32_t cm = s.comm[p];
      for (uint32_t q = g0; q < g1; ++q)
        if (m.rg_group[q] == cm) {
          slot = m.rg_slot[q];
          break;
        }
    }
    const bool part = slot != kNoPos;
    uint64_t idx = 0;
    unsigned long long ks = 0, ke = 0;
    if (part) {
      const int64_t it = iter_of(s.op[p], m.opn) - it_min;
      idx = (static_cast<uint64_t>(js) * M + slot) * n_it + it;
      ks = static_cast<unsigned long long>(dkey(as_double(s.pa[p])));
      ke = static_cast<unsigned long long>(dkey(s.ts[p]));
    }
    warp_cell_minmax(part, idx, ks, ke, tbl_s, tbl_e);
  }
}

// Incremental form for trips in time order: the prefix of straggler trip js
// (records before the first ts > t_js) contains the prefix of trip js - 1,
// so each record is folded into the table of the first trip whose prefix
// holds it (one pass over the store instead of one per trip), and
// k_iter_prefix then combines the tables over the trips (running min/max
// per (slot, iteration) cell). kIterParts warps per rank, each over one
// contiguous part of the rank's segment (the walk is load-latency bound:
// one warp per rank left 8 warps per SM on the C2 store).
constexpr int kIterParts = 8;
constexpr int kIterUnroll = 4;
__global__ void k_iter_tables_inc(StoreView s, ModelView m, int32_t Js,
                                  const int32_t* __restrict__ strag_trip,
                                  const RankSum* __restrict__ rs, int64_t it_min,
                                  int32_t n_it, uint32_t M, int32_t cached_js,
                                  unsigned long long* __restrict__ tbl_s,
                                  unsigned long long* __restrict__ tbl_e) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t wr = w / kIterParts;
  const int part = static_cast<int>(w % kIterParts);
  if (wr >= s.R || wr >= m.rank_space) return;
  const int32_t r = static_cast<int32_t>(wr);
  const uint32_t g0 = m.rg_off[r], g1 = m.rg_off[r + 1];
  if (g0 == g1) return;
  const uint32_t b = s.rank_off[r], e = s.rank_off[r + 1];
  // one block per rank (kIterParts warps): the trips' prefix ends once, in
  // shared memory (cached_js of them; the rest are read from global)
  extern __shared__ uint32_t s_cend[];
  auto cend_g = [&](int32_t js) {
    return min(b + rs[static_cast<uint64_t>(strag_trip[js]) * s.R + r].cutoff, e);
  };
  const int32_t cached = min(Js, cached_js);
  for (int32_t js = threadIdx.x; js < cached; js += blockDim.x) s_cend[js] = cend_g(js);
  __syncthreads();
  auto cend_of = [&](int32_t js) { return js < cached ? s_cend[js] : cend_g(js); };
  const uint32_t plen = (e - b + kIterParts - 1) / kIterParts;
  const uint32_t p0 = min(e, b + part * plen), p1 = min(e, p0 + plen);
  if (p0 >= p1) return;
  // the rank's (group, slot) pairs in registers (a rank sits in <= 3 groups)
  int32_t gq[4];
  uint32_t sq[4];
  const int ng = min(static_cast<int>(g1 - g0), 4);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    gq[q] = q < ng ? m.rg_group[g0 + q] : INT_MIN;
    sq[q] = q < ng ? m.rg_slot[g0 + q] : kNoPos;
  }
  const bool many = g1 - g0 > 4;
  // record p belongs to the first trip js (in order) with cend(js) > p; p
  // only grows along a lane, so each lane advances its own trip cursor
  int32_t jl = 0;
  uint32_t cl = Js > 0 ? cend_of(0) : 0;
  const uint4* meta = reinterpret_cast<const uint4*>(s.comm.p);
  const ulonglong2* tso = reinterpret_cast<const ulonglong2*>(s.ts.p);
  for (uint32_t pw = p0; pw < p1; pw += 32 * kIterUnroll) {
    // every load of the batch issued before any is used: the walk is bound
    // by the dependent meta -> payload round trips, not by bandwidth
    uint4 mt[kIterUnroll];
#pragma unroll
    for (int u = 0; u < kIterUnroll; ++u) {
      const uint32_t p = pw + u * 32 + lane;
      mt[u] = p < p1 ? meta[p] : make_uint4(0, 0, 0, 0);
    }
    ulonglong2 to[kIterUnroll];
    unsigned long long pv[kIterUnroll];
#pragma unroll
    for (int u = 0; u < kIterUnroll; ++u) {
      const uint32_t p = pw + u * 32 + lane;
      const bool cmp = p < p1 && ko_kind(static_cast<uint8_t>(mt[u].w)) == CSG_KIND_COMPLETION;
      to[u] = cmp ? tso[p] : make_ulonglong2(0, 0);
      pv[u] = cmp ? *reinterpret_cast<const unsigned long long*>(
                        s.pa.recs + static_cast<uint64_t>(mt[u].z) * 48 + 32)
                  : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kIterUnroll; ++u) {
      const uint32_t p = pw + u * 32 + lane;
      if (p >= p1 || ko_kind(static_cast<uint8_t>(mt[u].w)) != CSG_KIND_COMPLETION) continue;
      while (jl < Js && cl <= p) {
        ++jl;
        cl = jl < Js ? cend_of(jl) : 0;
      }
      if (jl >= Js) continue;
      const int32_t cm = static_cast<int32_t>(mt[u].x);
      uint32_t slot = kNoPos;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (slot == kNoPos && gq[q] == cm) slot = sq[q];
      if (slot == kNoPos && many)
        for (uint32_t q = g0 + 4; q < g1; ++q)
          if (m.rg_group[q] == cm) {
            slot = m.rg_slot[q];
            break;
          }
      if (slot == kNoPos) continue;
      const int64_t it = iter_of(static_cast<int64_t>(to[u].y), m.opn) - it_min;
      const uint64_t idx = (static_cast<uint64_t>(jl) * M + slot) * n_it + it;
      atomicMin(&tbl_s[idx], static_cast<unsigned long long>(dkey(__longlong_as_double(
                                 static_cast<long long>(pv[u])))));
      atomicMax(&tbl_e[idx], static_cast<unsigned long long>(dkey(__longlong_as_double(
                                 static_cast<long long>(to[u].x)))));
    }
  }
}

// Running min/max over the trips' incremental tables, and the presence
// counts: pc[(js, group, it)] += 1 for the trip at which a membership slot's
// (slot, it) cell first holds a completion (k_pc_prefix turns them into the
// number of the group's members present at iteration it for trip js).
__global__ void k_iter_prefix(int32_t Js, uint64_t cells, int32_t n_it, int32_t G,
                              const uint32_t* __restrict__ slot_group,
                              const int32_t* __restrict__ members, int32_t own_lo,
                              int32_t own_hi,
                              unsigned long long* __restrict__ tbl_s,
                              unsigned long long* __restrict__ tbl_e,
                              uint32_t* __restrict__ pc) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < cells;
       c += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t slot = static_cast<uint32_t>(c / n_it);
    // sharded: other shards' members have empty cells here
    const int32_t mr = members[slot];
    if (mr < own_lo || mr > own_hi) continue;
    unsigned long long a = tbl_s[c], z = tbl_e[c];
    const uint64_t gi0 = static_cast<uint64_t>(slot_group[slot]) * n_it + c % n_it;
    const uint64_t gstride = static_cast<uint64_t>(G) * n_it;
    if (a != ~0ull) atomicAdd(&pc[gi0], 1u);
    for (int32_t js = 1; js < Js; ++js) {
      const uint64_t i = static_cast<uint64_t>(js) * cells + c;
      const unsigned long long a1 = min(a, tbl_s[i]);
      if (a == ~0ull && a1 != ~0ull) atomicAdd(&pc[js * gstride + gi0], 1u);
      a = a1;
      z = max(z, tbl_e[i]);
      tbl_s[i] = a;
      tbl_e[i] = z;
    }
  }
}

// Presence counts of per-trip (non-cumulative) tables: every present cell.
__global__ void k_iter_count(int32_t Js, uint64_t cells, int32_t n_it, int32_t G,
                             const uint32_t* __restrict__ slot_group,
                             const unsigned long long* __restrict__ tbl_s,
                             uint32_t* __restrict__ pc) {
  const uint64_t total = static_cast<uint64_t>(Js) * cells;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (tbl_s[i] == ~0ull) continue;
    const uint64_t js = i / cells, c = i % cells;
    const uint32_t slot = static_cast<uint32_t>(c / n_it);
    atomicAdd(&pc[(js * G + slot_group[slot]) * n_it + c % n_it], 1u);
  }
}

__global__ void k_pc_prefix(int32_t Js, uint64_t cells, uint32_t* __restrict__ pc) {
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < cells;
       c += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t a = pc[c];
    for (int32_t js = 1; js < Js; ++js) {
      a += pc[static_cast<uint64_t>(js) * cells + c];
      pc[static_cast<uint64_t>(js) * cells + c] = a;
    }
  }
}

// Sharded stores: the only table cells read after k_group_iters are the
// members' cells at each group's last k common iterations (gi_last); they
// are packed (dir 0), min/max all-reduced, and written back (dir 1) instead
// of all-reducing the whole (trip, slot, iteration) tables.
__global__ void k_win_xfer(ModelView m, int32_t Js, int64_t it_min, int32_t n_it,
                           uint32_t M, int32_t k, const GroupIter* __restrict__ gi,
                           const int64_t* __restrict__ gi_last,
                           unsigned long long* __restrict__ tbl_s,
                           unsigned long long* __restrict__ tbl_e,
                           unsigned long long* __restrict__ pk_s,
                           unsigned long long* __restrict__ pk_e, int dir) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= static_cast<int64_t>(m.n_groups) * Js) return;
  const int32_t js = static_cast<int32_t>(w / m.n_groups);
  const int32_t g = static_cast<int32_t>(w % m.n_groups);
  const uint64_t gidx = static_cast<uint64_t>(js) * m.n_groups + g;
  const int32_t cnt = gi[gidx].n_common;
  const uint32_t mo = m.member_off[g];
  const int32_t mm = static_cast<int32_t>(m.member_off[g + 1] - mo);
  if (mm < 2 || cnt <= 0) return;
  const int32_t q0 = k - min(cnt, k);
  const int32_t nq = k - q0;
  for (int32_t t = lane; t < mm * nq; t += 32) {
    const int32_t x = t / nq, q = q0 + t % nq;
    const uint64_t row = static_cast<uint64_t>(js) * M + m.member_slot[mo + x];
    const uint64_t cell = row * n_it + static_cast<uint64_t>(gi_last[gidx * k + q] - it_min);
    const uint64_t pi = row * k + q;
    if (dir == 0) {
      pk_s[pi] = tbl_s[cell];
      pk_e[pi] = tbl_e[cell];
    } else {
      tbl_s[cell] = pk_s[pi];
      tbl_e[cell] = pk_e[pi];
    }
  }
}

// ---------------------------------------------------------------------------
// K3: complete_iterations (rca.cpp:352-372) + group_has_late_member
// (rca.cpp:374-396), one warp per (straggler trip, group).
// ---------------------------------------------------------------------------
// Presence of a group at an iteration comes from the member counts pc
// (k_iter_prefix / k_iter_count); mode 1 finds the common iterations only,
// mode 2 the medians / late flag at the latest one (after the sharded window
// exchange), mode 3 both.
__global__ void k_group_iters(ModelView m, int32_t Js, int64_t it_min,
                              int32_t n_it, uint32_t M, int32_t k,
                              double thr,
                              const unsigned long long* __restrict__ tbl_s,
                              const unsigned long long* __restrict__ tbl_e,
                              const uint32_t* __restrict__ pc, int mode,
                              GroupIter* __restrict__ gi,
                              int64_t* __restrict__ gi_last) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= static_cast<int64_t>(m.n_groups) * Js) return;
  const int32_t js = static_cast<int32_t>(w / m.n_groups);
  const int32_t g = static_cast<int32_t>(w % m.n_groups);
  const uint32_t mo = m.member_off[g];
  const int32_t mm = static_cast<int32_t>(m.member_off[g + 1] - mo);
  const uint64_t gidx = static_cast<uint64_t>(js) * m.n_groups + g;
  GroupIter out{0, 0};
  int64_t* last = gi_last + gidx * k;
  if (mm >= 2 && m.opn > 0) {
    const uint64_t rowbase = static_cast<uint64_t>(js) * M;
    int32_t count = 0;
    int64_t latest = 0;
    if (mode & 1) {
      const uint32_t* pcg = pc + gidx * n_it;
      int32_t got = 0;
      for (int64_t top = n_it - 1; top >= 0; top -= 32) {
        const int64_t it = top - lane;
        const bool present = it >= 0 && pcg[it] == static_cast<uint32_t>(mm);
        unsigned bm = __ballot_sync(FULL, present);
        if (count == 0 && bm) latest = top - (__ffs(bm) - 1);
        count += __popc(bm);
        while (bm && got < k) {
          const int f = __ffs(bm) - 1;
          if (lane == 0) last[k - 1 - got] = top - f + it_min;
          ++got;
          bm &= bm - 1;
        }
      }
    } else {
      count = gi[gidx].n_common;
      if (count > 0) latest = last[k - 1] - it_min;
    }
    out.n_common = count;
    if ((mode & 2) && count > 0) {
      // lower medians of starts / ends at the latest common iteration
      auto sv = [&](int i) {
        return dkey_inv(tbl_s[(rowbase + m.member_slot[mo + i]) * n_it + latest]);
      };
      auto ev = [&](int i) {
        return dkey_inv(tbl_e[(rowbase + m.member_slot[mo + i]) * n_it + latest]);
      };
      bool late = false;
      constexpr int S = 8;
      if (mm <= 32 * S) {  // the members' cells once, in registers
        double vs[S], ve[S];
#pragma unroll
        for (int q = 0; q < S; ++q) {
          const int i = q * 32 + lane;
          vs[q] = i < mm ? sv(i) : 0.0;
          ve[q] = i < mm ? ev(i) : 0.0;
        }
        const double ms = warp_lower_median_reg(mm, vs);
        const double me = warp_lower_median_reg(mm, ve);
#pragma unroll
        for (int q = 0; q < S; ++q)
          if (q * 32 + lane < mm) late |= (vs[q] - ms >= thr) || (ve[q] - me >= thr);
      } else {
        const double ms = warp_lower_median(mm, sv);
        const double me = warp_lower_median(mm, ev);
        for (int32_t i = lane; i < mm; i += 32)
          late |= (sv(i) - ms >= thr) || (ev(i) - me >= thr);
      }
      out.late = __any_sync(FULL, late) ? 1 : 0;
    }
  }
  if (lane == 0) gi[gidx] = out;
}

// ---------------------------------------------------------------------------
// K4: affected_groups (rca.cpp:400-461), grid (trip, slice): each block
// flags one slice of the groups (latency-bound member lookups spread over
// the GPU), the last block of a trip to finish compacts the flags in group
// order. Reachability from the trigger rank's groups is the static group
// graph's connected component (computed once per model on the host).
// ---------------------------------------------------------------------------
constexpr int kAffSlices = 16;
__global__ void k_affected(StoreView s, ModelView m, int32_t J,
                           const int32_t* __restrict__ trip_kind,
                           const int32_t* __restrict__ trip_rank,
                           const int32_t* __restrict__ js_of,
                           const RankSum* __restrict__ rs,
                           const GroupIter* __restrict__ gi,
                           int32_t* __restrict__ aff,
                           uint8_t* __restrict__ aff_flag,
                           int32_t* __restrict__ n_aff,
                           unsigned* __restrict__ slices_done) {
  pdl_wait();
  pdl_trigger();
  __shared__ int32_t comps[64];
  __shared__ int32_t ncomp;
  __shared__ int32_t wsum[32];
  __shared__ int32_t base;
  __shared__ bool last;
  const int32_t j = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  if (tid == 0) {
    ncomp = 0;
    base = 0;
    const int32_t sr = trip_rank[j];
    if (sr >= 0 && sr < m.rank_space) {
      for (uint32_t q = m.rg_off[sr]; q < m.rg_off[sr + 1]; ++q) {
        const int32_t cid = m.comp[m.rg_group[q]];
        bool seen = false;
        for (int32_t i = 0; i < ncomp; ++i) seen |= comps[i] == cid;
        if (!seen && ncomp < 64) comps[ncomp++] = cid;
      }
    }
  }
  __syncthreads();
  const bool strag = trip_kind[j] == CSG_TRIGGER_STRAGGLER;
  const int32_t js = js_of[j];
  // pass 1, a warp per group: any member stuck (lanes over the members), or
  // late for straggler trips; reachable = same connected component
  uint8_t* af = aff_flag + static_cast<uint64_t>(j) * m.n_groups;
  for (int32_t g = blockIdx.y * nwarps + warp; g < m.n_groups; g += gridDim.y * nwarps) {
    bool reach = false;
    const int32_t cg = m.comp[g];
    for (int32_t i = 0; i < ncomp; ++i) reach |= comps[i] == cg;
    bool flag = false;
    if (reach) {
      const uint32_t q0 = m.member_off[g], q1 = m.member_off[g + 1];
      for (uint32_t qb = q0; qb < q1 && !flag; qb += 32) {
        const uint32_t q = qb + lane;
        bool st = false;
        if (q < q1) {
          const int32_t r = m.members[q];
          st = r >= 0 && r < s.R && (rs[static_cast<uint64_t>(j) * s.R + r].flags & RS_STUCK);
        }
        flag = __any_sync(FULL, st);
      }
      if (!flag && strag && js >= 0 && gi[static_cast<uint64_t>(js) * m.n_groups + g].late)
        flag = true;
    }
    if (lane == 0) af[g] = flag ? 1 : 0;
  }
  // the last slice of trip j to finish compacts (its flag reads bypass L1)
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const unsigned prev = atomicAdd(slices_done + j, 1u);
    last = prev == gridDim.y - 1;
    if (last) slices_done[j] = 0;  // ready for the next launch
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // pass 2: ordered compaction of the flagged groups
  for (int32_t g0 = 0; g0 < m.n_groups; g0 += blockDim.x) {
    const int32_t g = g0 + tid;
    const int hit = g < m.n_groups ? __ldcg(af + g) : 0;
    int x = hit;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int v = lane < nwarps ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, v, o);
        if (lane >= o) v += y;
      }
      wsum[lane] = v;
    }
    __syncthreads();
    if (hit)
      aff[static_cast<uint64_t>(j) * m.n_groups + base + (warp ? wsum[warp - 1] : 0) +
          x - 1] = g;
    __syncthreads();
    if (tid == 0) base += wsum[nwarps - 1];
    __syncthreads();
  }
  if (tid == 0) n_aff[j] = base;
}

// ---------------------------------------------------------------------------
// K5: straggler flow rules (rca.cpp:702-786) per (straggler trip, member of
// an affected group with enough history): the first op (ascending) with a
// skewed window flow, and the first op with an incomplete window flow.
// ---------------------------------------------------------------------------
constexpr int kFlowWarps = 4;
__device__ void flow_scan_one(int64_t w, StoreView s, ModelView m, int32_t Js,
                              const int32_t* __restrict__ strag_trip,
                              const double* __restrict__ trip_t, double delta_a,
                              double skew, int32_t k, uint32_t M,
                              const uint32_t* __restrict__ slot_group,
                              const RankSum* __restrict__ rs,
                              const GroupIter* __restrict__ gi,
                              const uint8_t* __restrict__ aff_flag,
                              FlowSum* __restrict__ fs, uint32_t* __restrict__ err,
                              uint32_t (*buf)[kFlowBuf], uint32_t (*sbits)[kChTbl / 32],
                              uint32_t (*cbits)[kChTbl / 32]) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  if (w >= static_cast<int64_t>(M) * Js) return;
  const int32_t js = static_cast<int32_t>(w / M);
  const uint32_t slot = static_cast<uint32_t>(w % M);
  const int32_t g = static_cast<int32_t>(slot_group[slot]);
  const int32_t j = strag_trip[js];
  FlowSum out;
  memset(&out, 0, sizeof(out));
  const uint64_t gidx = static_cast<uint64_t>(js) * m.n_groups + g;
  const bool run = aff_flag[static_cast<uint64_t>(j) * m.n_groups + g] &&
                   m.member_off[g + 1] - m.member_off[g] >= 2 &&
                   gi[gidx].n_common >= k && m.member_slot[slot] == slot;
  const int32_t r = m.members[slot];
  if (!run || r < 0 || r >= s.R) {
    if (lane == 0) fs[static_cast<uint64_t>(js) * M + slot] = out;
    return;
  }
  const double t = trip_t[j];
  const double ws = t - delta_a;
  const uint32_t b = s.rank_off[r];
  const uint32_t e =
      min(b + rs[static_cast<uint64_t>(j) * s.R + r].cutoff, s.rank_off[r + 1]);
  // records before p0 all have ts < ws (running max below ws)
  const uint32_t p0 = min(seg_first(s, r, ws, false), e);
  auto win_comp = [&](uint32_t p) {
    const uint8_t ko = s.ko[p];
    return ko_kind(ko) == CSG_KIND_COMPLETION && ko_opname(ko) != CSG_OP_RECV &&
           s.comm[p] == g && s.ts[p] >= ws;
  };
  auto win_state = [&](uint32_t p) {
    const uint8_t ko = s.ko[p];
    if (ko_kind(ko) != CSG_KIND_STATE || s.comm[p] != g || s.ts[p] < ws)
      return false;
    const uint64_t pi = static_cast<uint64_t>(s.op[p]) % static_cast<uint64_t>(m.opn);
    return m.op_name[pi] != CSG_OP_RECV;
  };
  // (a) FlowSkewed: ops ascending
  {
    bool have_prev = false;
    int64_t prev = 0;
    for (;;) {
      long long cur = LLONG_MAX;
      for (uint32_t p = p0 + lane; p < e; p += 32)
        if (win_comp(p)) {
          const int64_t op = s.op[p];
          if ((!have_prev || op > prev) && op < cur) cur = op;
        }
#pragma unroll
      for (int x = 16; x; x >>= 1) cur = min(cur, __shfl_xor_sync(FULL, cur, x));
      if (cur == LLONG_MAX) break;
      int n = 0;
      for (uint32_t base = p0; base < e; base += 32) {
        const uint32_t p = base + lane;
        const bool pr = p < e && win_comp(p) && s.op[p] == cur;
        const unsigned mm = __ballot_sync(FULL, pr);
        if (pr) {
          const int idx = n + __popc(mm & ((1u << lane) - 1u));
          if (idx < kFlowBuf) buf[wib][idx] = p;
        }
        n += __popc(mm);
      }
      __syncwarp();
      if (n > kFlowBuf) {
        if (lane == 0) atomicOr(err, DEV_ERR_TOO_MANY_COMPS);
        break;
      }
      if (n >= 2) {
        auto dur = [&](int i) {
          const uint32_t p = buf[wib][i];
          return s.ts[p] - as_double(s.pa[p]);
        };
        const double med = warp_lower_median(n, dur);
        int hit = -1;
        if (med > 0) {
          const double lim = __dmul_rn(skew, med);
          for (int base = 0; base < n && hit < 0; base += 32) {
            const int i = base + lane;
            const unsigned mm = __ballot_sync(FULL, i < n && dur(i) > lim);
            if (mm) hit = base + __ffs(mm) - 1;
          }
        }
        if (hit >= 0) {
          const uint32_t p = buf[wib][hit];
          out.flags |= 1;
          out.skew_op = cur;
          out.skew_chan = s.chan[p];
          out.skew_start = as_double(s.pa[p]);
          out.skew_end = s.ts[p];
          break;
        }
      }
      __syncwarp();
      have_prev = true;
      prev = cur;
    }
  }
  // (b) FlowIncomplete: window state ops ascending
  {
    const int words = (s.nch + 31) / 32;
    bool have_prev = false;
    int64_t prev = 0;
    for (;;) {
      long long cur = LLONG_MAX;
      for (uint32_t p = p0 + lane; p < e; p += 32)
        if (win_state(p)) {
          const int64_t op = s.op[p];
          if ((!have_prev || op > prev) && op < cur) cur = op;
        }
#pragma unroll
      for (int x = 16; x; x >>= 1) cur = min(cur, __shfl_xor_sync(FULL, cur, x));
      if (cur == LLONG_MAX) break;
      for (int q = lane; q < words; q += 32) {
        sbits[wib][q] = 0;
        cbits[wib][q] = 0;
      }
      __syncwarp();
      for (uint32_t p = p0 + lane; p < e; p += 32)
        if (win_state(p) && s.op[p] == cur) {
          const int32_t ch = s.chan[p];
          atomicOr(&sbits[wib][ch >> 5], 1u << (ch & 31));
        }
      // completed_channels: every prefix completion of the group (not just
      // the window), Recv completions excluded (rca.cpp:718,724).
      for (uint32_t p = b + lane; p < e; p += 32) {
        const uint8_t ko = s.ko[p];
        if (ko_kind(ko) == CSG_KIND_COMPLETION && ko_opname(ko) != CSG_OP_RECV &&
            s.comm[p] == g && s.op[p] == cur) {
          const int32_t ch = s.chan[p];
          atomicOr(&cbits[wib][ch >> 5], 1u << (ch & 31));
        }
      }
      __syncwarp();
      bool any = false;
      int first = -1;
      for (int q = 0; q < words; ++q) {
        const uint32_t sb = sbits[wib][q], cb = cbits[wib][q];
        any |= (sb & cb) != 0;
        if (first < 0 && (sb & ~cb)) first = q * 32 + __ffs(sb & ~cb) - 1;
      }
      if (any && first >= 0) {
        out.flags |= 2;
        out.inc_op = cur;
        out.inc_chan = first;
        break;
      }
      __syncwarp();
      have_prev = true;
      prev = cur;
    }
  }
  if (lane == 0) fs[static_cast<uint64_t>(js) * M + slot] = out;
}

// k_flow: one warp per (straggler trip, membership slot), or per listed
// (trip, slot) item (the members k_flow_fi could not stage)
__global__ void __launch_bounds__(kFlowWarps * 32)
    k_flow(StoreView s, ModelView m, int32_t Js, const int32_t* __restrict__ strag_trip,
           const double* __restrict__ trip_t, double delta_a, double skew, int32_t k,
           uint32_t M, const uint32_t* __restrict__ slot_group,
           const RankSum* __restrict__ rs, const GroupIter* __restrict__ gi,
           const uint8_t* __restrict__ aff_flag, FlowSum* __restrict__ fs,
           uint32_t* __restrict__ err, const uint32_t* __restrict__ only,
           const unsigned* __restrict__ n_only) {
  __shared__ uint32_t buf[kFlowWarps][kFlowBuf];
  __shared__ uint32_t sbits[kFlowWarps][kChTbl / 32];
  __shared__ uint32_t cbits[kFlowWarps][kChTbl / 32];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (!only) {
    flow_scan_one(gw, s, m, Js, strag_trip, trip_t, delta_a, skew, k, M, slot_group, rs, gi,
                  aff_flag, fs, err, buf, sbits, cbits);
    return;
  }
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = gw; i < static_cast<int64_t>(*n_only); i += nw)
    flow_scan_one(only[i], s, m, Js, strag_trip, trip_t, delta_a, skew, k, M, slot_group, rs,
                  gi, aff_flag, fs, err, buf, sbits, cbits);
}

// k_flow over the flow index: the member's window records of the group are
// staged once in shared memory in (op, store order) order — the segment's
// own order when its op_seq never descends, else the flow index's — and
// both rules walk the staged op runs: (a) per op the lower median of the
// window completions' durations and the first (store order) one above
// skew x median; (b) per window state op the state channels and, by a range
// lookup in the flow index, the op's prefix completions of the group
// ("completed_channels" covers the whole prefix, not just the window). A
// member whose window exceeds the staging area takes k_flow's scans.
constexpr int kFlowStage = 256;
constexpr int kFlow2Warps = 4;
__global__ void __launch_bounds__(kFlow2Warps * 32)
    k_flow_fi(StoreView s, FlowView fv, ModelView m, int32_t Js,
              const int32_t* __restrict__ strag_trip, const double* __restrict__ trip_t,
              double delta_a, double skew, int32_t k, uint32_t M,
              const uint32_t* __restrict__ slot_group, const RankSum* __restrict__ rs,
              const GroupIter* __restrict__ gi, const uint8_t* __restrict__ aff_flag,
              FlowSum* __restrict__ fs, uint32_t* __restrict__ err,
              uint32_t* __restrict__ spill, unsigned* __restrict__ n_spill) {
  __shared__ uint32_t sp[kFlow2Warps][kFlowStage];   // staged rank-major positions
  __shared__ uint32_t sbits[kFlow2Warps][kChTbl / 32];
  __shared__ uint32_t cbits[kFlow2Warps][kChTbl / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= static_cast<int64_t>(M) * Js) return;
  const int32_t js = static_cast<int32_t>(w / M);
  const uint32_t slot = static_cast<uint32_t>(w % M);
  const int32_t g = static_cast<int32_t>(slot_group[slot]);
  const int32_t j = strag_trip[js];
  FlowSum out;
  memset(&out, 0, sizeof(out));
  const uint64_t gidx = static_cast<uint64_t>(js) * m.n_groups + g;
  const bool run = aff_flag[static_cast<uint64_t>(j) * m.n_groups + g] &&
                   m.member_off[g + 1] - m.member_off[g] >= 2 &&
                   gi[gidx].n_common >= k && m.member_slot[slot] == slot;
  const int32_t r = m.members[slot];
  if (!run || r < 0 || r >= s.R) {
    if (lane == 0) fs[static_cast<uint64_t>(js) * M + slot] = out;
    return;
  }
  const double t = trip_t[j];
  const double ws = t - delta_a;
  const uint32_t b = s.rank_off[r], se = s.rank_off[r + 1];
  const uint32_t e = min(b + rs[static_cast<uint64_t>(j) * s.R + r].cutoff, se);
  const uint32_t p0 = min(seg_first(s, r, ws, false), e);
  const bool uns = fv.unsorted[r] != 0;
  auto win_rec = [&](uint32_t p) -> int {  // 1 completion, 2 state, 0 neither
    if (s.comm[p] != g || s.ts[p] < ws) return 0;
    const uint8_t ko = s.ko[p];
    if (ko_kind(ko) == CSG_KIND_COMPLETION) return ko_opname(ko) != CSG_OP_RECV ? 1 : 0;
    const uint64_t pi = static_cast<uint64_t>(s.op[p]) % static_cast<uint64_t>(m.opn);
    return m.op_name[pi] != CSG_OP_RECV ? 2 : 0;
  };
  // stage the window records in (op, store order) order
  int n = 0;
  if (!uns) {
    for (uint32_t base = p0; base < e; base += 32) {
      const uint32_t p = base + lane;
      const bool ok = p < e && win_rec(p) != 0;
      const unsigned mm = __ballot_sync(FULL, ok);
      const int at = n + __popc(mm & ((1u << lane) - 1u));
      if (ok && at < kFlowStage) sp[wib][at] = p;
      n += __popc(mm);
    }
  } else {
    // unsorted segment: the window's op range in flow order, filtered to
    // prefix positions at or after p0 (positions before p0 are all < ws)
    long long lo = LLONG_MAX, hi = LLONG_MIN;
    for (uint32_t p = p0 + lane; p < e; p += 32)
      if (win_rec(p)) {
        lo = min(lo, static_cast<long long>(s.op[p]));
        hi = max(hi, static_cast<long long>(s.op[p]));
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(FULL, lo, o));
      hi = max(hi, __shfl_xor_sync(FULL, hi, o));
    }
    if (lo <= hi) {
      const uint32_t fo = warp_partition_point(b, se, [&](uint32_t i) {
        return s.op[fv.at(true, i)] >= lo;
      });
      const uint32_t fe = warp_partition_point(fo, se, [&](uint32_t i) {
        return s.op[fv.at(true, i)] > hi;
      });
      for (uint32_t base = fo; base < fe; base += 32) {
        const uint32_t i = base + lane;
        uint32_t p = 0;
        bool ok = false;
        if (i < fe) {
          p = fv.at(true, i);
          ok = p >= p0 && p < e && win_rec(p) != 0;
        }
        const unsigned mm = __ballot_sync(FULL, ok);
        const int at = n + __popc(mm & ((1u << lane) - 1u));
        if (ok && at < kFlowStage) sp[wib][at] = p;
        n += __popc(mm);
      }
    }
  }
  __syncwarp();
  if (n > kFlowStage) {  // the scan kernel's path for this member
    if (lane == 0) {
      const unsigned at = atomicAdd(n_spill, 1u);
      spill[at] = static_cast<uint32_t>(w);
    }
    return;
  }
  const uint32_t* st = sp[wib];
  auto dur = [&](uint32_t p) { return s.ts[p] - as_double(s.pa[p]); };
  // (a) FlowSkewed: first op (ascending) with a skewed window flow
  for (int q0 = 0; q0 < n;) {
    const int64_t op = s.op[st[q0]];
    int q1 = q0 + 1;
    while (q1 < n && s.op[st[q1]] == op) ++q1;
    // completions of this op, store order
    int nc = 0;
    for (int q = q0; q < q1; ++q) nc += s.ko[st[q]] & 1 ? 0 : 1;  // CSG_KIND_COMPLETION == 0
    if (nc >= 2) {
      auto cv = [&](int i) {  // i-th completion of the run
        int c = -1;
        for (int q = q0; q < q1; ++q)
          if (!(s.ko[st[q]] & 1) && ++c == i) return dur(st[q]);
        return 0.0;
      };
      const double med = warp_lower_median(nc, cv);
      int hit = -1;
      if (med > 0) {
        const double lim = __dmul_rn(skew, med);
        for (int base = 0; base < nc && hit < 0; base += 32) {
          const int i = base + lane;
          const unsigned mm = __ballot_sync(FULL, i < nc && cv(i) > lim);
          if (mm) hit = base + __ffs(mm) - 1;
        }
      }
      if (hit >= 0) {
        int c = -1;
        uint32_t p = 0;
        for (int q = q0; q < q1; ++q)
          if (!(s.ko[st[q]] & 1) && ++c == hit) p = st[q];
        out.flags |= 1;
        out.skew_op = op;
        out.skew_chan = s.chan[p];
        out.skew_start = as_double(s.pa[p]);
        out.skew_end = s.ts[p];
        break;
      }
    }
    q0 = q1;
  }
  // (b) FlowIncomplete: first window state op (ascending) with a state
  // channel left incomplete while another completed
  const int words = (s.nch + 31) / 32;
  for (int q0 = 0; q0 < n;) {
    const int64_t op = s.op[st[q0]];
    int q1 = q0 + 1;
    while (q1 < n && s.op[st[q1]] == op) ++q1;
    bool has_state = false;
    for (int q = q0; q < q1 && !has_state; ++q) has_state = s.ko[st[q]] & 1;
    if (has_state) {
      for (int q = lane; q < words; q += 32) {
        sbits[wib][q] = 0;
        cbits[wib][q] = 0;
      }
      __syncwarp();
      for (int q = q0 + lane; q < q1; q += 32)
        if (s.ko[st[q]] & 1) {
          const int32_t ch = s.chan[st[q]];
          atomicOr(&sbits[wib][ch >> 5], 1u << (ch & 31));
        }
      // prefix completions of (r, op) in the group: the op's flow-index range
      const uint32_t fo = warp_partition_point(b, se, [&](uint32_t i) {
        return s.op[fv.at(uns, i)] >= op;
      });
      const uint32_t fe = warp_partition_point(fo, se, [&](uint32_t i) {
        return s.op[fv.at(uns, i)] > op;
      });
      for (uint32_t i = fo + lane; i < fe; i += 32) {
        const uint32_t p = fv.at(uns, i);
        const uint8_t ko = s.ko[p];
        if (p < e && ko_kind(ko) == CSG_KIND_COMPLETION && ko_opname(ko) != CSG_OP_RECV &&
            s.comm[p] == g) {
          const int32_t ch = s.chan[p];
          atomicOr(&cbits[wib][ch >> 5], 1u << (ch & 31));
        }
      }
      __syncwarp();
      bool any = false;
      int first = -1;
      for (int q = 0; q < words; ++q) {
        const uint32_t sb = sbits[wib][q], cb = cbits[wib][q];
        any |= (sb & cb) != 0;
        if (first < 0 && (sb & ~cb)) first = q * 32 + __ffs(sb & ~cb) - 1;
      }
      __syncwarp();
      if (any && first >= 0) {
        out.flags |= 2;
        out.inc_op = op;
        out.inc_chan = first;
        break;
      }
    }
    q0 = q1;
  }
  (void)err;
  if (lane == 0) fs[static_cast<uint64_t>(js) * M + slot] = out;
}

// ---------------------------------------------------------------------------
// K6: per-trip decision (one block per trip).
// ---------------------------------------------------------------------------
// Straggler trip state carried from candidate generation (k_decide phase
// 1) through the parallel self-evidence filter (k_self_faulted) to the
// report (k_decide phase 2).
struct StragState {
  int32_t C;  // candidates (0: decided in phase 1, -1: aborted)
  int32_t any_history;
  uint32_t cev_used, pad;
  unsigned long long cand_base, cev_base, sus_base, exo_base, ev_base, cap_cand, cap_cev;
};

struct DecideArgs {
  int debug;
  int phase;             // 1: candidates, 2: filter + report
  StragState* state;     // [J]
  uint32_t* sf_scratch;  // per k_self_faulted block
  uint32_t sf_words;
  // batch-wide cohort-median table (open addressing, power-of-two capacity)
  unsigned long long* coh_key;  // ~0 = empty
  double* coh_val;
  unsigned* coh_state;          // 2 = value published
  longlong2* coh_meta;          // claimed slot: {iteration, trip << 8 | op name}
  // per (op name, iteration) over all entries: median, latest timestamp
  unsigned long long* coh2_key;
  double* coh2_val;
  double* coh2_mx;
  unsigned* coh2_state;
  uint32_t coh_cap;
  StoreView s;
  ModelView m;
  int32_t J;
  const double* trip_t;
  const int32_t* trip_kind;
  const int32_t* trip_rank;
  const int32_t* js_of;
  const RankSum* rs;
  const unsigned long long* chan_key;
  int32_t nch;
  const int32_t* aff;
  const int32_t* n_aff;
  const GroupIter* gi;
  const int64_t* gi_last;
  int32_t k;
  const FlowSum* fs;
  const unsigned long long* tbl_s;
  const unsigned long long* tbl_e;
  int64_t it_min;
  int32_t n_it;
  uint32_t M;
  double delta_a, thr, skew;
  uint64_t N;
  const uint64_t* opk;
  const int32_t* oprank;
  const double* op_ts;
  const double* op_dur;
  const uint8_t* op_nm;
  uint64_t n_opidx;
  int sharded;
  int64_t min_op, max_op;
  // sorted self-evidence path (k_sf_prep / k_opsort / k_sf_fast): per op
  // key (op - min_op) the op index segment [opoff[k], opoff[k+1]), its
  // durations sorted ascending as ordered keys (sdur, same positions) and
  // the segment's latest timestamp (opmax; NaN = not sorted)
  FlowView f;
  const uint32_t* opoff;
  unsigned long long* sdur;
  double* sts;     // timestamps of the sorted entries
  int32_t* srank;  // ranks of the sorted entries
  double* opmax;
  struct SfPlan* plan;
  int64_t* pend_ops;  // [candidate][kSfPend] ops waiting for a cohort (k_sf_fast)
  uint8_t* pend_n;
  int sf_fast;  // k_self_faulted takes only the candidates k_sf_fast deferred
  // parallel straggler candidates (k_sl_*): per (straggler trip, membership
  // slot) lateness | flow-candidate bits, per (straggler trip, affected
  // group index) candidate / evidence counts, then offsets
  uint32_t* emit_rank;  // per trip: per-rank first position, rank bitmap, offsets
  uint64_t emit_stride;
  int sl_par;
  const int32_t* strag_trip;
  uint8_t* sl_late;
  uint2* sl_cnt;
  uint32_t scratch_per_trip;  // u32 words
  Pools pools;
  TripOut* out;
  uint32_t* err;
};

enum { P_CAND = 0, P_CEV = 1, P_SUS = 2, P_EV = 3, P_BITS = 4 };

struct BlockShared {
  int abort;
  uint32_t dbg_n, dbg_d;  // self_faulted sizes (CSG_DEBUG_EXO)
  // per-block cache of cohort medians (trip, iteration, op name) -> median
  // (rca.cpp:833-840: the cohort does not depend on the candidate)
  int32_t coh_n;
  unsigned long long coh_key[32];
  double coh_val[32];
  int32_t ncand;
  uint32_t cev_used;
  int32_t nret;
  int32_t nexo;
  int32_t nsus;
  uint32_t nev;
  unsigned long long cand_base, cev_base, sus_base, exo_base, ev_base,
      bits_base;
  unsigned long long cap_cand, cap_cev;
  int64_t i64a, i64b;
  int32_t i32a, i32b, i32c;
  uint64_t u64a, u64b, u64c;
  double med_s[kMaxK], med_e[kMaxK];
  int64_t win[kMaxK];
  int32_t red_i[32];
  long long red_l[32];
  unsigned long long red_u[3][32];
  uint32_t chtbl[kChTbl];
  uint32_t hist[256];
};

__device__ unsigned long long pool_alloc(unsigned long long* used, int which,
                                         unsigned long long n,
                                         unsigned long long cap, uint32_t* err,
                                         uint32_t flag, bool* ok) {
  const unsigned long long b = atomicAdd(&used[which], n);
  *ok = b + n <= cap;
  if (!*ok) atomicOr(err, flag);
  return b;
}

__device__ int block_sum_i(int v, BlockShared& sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  __syncthreads();
  if (lane == 0) sh.red_i[warp] = v;
  __syncthreads();
  int t = 0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh.red_i[i];
  __syncthreads();
  return t;
}

// Stable order-preserving compaction of pred over [0, n) into dst (block).
template <typename P>
__device__ int block_compact(int n, P pred, uint32_t* dst, BlockShared& sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  int base = 0;
  for (int i0 = 0; i0 < n; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    const int hit = (i < n && pred(i)) ? 1 : 0;
    const unsigned mm = __ballot_sync(FULL, hit);
    __syncthreads();
    if (lane == 0) sh.red_i[warp] = __popc(mm);
    __syncthreads();
    int before = 0, total = 0;
    for (int q = 0; q < nw; ++q) {
      if (q < warp) before += sh.red_i[q];
      total += sh.red_i[q];
    }
    if (hit) dst[base + before + __popc(mm & ((1u << lane) - 1u))] = i;
    base += total;
  }
  __syncthreads();
  return base;
}

// Stable placement sort of n items by a strict-weak "less(a, b)" on item
// indices: out[pos(i)] = in[i] where pos = #less + #equal-before.
template <typename L>
__device__ void block_stable_sort(int n, const uint32_t* in, uint32_t* out,
                                  L less) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int pos = 0;
    const uint32_t a = in[i];
    for (int q = 0; q < n; ++q) {
      const uint32_t b = in[q];
      if (less(b, a) || (q < i && !less(a, b))) ++pos;
    }
    out[pos] = a;
  }
  __syncthreads();
}

// k-th smallest of a virtual list (radix select on ordered double keys).
// get(i, &key) returns false for excluded items.
template <typename G>
__device__ double block_select(uint64_t n, uint64_t kth, G get,
                               BlockShared& sh) {
  uint64_t prefix = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh.hist[i] = 0;
    __syncthreads();
    const uint64_t mask = shift == 56 ? 0ull : (~0ull << (shift + 8));
    // warp-aggregated digit counts: skewed key sets (durations share their
    // top bytes) would serialise on one shared-memory counter otherwise
    for (uint64_t b0 = 0; b0 < n; b0 += blockDim.x) {
      const uint64_t i = b0 + threadIdx.x;
      uint32_t d = 256;
      uint64_t key;
      if (i < n && get(i, &key) && (key & mask) == (prefix & mask))
        d = static_cast<uint32_t>((key >> shift) & 255);
      const unsigned peers = __match_any_sync(FULL, d);
      if (d < 256 && (threadIdx.x & 31) == __ffs(peers) - 1)
        atomicAdd(&sh.hist[d], static_cast<uint32_t>(__popc(peers)));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t acc = 0;
      int bsel = 255;
      for (int bk = 0; bk < 256; ++bk) {
        if (acc + sh.hist[bk] > kth) {
          bsel = bk;
          break;
        }
        acc += sh.hist[bk];
      }
      sh.u64a = prefix | (static_cast<uint64_t>(bsel) << shift);
      sh.u64b = kth - acc;
    }
    __syncthreads();
    prefix = sh.u64a;
    kth = sh.u64b;
    __syncthreads();
  }
  return dkey_inv(prefix);
}

__device__ void write_trip(const DecideArgs& a, int32_t j, int verdict,
                           int32_t naff, uint64_t scanned, BlockShared& sh) {
  if (threadIdx.x == 0) {
    TripOut o;
    o.verdict = verdict;
    o.n_aff = naff;
    o.scanned = scanned;
    o.sus_off = static_cast<uint32_t>(sh.sus_base);
    o.n_sus = sh.nsus;
    o.exo_off = static_cast<uint32_t>(sh.exo_base);
    o.n_exo = sh.nexo;
    o.ev_off = static_cast<uint32_t>(sh.ev_base);
    o.n_ev = sh.nev;
    a.out[j] = o;
  }
}

__device__ csg_suspect to_suspect(const Cand& c) {
  csg_suspect s;
  s.rank = c.rank;
  s.category = c.cat;
  s.side = c.side;
  s.reserved = 0;
  s.group = c.group;
  s.reserved2 = 0;
  s.stuck_op = c.op;
  s.onset_ms = c.onset;
  return s;
}

// Appends one evidence ref to the current candidate (thread 0 only).
__device__ void add_cev(const DecideArgs& a, BlockShared& sh, Cand& c,
                        int32_t rank, int32_t ch, double tms, int64_t op) {
  if (sh.cev_used >= sh.cap_cev) {
    atomicOr(a.err, DEV_ERR_POOL);
    sh.abort = 1;
    return;
  }
  csg_evidence e;
  e.rank = rank;
  e.channel = ch;
  e.time_ms = tms;
  e.op_seq = op;
  a.pools.cev[sh.cev_base + sh.cev_used] = e;
  ++sh.cev_used;
  ++c.ev_n;
}

__device__ void push_cand(const DecideArgs& a, BlockShared& sh, const Cand& c) {
  if (sh.ncand >= static_cast<int32_t>(sh.cap_cand)) {
    atomicOr(a.err, DEV_ERR_POOL);
    sh.abort = 1;
    return;
  }
  a.pools.cand[sh.cand_base + sh.ncand] = c;
  ++sh.ncand;
}

// Final assembly shared by both analyzers: given candidates (in append
// order) and a keep mask / exoneration decisions already made by the
// caller in sorted order (ord/keep), emit exonerated + de-duplicated
// suspects (first per rank wins, evidence in candidate order) and sort the
// suspects by rank (stable).
__device__ void emit_reports(const DecideArgs& a, BlockShared& sh,
                             const uint32_t* ord, const uint8_t* keep, int C,
                             uint32_t* scratch) {
  const Cand* cands = a.pools.cand + sh.cand_base;
  // first-retained-per-rank flags
  uint8_t* first = reinterpret_cast<uint8_t*>(scratch);
  for (int x = threadIdx.x; x < C; x += blockDim.x) {
    uint8_t f = 0;
    if (keep[x]) {
      f = 1;
      const int32_t r = cands[ord[x]].rank;
      for (int y = 0; y < x; ++y)
        if (keep[y] && cands[ord[y]].rank == r) {
          f = 0;
          break;
        }
    }
    first[x] = f;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int nsus = 0, nexo = 0;
    uint32_t nev = 0;
    for (int x = 0; x < C; ++x) {
      const Cand& c = cands[ord[x]];
      if (!keep[x]) {
        a.pools.sus[sh.exo_base + nexo++] = to_suspect(c);
      } else if (first[x]) {
        a.pools.sus[sh.sus_base + nsus++] = to_suspect(c);
        for (uint32_t q = 0; q < c.ev_n; ++q)
          a.pools.ev[sh.ev_base + nev++] = a.pools.cev[sh.cev_base + c.ev_off + q];
      }
    }
    sh.nsus = nsus;
    sh.nexo = nexo;
    sh.nev = nev;
  }
  __syncthreads();
  // stable sort suspects by rank
  csg_suspect* sus = a.pools.sus + sh.sus_base;
  const int ns = sh.nsus;
  uint32_t* idx = scratch;
  uint32_t* srt = scratch + ns;
  for (int i = threadIdx.x; i < ns; i += blockDim.x) idx[i] = i;
  __syncthreads();
  block_stable_sort(ns, idx, srt, [&](uint32_t x, uint32_t y) {
    return sus[x].rank < sus[y].rank;
  });
  csg_suspect* tmp = a.pools.sus + sh.exo_base + sh.nexo;  // spare room
  for (int i = threadIdx.x; i < ns; i += blockDim.x) tmp[i] = sus[srt[i]];
  __syncthreads();
  for (int i = threadIdx.x; i < ns; i += blockDim.x) sus[i] = tmp[i];
  __syncthreads();
}

// ---- failure: see k_fail_count / k_fail_cands / k_exonerate ---------------

// ---- straggler -------------------------------------------------------------

// op-index segment [lo_key, hi_key] (keys = op - min_op), block-uniform;
// warp 0 searches with 32-ary probes (a handful of dependent rounds over the
// ~1e8-entry index instead of ~27 by one thread)
__device__ void op_segment(const DecideArgs& a, uint64_t k0, uint64_t k1,
                           bool empty, BlockShared& sh, uint64_t& sb,
                           uint64_t& se) {
  if (threadIdx.x < 32) {
    auto first = [&](uint64_t lo, uint64_t hi, auto pred) {
      const int lane = threadIdx.x;
      while (hi - lo > 32) {
        const uint64_t len = hi - lo, step = (len + 31) / 32;
        uint64_t off = (lane + 1) * step;
        if (off > len) off = len;
        const unsigned mm = __ballot_sync(FULL, pred(lo + off - 1));
        if (!mm) return hi;
        const int f = __ffs(mm) - 1;
        uint64_t offf = (f + 1) * step;
        if (offf > len) offf = len;
        const uint64_t qf = lo + offf - 1;
        if (f) {
          uint64_t offp = f * step;
          if (offp > len) offp = len;
          lo = lo + offp;
        }
        hi = qf;
      }
      const uint64_t q = lo + lane;
      const unsigned mm = __ballot_sync(FULL, q < hi && pred(q));
      return mm ? lo + __ffs(mm) - 1 : hi;
    };
    const uint64_t l = first(0, a.n_opidx, [&](uint64_t i) { return a.opk[i] >= k0; });
    const uint64_t h = empty ? l : first(l, a.n_opidx, [&](uint64_t i) { return a.opk[i] > k1; });
    if (threadIdx.x == 0) {
      sh.u64a = l;
      sh.u64b = h;
    }
  }
  __syncthreads();
  sb = sh.u64a;
  se = sh.u64b;
  __syncthreads();
}

// Lower median of the qualifying keys of a range in one pass: keys staged
// in shared memory (up to 2048), bitonic-sorted there, element (m-1)/2
// returned with the count m. Ranges with more qualifying keys fall back to
// the radix select (count in *m; caller handles m == 0). Block-collective.
template <typename G>
__device__ double staged_lower_median(uint64_t n, G get, BlockShared& sh, int* m_out) {
  constexpr uint32_t kCap = kChTbl / 2;  // u64 keys in sh.chtbl
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(sh.chtbl);
  __shared__ uint32_t s_n;
  __shared__ int s_over;
  if (threadIdx.x == 0) {
    s_n = 0;
    s_over = 0;
  }
  __syncthreads();
  for (uint64_t b0 = 0; b0 < n; b0 += blockDim.x) {
    const uint64_t i = b0 + threadIdx.x;
    uint64_t key = 0;
    const bool ok = i < n && get(i, &key);
    const unsigned mm = __ballot_sync(FULL, ok);  // one counter update per warp
    uint32_t at = 0;
    if ((threadIdx.x & 31) == 0 && mm) at = atomicAdd(&s_n, static_cast<uint32_t>(__popc(mm)));
    at = __shfl_sync(FULL, at, 0) + __popc(mm & ((1u << (threadIdx.x & 31)) - 1u));
    if (ok) {
      if (at < kCap) keys[at] = key; else s_over = 1;
    }
  }
  __syncthreads();
  const uint32_t m = s_n;
  *m_out = static_cast<int>(m);
  if (m == 0) return 0;
  if (s_over) {
    __syncthreads();
    return block_select(n, static_cast<uint64_t>((m - 1) / 2), get, sh);
  }
  uint32_t P = 1;
  while (P < m) P <<= 1;
  for (uint32_t i = m + threadIdx.x; i < P; i += blockDim.x) keys[i] = ~0ull;
  __syncthreads();
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
      for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
        const uint32_t l = i ^ jj;
        if (l > i) {
          const unsigned long long x = keys[i], y = keys[l];
          if ((x > y) == ((i & k) == 0)) {
            keys[i] = y;
            keys[l] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  const double r = dkey_inv(keys[(m - 1) / 2]);
  __syncthreads();
  return r;
}

// Lower median (index kth of the qualifying keys) of a small candidate set:
// keys staged in shared memory, then one rank count per key (O(n^2 / T));
// larger sets go through the radix select.
template <typename G>
__device__ double small_select(uint64_t n, uint64_t kth, G get, BlockShared& sh) {
  constexpr uint32_t kCap = 512;  // O(n^2 / T) beats the radix passes below this
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(sh.chtbl);
  if (n > kCap) return block_select(n, kth, get, sh);
  __shared__ uint32_t s_n;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  for (uint64_t b0 = 0; b0 < n; b0 += blockDim.x) {
    const uint64_t i = b0 + threadIdx.x;
    uint64_t key = 0;
    const bool ok = i < n && get(i, &key);
    const unsigned mm = __ballot_sync(FULL, ok);
    uint32_t at = 0;
    if ((threadIdx.x & 31) == 0 && mm) at = atomicAdd(&s_n, static_cast<uint32_t>(__popc(mm)));
    at = __shfl_sync(FULL, at, 0) + __popc(mm & ((1u << (threadIdx.x & 31)) - 1u));
    if (ok) keys[at] = key;
  }
  __syncthreads();
  const uint32_t m = s_n;
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
    const unsigned long long v = keys[i];
    uint32_t less = 0, leq = 0;
    for (uint32_t q = 0; q < m; ++q) {
      less += keys[q] < v;
      leq += keys[q] <= v;
    }
    if (less <= kth && kth < leq) sh.u64c = v;
  }
  __syncthreads();
  const double r = dkey_inv(sh.u64c);
  __syncthreads();
  return r;
}

// op range holding exactly the ops with static_cast<long>(op / opn) == it
// (C++ division truncates toward zero, so iteration 0 also holds (-opn, 0))
__device__ inline void iter_ops(int64_t it, int32_t opn, int64_t& lo, int64_t& hi) {
  lo = it > 0 ? it * opn : it * opn - (opn - 1);
  hi = it >= 0 ? it * opn + (opn - 1) : it * opn;
}

// Lower median of the (program op name nm, iteration it) cohort of non-Recv
// completions with ts <= t (rca.cpp:833-840); 0 when fewer than two (the
// caller skips the op). Block-collective.
__device__ double cohort_median(const DecideArgs& a, int64_t it, uint8_t nm, double t,
                                BlockShared& sh) {
  int64_t olo, ohi;
  iter_ops(it, a.m.opn, olo, ohi);
  const bool empty = ohi < a.min_op;
  const uint64_t k0 = olo < a.min_op ? 0 : static_cast<uint64_t>(olo - a.min_op);
  const uint64_t k1 = empty ? 0 : static_cast<uint64_t>(ohi - a.min_op);
  uint64_t cb, ce;
  op_segment(a, k0, k1, empty, sh, cb, ce);
  int nco = 0;
  const double med = staged_lower_median(ce - cb,
                                         [&](uint64_t i, uint64_t* key) {
                                           const uint64_t y = cb + i;
                                           if (a.op_nm[y] != nm || a.op_ts[y] > t) return false;
                                           *key = dkey(a.op_dur[y]);
                                           return true;
                                         },
                                         sh, &nco);
  return nco < 2 ? 0 : med;
}

// self_faulted (rca.cpp:821-848) for one lateness candidate. "mine" are the
// candidate rank's completions (ts <= t, not Recv) in its iteration window:
// from its rank-major segment on a single GPU, from the (gathered) op index
// when the store is sharded; sibling and cohort medians always come from the
// op index, which then holds every shard's entries.
__device__ bool self_faulted(const DecideArgs& a, int32_t j, const Cand& c,
                             BlockShared& sh, uint32_t* lst) {
  const double t = a.trip_t[j];
  const int32_t r = c.rank;
  const int32_t opn = a.m.opn;
  int n = 0;
  uint64_t mb = 0;  // op-index base of the "mine" scan (sharded form)
  if (!a.sharded) {
    if (r < 0 || r >= a.s.R) return false;
    const uint32_t b = a.s.rank_off[r], e = a.s.rank_off[r + 1];
    mb = b;
    n = block_compact(static_cast<int>(e - b), [&](int i) {
      const uint32_t p = b + i;
      const uint8_t ko = a.s.ko[p];
      if (ko_kind(ko) != CSG_KIND_COMPLETION || ko_opname(ko) == CSG_OP_RECV)
        return false;
      if (a.s.ts[p] > t) return false;
      const int64_t it = iter_of(a.s.op[p], opn);
      return it >= c.it_lo && it <= c.it_hi;
    }, lst, sh);
  } else {
    int64_t olo, ohi, x0, x1;
    iter_ops(c.it_lo, opn, olo, x1);
    iter_ops(c.it_hi, opn, x0, ohi);
    const bool empty = ohi < a.min_op;
    const uint64_t k0 = olo < a.min_op ? 0 : static_cast<uint64_t>(olo - a.min_op);
    const uint64_t k1 = empty ? 0 : static_cast<uint64_t>(ohi - a.min_op);
    uint64_t sb, se;
    op_segment(a, k0, k1, empty, sh, sb, se);
    mb = sb;
    n = block_compact(static_cast<int>(se - sb), [&](int i) {
      const uint64_t y = sb + i;
      return a.oprank[y] == r && a.op_ts[y] <= t;
    }, lst, sh);
  }
  auto mine_op = [&](int x) -> int64_t {
    return a.sharded ? static_cast<int64_t>(a.opk[mb + lst[x]]) + a.min_op
                     : a.s.op[mb + lst[x]];
  };
  auto mine_dur = [&](int x) -> double {
    if (a.sharded) return a.op_dur[mb + lst[x]];
    const uint32_t p = static_cast<uint32_t>(mb) + lst[x];
    return a.s.ts[p] - as_double(a.s.pa[p]);
  };
  if (threadIdx.x == 0) {
    sh.dbg_n = n;
    sh.dbg_d = 0;
  }
  for (int x = 0; x < n; ++x) {
    const int64_t o = mine_op(x);
    // per-channel completions of one op sit next to each other: the common
    // duplicate is decided without a block-wide pass
    if (x > 0 && mine_op(x - 1) == o) continue;
    bool dup = false;
    for (int y = threadIdx.x; y < x; y += blockDim.x) dup |= mine_op(y) == o;
    if (__syncthreads_or(dup)) continue;
    if (threadIdx.x == 0) ++sh.dbg_d;
    // max of my durations for op o
    double mine = -INFINITY;
    for (int y = x + threadIdx.x; y < n; y += blockDim.x)
      if (mine_op(y) == o) mine = fmax(mine, mine_dur(y));
    {
      unsigned long long kk = mine == -INFINITY ? 0ull : dkey(mine);
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
      for (int q = 16; q; q >>= 1) kk = max(kk, __shfl_xor_sync(FULL, kk, q));
      __syncthreads();
      if (lane == 0) sh.red_u[0][warp] = kk;
      __syncthreads();
      kk = 0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) kk = max(kk, sh.red_u[0][q]);
      __syncthreads();
      mine = dkey_inv(kk);
    }
    // siblings: other ranks' durations of op o (ts <= t)
    uint64_t sb, se;
    {
      const uint64_t key = static_cast<uint64_t>(o - a.min_op);
      op_segment(a, key, key, false, sh, sb, se);
    }
    int nsib = 0;
    double med = staged_lower_median(se - sb,
                                     [&](uint64_t i, uint64_t* key) {
                                       const uint64_t y = sb + i;
                                       if (a.oprank[y] == r || a.op_ts[y] > t) return false;
                                       *key = dkey(a.op_dur[y]);
                                       return true;
                                     },
                                     sh, &nsib);
    if (nsib > 0) {
    } else {
      // cohort of (program op name, iteration) (rca.cpp:833-840)
      const int64_t it = iter_of(o, opn);
      const uint8_t nm = a.m.op_name[static_cast<uint64_t>(o % opn)];
      const unsigned long long ckey =
          (static_cast<unsigned long long>(j) << 44) ^
          (static_cast<unsigned long long>(nm) << 36) ^
          (static_cast<unsigned long long>(it) & ((1ull << 36) - 1));
      // Block cache first, then the batch-wide table: the first block to need
      // a cohort claims its slot and computes it, later ones wait for the
      // published value (the claimer is running, so the wait terminates).
      __shared__ int s_hit, s_slot;
      __shared__ double s_med;
      if (threadIdx.x == 0) {
        s_hit = 0;
        s_slot = -1;
        for (int q = 0; q < sh.coh_n && q < 32; ++q)
          if (sh.coh_key[q] == ckey) {
            s_hit = 1;
            s_med = sh.coh_val[q];
          }
        if (!s_hit && a.coh_cap) {
          const uint32_t mask = a.coh_cap - 1;
          uint32_t h = static_cast<uint32_t>((ckey * 0x9E3779B97F4A7C15ull) >> 40) & mask;
          for (uint32_t probe = 0; probe < a.coh_cap; ++probe, h = (h + 1) & mask) {
            const unsigned long long k = atomicCAS(a.coh_key + h, ~0ull, ckey);
            if (k == ~0ull) {  // claimed: this block computes it
              s_slot = static_cast<int>(h);
              break;
            }
            if (k == ckey) {  // someone else's: wait for the value
              volatile unsigned* stv = a.coh_state + h;
              while (*stv < 2u) {
              }
              __threadfence();
              if (*stv == 2u) {  // 3: abandoned (k_coh_collect overflow), compute here
                s_med = *reinterpret_cast<volatile double*>(a.coh_val + h);
                s_hit = 1;
              }
              break;
            }
          }
        }
      }
      __syncthreads();
      if (s_hit) {
        med = s_med;
        if (threadIdx.x == 0 && sh.coh_n < 32) {
          sh.coh_key[sh.coh_n] = ckey;
          sh.coh_val[sh.coh_n++] = med;
        }
        __syncthreads();
        if (med <= 0) continue;
        if (mine > __dmul_rn(a.skew, med)) return true;
        continue;
      }
      __syncthreads();
      const double cm = cohort_median(a, it, nm, t, sh);
      const int nco = cm > 0 ? 2 : 0;  // non-positive: skip the op
      med = cm;
      if (threadIdx.x == 0) {
        const int q = sh.coh_n < 32 ? sh.coh_n++ : static_cast<int>(ckey % 32);
        sh.coh_key[q] = ckey;
        sh.coh_val[q] = med;
        if (s_slot >= 0) {  // publish
          a.coh_val[s_slot] = med;
          __threadfence();
          atomicExch(a.coh_state + s_slot, 2u);
        }
      }
      __syncthreads();
      if (nco < 2) continue;
    }
    if (med <= 0) continue;
    if (mine > __dmul_rn(a.skew, med)) return true;
  }
  return false;
}

// Lower median sorted[(n-1)/2] of n virtual values (block; O(n^2/threads)).
template <typename V>
__device__ double block_lower_median(int n, V val, BlockShared& sh) {
  const int k = (n - 1) / 2;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double vi = val(i);
    int less = 0, leq = 0;
    for (int q = 0; q < n; ++q) {
      const double vq = val(q);
      less += vq < vi;
      leq += vq <= vi;
    }
    if (less <= k && k < leq) {
      uint64_t u;
      memcpy(&u, &vi, 8);
      sh.u64c = u;
    }
  }
  __syncthreads();
  const double r = as_double(sh.u64c);
  __syncthreads();
  return r;
}

__device__ void decide_straggler(const DecideArgs& a, int32_t j,
                                 BlockShared& sh, uint32_t* scratch) {
  const int32_t naff = a.n_aff[j];
  const int32_t* aff = a.aff + static_cast<uint64_t>(j) * a.m.n_groups;
  const int32_t R = a.s.R;
  const double t = a.trip_t[j];
  const int32_t js = a.js_of[j];
  const long long clk_g0 = clock64();
  const int32_t k = a.k;
  const int32_t opn = a.m.opn;
  int tot = 0;
  for (int32_t i = threadIdx.x; i < naff; i += blockDim.x) {
    const int32_t g = aff[i];
    tot += static_cast<int>(a.m.member_off[g + 1] - a.m.member_off[g]);
  }
  tot = block_sum_i(tot, sh);
  if (threadIdx.x == 0) {
    bool ok1, ok2, ok3, ok4;
    sh.cap_cand = 2ull * tot;
    sh.cap_cev = static_cast<unsigned long long>(tot) * (k + 1);
    sh.cand_base = pool_alloc(a.pools.used, P_CAND, sh.cap_cand,
                              a.pools.cand_cap, a.err, DEV_ERR_POOL, &ok1);
    sh.cev_base = pool_alloc(a.pools.used, P_CEV, sh.cap_cev, a.pools.cev_cap,
                             a.err, DEV_ERR_POOL, &ok2);
    sh.sus_base = pool_alloc(a.pools.used, P_SUS, 3 * sh.cap_cand,
                             a.pools.sus_cap, a.err, DEV_ERR_POOL, &ok3);
    sh.exo_base = sh.sus_base + sh.cap_cand;
    sh.ev_base = pool_alloc(a.pools.used, P_EV, sh.cap_cev, a.pools.ev_cap,
                            a.err, DEV_ERR_POOL, &ok4);
    sh.abort = !(ok1 && ok2 && ok3 && ok4);
    sh.ncand = 0;
    sh.cev_used = 0;
  }
  __syncthreads();
  if (sh.abort) return;
  // scratch: already_candidate bitmap | A | B
  uint32_t* mark = scratch;
  const uint32_t mwords = static_cast<uint32_t>((R + 31) / 32 + 1);
  const uint32_t P = (a.scratch_per_trip - mwords) / 2;
  uint32_t* A = scratch + mwords;
  uint32_t* B = A + P;
  for (uint32_t i = threadIdx.x; i < mwords; i += blockDim.x) mark[i] = 0;
  __syncthreads();
  auto is_marked = [&](int32_t r) {
    return r >= 0 && r < R && ((mark[r >> 5] >> (r & 31)) & 1u);
  };
  auto set_mark = [&](int32_t r) {
    if (r >= 0 && r < R) mark[r >> 5] |= 1u << (r & 31);
  };
  bool any_history = false;
  const uint64_t rowbase = static_cast<uint64_t>(js) * a.M;
  for (int32_t ai = 0; ai < naff; ++ai) {
    const int32_t g = aff[ai];
    const uint32_t mo = a.m.member_off[g];
    const int32_t m = static_cast<int32_t>(a.m.member_off[g + 1] - mo);
    if (m < 2) continue;
    const uint64_t gidx = static_cast<uint64_t>(js) * a.m.n_groups + g;
    if (a.gi[gidx].n_common < k) continue;
    any_history = true;
    const int64_t gfo = a.m.group_first_op[g];
    for (int q = threadIdx.x; q < k; q += blockDim.x)
      sh.win[q] = a.gi_last[gidx * k + q];
    __syncthreads();
    auto cell = [&](int i, int q) {
      return (rowbase + a.m.member_slot[mo + i]) * a.n_it +
             static_cast<uint64_t>(sh.win[q] - a.it_min);
    };
    // lower medians of starts / ends per window iteration (rca.cpp:670-681)
    for (int q = 0; q < k; ++q) {
      const double ms = block_lower_median(
          m, [&](int i) { return dkey_inv(a.tbl_s[cell(i, q)]); }, sh);
      const double me = block_lower_median(
          m, [&](int i) { return dkey_inv(a.tbl_e[cell(i, q)]); }, sh);
      if (threadIdx.x == 0) {
        sh.med_s[q] = ms;
        sh.med_e[q] = me;
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      bool sl = true, el = true;
      for (int q = 0; q < k; ++q) {
        if (dkey_inv(a.tbl_s[cell(i, q)]) - sh.med_s[q] < a.thr) sl = false;
        if (dkey_inv(a.tbl_e[cell(i, q)]) - sh.med_e[q] < a.thr) el = false;
      }
      A[i] = (sl ? 1u : 0u) | (el ? 2u : 0u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 0; i < m && !sh.abort; ++i) {
        if (!A[i]) continue;
        const int32_t r = a.m.members[mo + i];
        Cand c;
        memset(&c, 0, sizeof(c));
        c.rank = r;
        c.cat = (A[i] & 1u) ? CSG_RC_STRAGGLER_LATE_START
                            : CSG_RC_STRAGGLER_LATE_END;
        c.side = CSG_SIDE_LOCAL;
        c.group = g;
        c.op = sh.win[k - 1] * opn + gfo;
        c.onset = dkey_inv(a.tbl_s[cell(i, 0)]);
        c.it_lo = sh.win[0];
        c.it_hi = sh.win[k - 1];
        c.ev_off = sh.cev_used;
        for (int q = 0; q < k; ++q)
          add_cev(a, sh, c, r, -1, dkey_inv(a.tbl_s[cell(i, q)]),
                  sh.win[q] * opn + gfo);
        set_mark(r);
        push_cand(a, sh, c);
      }
    }
    __syncthreads();
    if (sh.abort) return;
    // flow-level supplement: (rank, op) map order == ascending rank
    for (int i = threadIdx.x; i < m; i += blockDim.x) A[i] = i;
    __syncthreads();
    block_stable_sort(m, A, B, [&](uint32_t x, uint32_t y) {
      return a.m.members[mo + x] < a.m.members[mo + y];
    });
    if (threadIdx.x == 0) {
      for (int pass = 0; pass < 2 && !sh.abort; ++pass) {
        for (int x = 0; x < m && !sh.abort; ++x) {
          const uint32_t i = B[x];
          const int32_t r = a.m.members[mo + i];
          if (r < 0 || r >= R || is_marked(r)) continue;
          const FlowSum f = a.fs[static_cast<uint64_t>(js) * a.M +
                                 a.m.member_slot[mo + i]];
          Cand c;
          memset(&c, 0, sizeof(c));
          c.rank = r;
          c.side = CSG_SIDE_LOCAL;
          c.group = g;
          c.it_lo = 0;
          c.it_hi = -1;
          c.ev_off = sh.cev_used;
          if (pass == 0 && (f.flags & 1)) {
            c.cat = CSG_RC_FLOW_SKEWED;
            c.op = f.skew_op;
            c.onset = f.skew_start;
            add_cev(a, sh, c, r, f.skew_chan, f.skew_end, f.skew_op);
          } else if (pass == 1 && (f.flags & 2)) {
            c.cat = CSG_RC_FLOW_INCOMPLETE;
            c.op = f.inc_op;
            c.onset = t;
            add_cev(a, sh, c, r, f.inc_chan, t, f.inc_op);
          } else {
            continue;
          }
          set_mark(r);
          push_cand(a, sh, c);
        }
      }
    }
    __syncthreads();
    if (sh.abort) return;
  }
  const int C = sh.ncand;
  if (C == 0) {
    write_trip(a, j,
               any_history ? CSG_VERDICT_NO_STRAGGLER
                           : CSG_VERDICT_INSUFFICIENT_HISTORY,
               naff, 2 * a.N, sh);
    if (threadIdx.x == 0) a.state[j].C = 0;
    return;
  }
  // the self-evidence filter (rca.cpp:795-869) runs in k_self_faulted, one
  // block per candidate over every straggler trip
  if (threadIdx.x == 0) {
    StragState& S = a.state[j];
    S.C = C;
    S.any_history = any_history ? 1 : 0;
    S.cev_used = sh.cev_used;
    S.cand_base = sh.cand_base;
    S.cev_base = sh.cev_base;
    S.sus_base = sh.sus_base;
    S.exo_base = sh.exo_base;
    S.ev_base = sh.ev_base;
    S.cap_cand = sh.cap_cand;
    S.cap_cev = sh.cap_cev;
  }
}

// Candidate order for the report (rca.cpp:850-853: stable sort by
// (stuck_op, rank)) as a bitonic sort of packed (op - min op, rank, index)
// keys in the trip's scratch; the O(C^2) rank-count sort when the packing
// does not fit.
__device__ void strag_order(const DecideArgs& a, const Cand* cands, int C, uint32_t* A,
                            uint32_t P, uint32_t* ord, BlockShared& sh) {
  long long mn = LLONG_MAX, mx = LLONG_MIN;
  int rmax = 0;
  for (int x = threadIdx.x; x < C; x += blockDim.x) {
    mn = min(mn, static_cast<long long>(cands[x].op));
    mx = max(mx, static_cast<long long>(cands[x].op));
    rmax = max(rmax, cands[x].rank);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(FULL, mn, o));
    mx = max(mx, __shfl_xor_sync(FULL, mx, o));
    rmax = max(rmax, __shfl_xor_sync(FULL, rmax, o));
  }
  __syncthreads();
  if (lane == 0) {
    sh.red_l[warp] = mn;
    sh.red_u[0][warp] = static_cast<unsigned long long>(mx);
    sh.red_i[warp] = rmax;
  }
  __syncthreads();
  mn = LLONG_MAX;
  mx = LLONG_MIN;
  rmax = 0;
  for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) {
    mn = min(mn, sh.red_l[q]);
    mx = max(mx, static_cast<long long>(sh.red_u[0][q]));
    rmax = max(rmax, sh.red_i[q]);
  }
  __syncthreads();
  int ib = 1, rb = 1;
  while ((1ll << ib) < C) ++ib;
  while ((1ll << rb) <= rmax) ++rb;
  const int ob = 64 - ib - rb;
  uint32_t Pw = 1;
  while (Pw < static_cast<uint32_t>(C)) Pw <<= 1;
  unsigned long long* K = reinterpret_cast<unsigned long long*>(
      (reinterpret_cast<uintptr_t>(A) + 7) & ~static_cast<uintptr_t>(7));
  const bool fits = rmax >= 0 && ob > 0 && ob < 63 && mx - mn < (1ll << ob) &&
                    2ull * Pw + 2 <= P;
  if (!fits) {
    for (int i = threadIdx.x; i < C; i += blockDim.x) A[i] = i;
    __syncthreads();
    block_stable_sort(C, A, ord, [&](uint32_t x, uint32_t y) {
      if (cands[x].op != cands[y].op) return cands[x].op < cands[y].op;
      return cands[x].rank < cands[y].rank;
    });
    return;
  }
  for (uint32_t x = threadIdx.x; x < Pw; x += blockDim.x)
    K[x] = x < static_cast<uint32_t>(C)
               ? (static_cast<unsigned long long>(cands[x].op - mn) << (rb + ib)) |
                     (static_cast<unsigned long long>(cands[x].rank) << ib) | x
               : ~0ull;
  __syncthreads();
  for (uint32_t k = 2; k <= Pw; k <<= 1) {
    for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
      for (uint32_t i = threadIdx.x; i < Pw; i += blockDim.x) {
        const uint32_t l = i ^ jj;
        if (l > i) {
          const unsigned long long x = K[i], y = K[l];
          if ((x > y) == ((i & k) == 0)) {
            K[i] = y;
            K[l] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  const unsigned long long im = (1ull << ib) - 1;
  for (int x = threadIdx.x; x < C; x += blockDim.x) ord[x] = static_cast<uint32_t>(K[x] & im);
  __syncthreads();
}

// Report assembly (rca.cpp:854-866) in parallel: exonerated in sorted order;
// suspects = the first retained entry per rank (a per-rank minimum of the
// sorted position), their evidence in sorted order; suspects then ordered by
// rank (ranks are unique among them: a prefix popcount over a rank bitmap).
__device__ void emit_reports_par(const DecideArgs& a, BlockShared& sh, int32_t j,
                                 const uint32_t* ord, const uint8_t* keep, int C) {
  const Cand* cands = a.pools.cand + sh.cand_base;
  const int32_t RS = a.m.rank_space;
  const uint32_t rw = static_cast<uint32_t>(RS + 31) / 32;
  uint32_t* minpos = a.emit_rank + static_cast<uint64_t>(j) * a.emit_stride;
  uint32_t* rbits = minpos + RS;
  uint32_t* woff = rbits + rw;
  for (int32_t r = threadIdx.x; r < RS; r += blockDim.x) minpos[r] = 0xFFFFFFFFu;
  for (uint32_t w = threadIdx.x; w < rw; w += blockDim.x) rbits[w] = 0;
  __syncthreads();
  for (int x = threadIdx.x; x < C; x += blockDim.x)
    if (keep[x]) {
      const int32_t r = cands[ord[x]].rank;
      if (r >= 0 && r < RS) atomicMin(&minpos[r], static_cast<uint32_t>(x));
    }
  __syncthreads();
  csg_suspect* sus = a.pools.sus + sh.sus_base;
  csg_suspect* exo = a.pools.sus + sh.exo_base;
  csg_evidence* evo = a.pools.ev + sh.ev_base;
  const csg_evidence* cev = a.pools.cev + sh.cev_base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwb = blockDim.x >> 5;
  __shared__ uint32_t scan3[32][3];
  uint32_t run_e = 0, run_s = 0, run_v = 0;
  for (int base = 0; base < C; base += blockDim.x) {
    const int x = base + threadIdx.x;
    const bool valid = x < C;
    Cand c;
    if (valid) c = cands[ord[x]];
    const bool isexo = valid && !keep[x];
    const bool isfirst = valid && keep[x] && c.rank >= 0 && c.rank < RS &&
                         minpos[c.rank] == static_cast<uint32_t>(x);
    const uint32_t evn = isfirst ? c.ev_n : 0;
    uint32_t e = isexo, f = isfirst, v = evn;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t e2 = __shfl_up_sync(FULL, e, o), f2 = __shfl_up_sync(FULL, f, o),
                     v2 = __shfl_up_sync(FULL, v, o);
      if (lane >= o) {
        e += e2;
        f += f2;
        v += v2;
      }
    }
    if (lane == 31) {
      scan3[warp][0] = e;
      scan3[warp][1] = f;
      scan3[warp][2] = v;
    }
    __syncthreads();
    uint32_t be = 0, bf = 0, bv = 0, te = 0, tf = 0, tv = 0;
    for (int q = 0; q < nwb; ++q) {
      if (q < warp) {
        be += scan3[q][0];
        bf += scan3[q][1];
        bv += scan3[q][2];
      }
      te += scan3[q][0];
      tf += scan3[q][1];
      tv += scan3[q][2];
    }
    if (isexo) exo[run_e + be + e - 1] = to_suspect(c);
    if (isfirst) {
      sus[run_s + bf + f - 1] = to_suspect(c);
      atomicOr(&rbits[c.rank >> 5], 1u << (c.rank & 31));
      const uint32_t v0 = run_v + bv + v - evn;
      for (uint32_t q = 0; q < evn; ++q) evo[v0 + q] = cev[c.ev_off + q];
    }
    run_e += te;
    run_s += tf;
    run_v += tv;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    for (uint32_t w = 0; w < rw; ++w) {
      woff[w] = acc;
      acc += __popc(rbits[w]);
    }
    sh.nsus = static_cast<int32_t>(run_s);
    sh.nexo = static_cast<int32_t>(run_e);
    sh.nev = run_v;
  }
  __syncthreads();
  csg_suspect* tmp = exo + run_e;  // spare room behind the exonerated
  for (uint32_t i = threadIdx.x; i < run_s; i += blockDim.x) {
    const int32_t r = sus[i].rank;
    const uint32_t pos = woff[r >> 5] + __popc(rbits[r >> 5] & ((1u << (r & 31)) - 1u));
    tmp[pos] = sus[i];
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < run_s; i += blockDim.x) sus[i] = tmp[i];
  __syncthreads();
}

__device__ void decide_straggler_finish(const DecideArgs& a, int32_t j, BlockShared& sh,
                                        uint32_t* scratch) {
  const StragState S = a.state[j];
  if (S.C <= 0) return;  // decided in phase 1 (or aborted)
  const int32_t naff = a.n_aff[j];
  const int C = S.C;
  if (threadIdx.x == 0) {
    sh.ncand = C;
    sh.cev_used = S.cev_used;
    sh.cand_base = S.cand_base;
    sh.cev_base = S.cev_base;
    sh.sus_base = S.sus_base;
    sh.exo_base = S.exo_base;
    sh.ev_base = S.ev_base;
    sh.cap_cand = S.cap_cand;
    sh.cap_cev = S.cap_cev;
  }
  __syncthreads();
  const long long clk_g0 = clock64();
  const uint32_t mwords = static_cast<uint32_t>((a.s.R + 31) / 32 + 1);
  const uint32_t P = (a.scratch_per_trip - mwords) / 2;
  uint32_t* A = scratch + mwords;
  uint32_t* B = A + P;
  Cand* cands = a.pools.cand + sh.cand_base;
  int any_self = 0;
  for (int x = threadIdx.x; x < C; x += blockDim.x) any_self |= cands[x].pad ? 1 : 0;
  any_self = __syncthreads_or(any_self);
  uint32_t* ord = B;
  uint8_t* keep = reinterpret_cast<uint8_t*>(B + C);
  uint32_t* tail = reinterpret_cast<uint32_t*>(keep + ((C + 3) & ~3));
  strag_order(a, cands, C, A, P, ord, sh);
  for (int x = threadIdx.x; x < C; x += blockDim.x)
    keep[x] = (!any_self || cands[ord[x]].pad) ? 1 : 0;
  __syncthreads();
  const long long clk_g2 = clock64();
  if (a.emit_rank) emit_reports_par(a, sh, j, ord, keep, C);
  else emit_reports(a, sh, ord, keep, C, tail);
  write_trip(a, j, sh.nsus ? CSG_VERDICT_SUSPECTS : CSG_VERDICT_NO_STRAGGLER,
             naff, 3 * a.N, sh);
  if (a.debug && threadIdx.x == 0)
    printf("decide trip %d naff %d C %d any_self %d cycles: order %lld emit %lld\n",
           j, naff, C, any_self, clk_g2 - clk_g0, (long long)clock64() - clk_g2);
}

// ---------------------------------------------------------------------------
// Failure analysis (analyze_failure, proj/src/rca.cpp:540-631), three stages:
//  K_fail_count  warp per (trip, affected group): last_logs_of_group +
//                check_min_op, else check_min_data -> suspect count
//  (scan)        candidate offsets in (trip, group asc) order
//  K_fail_cands  warp per (trip, affected group): one Candidate per suspect,
//                rank-sorted inside the group, with progress + evidence
//                (own channels, then the ring successor's on the same op)
//  K_exonerate   block per trip: stable (op, rank) order, op-DAG
//                reachability bitsets, chunked greedy exoneration, report.
// ---------------------------------------------------------------------------
struct FailItem {
  int32_t j;      // trip
  int32_t g;      // affected group
};

struct GroupPick {
  int32_t mode;   // 0 no suspects, 1 strict min op, 2 min progress
  int32_t count;
  int64_t min_op;
  uint64_t d, t, r;  // min (done, tx, ready) for mode 2
};

__host__ __device__ constexpr int kEvSlots(int nch) { return 2 * nch + 1; }

__global__ void k_fail_count(StoreView s, ModelView m,
                             const FailItem* __restrict__ items, int32_t n_items,
                             const RankSum* __restrict__ rs,
                             GroupPick* __restrict__ pick,
                             uint32_t* __restrict__ cnt,
                             const unsigned* __restrict__ n_dev) {
  pdl_wait();
  pdl_trigger();
  // n_items: grid bound (and scan length - 1); n_dev: the planned count when
  // the items were planned on the device (the tail up to n_items scans as 0)
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w == 0 && lane == 0) cnt[n_items] = 0;  // closes the offset scan
  const int64_t ni = n_dev ? static_cast<int64_t>(*n_dev) : n_items;
  if (w >= ni) {
    if (lane == 0 && w < n_items) cnt[w] = 0;
    return;
  }
  const FailItem it = items[w];
  const RankSum* rsj = rs + static_cast<uint64_t>(it.j) * s.R;
  const uint32_t mo = m.member_off[it.g];
  const int32_t mm = static_cast<int32_t>(m.member_off[it.g + 1] - mo);
  int nlog = 0;
  long long mn = LLONG_MAX;
  for (int32_t i = lane; i < mm; i += 32) {
    const int32_t r = m.members[mo + i];
    if (r >= 0 && r < s.R && (rsj[r].flags & RS_HAS_LAST)) {
      ++nlog;
      mn = min(mn, static_cast<long long>(rsj[r].last_op));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    nlog += __shfl_xor_sync(FULL, nlog, o);
    mn = min(mn, __shfl_xor_sync(FULL, mn, o));
  }
  GroupPick pk;
  pk.mode = 0;
  pk.count = 0;
  pk.min_op = mn;
  pk.d = pk.t = pk.r = ~0ull;
  if (nlog > 0) {
    int neq = 0;
    for (int32_t i = lane; i < mm; i += 32) {
      const int32_t r = m.members[mo + i];
      neq += (r >= 0 && r < s.R && (rsj[r].flags & RS_HAS_LAST) &&
              rsj[r].last_op == mn);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) neq += __shfl_xor_sync(FULL, neq, o);
    if (neq < nlog) {
      pk.mode = 1;
      pk.count = neq;
    } else {
      uint64_t d = ~0ull, t = ~0ull, rd = ~0ull;
      int nk = 0;
      for (int32_t i = lane; i < mm; i += 32) {
        const int32_t r = m.members[mo + i];
        if (r >= 0 && r < s.R && (rsj[r].flags & RS_HAS_LAST) &&
            (rsj[r].flags & RS_PROG)) {
          ++nk;
          if (prog_less(rsj[r].done, rsj[r].tx, rsj[r].ready, d, t, rd)) {
            d = rsj[r].done;
            t = rsj[r].tx;
            rd = rsj[r].ready;
          }
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        nk += __shfl_xor_sync(FULL, nk, o);
        const uint64_t d2 = __shfl_xor_sync(FULL, d, o);
        const uint64_t t2 = __shfl_xor_sync(FULL, t, o);
        const uint64_t r2 = __shfl_xor_sync(FULL, rd, o);
        if (prog_less(d2, t2, r2, d, t, rd)) {
          d = d2;
          t = t2;
          rd = r2;
        }
      }
      if (nk > 0) {
        int ns = 0;
        for (int32_t i = lane; i < mm; i += 32) {
          const int32_t r = m.members[mo + i];
          ns += (r >= 0 && r < s.R && (rsj[r].flags & RS_HAS_LAST) &&
                 (rsj[r].flags & RS_PROG) && rsj[r].done == d && rsj[r].tx == t &&
                 rsj[r].ready == rd);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) ns += __shfl_xor_sync(FULL, ns, o);
        pk.mode = 2;
        pk.count = ns;
        pk.d = d;
        pk.t = t;
        pk.r = rd;
      }
    }
  }
  if (lane == 0) {
    pick[w] = pk;
    cnt[w] = static_cast<uint32_t>(pk.count);
  }
}

__device__ inline bool is_suspect(const GroupPick& pk, const RankSum* rsj,
                                  int32_t r, int32_t R) {
  if (r < 0 || r >= R || !(rsj[r].flags & RS_HAS_LAST)) return false;
  if (pk.mode == 1) return rsj[r].last_op == pk.min_op;
  if (pk.mode == 2)
    return (rsj[r].flags & RS_PROG) && rsj[r].done == pk.d &&
           rsj[r].tx == pk.t && rsj[r].ready == pk.r;
  return false;
}

__global__ void k_fail_cands(StoreView s, ModelView m,
                             const FailItem* __restrict__ items, int32_t n_items,
                             const RankSum* __restrict__ rs,
                             const unsigned long long* __restrict__ chan_key,
                             const SuccProg* __restrict__ sp,
                             const unsigned long long* __restrict__ sp_key,
                             uint32_t M, int32_t nch,
                             const GroupPick* __restrict__ pick,
                             const uint32_t* __restrict__ off,
                             Cand* __restrict__ cand,
                             csg_evidence* __restrict__ cev,
                             uint32_t* __restrict__ err,
                             const unsigned* __restrict__ n_dev) {
  pdl_wait();
  pdl_trigger();
  constexpr int kWarps = 4;
  constexpr int kStage = 256;  // members staged in shared memory
  __shared__ int32_t srank[kWarps][kStage];     // suspect ranks, else INT_MAX
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= (n_dev ? static_cast<int64_t>(*n_dev) : n_items)) return;
  const FailItem it = items[w];
  const GroupPick pk = pick[w];
  if (pk.mode == 0) return;
  const RankSum* rsj = rs + static_cast<uint64_t>(it.j) * s.R;
  const uint32_t mo = m.member_off[it.g];
  const int32_t mm = static_cast<int32_t>(m.member_off[it.g + 1] - mo);
  const uint32_t base = off[w];
  const int EV = kEvSlots(nch);
  const bool staged = mm <= kStage;
  if (staged) {
    for (int32_t i = lane; i < mm; i += 32) {
      const int32_t r = m.members[mo + i];
      srank[wib][i] = is_suspect(pk, rsj, r, s.R) ? r : INT_MAX;
    }
    __syncwarp();
  }
  // rank-sorted slot of a suspect among the group's suspects
  auto slot_of = [&](int32_t r) {
    uint32_t pos = 0;
    if (staged) {
      for (int32_t k = 0; k < mm; ++k) pos += srank[wib][k] < r;
    } else {
      for (int32_t k = 0; k < mm; ++k) {
        const int32_t rk = m.members[mo + k];
        pos += (rk < r && is_suspect(pk, rsj, rk, s.R));
      }
    }
    return pos;
  };
  for (int32_t i = lane; i < mm; i += 32) {
    const int32_t r = m.members[mo + i];
    if (staged ? srank[wib][i] == INT_MAX : !is_suspect(pk, rsj, r, s.R)) continue;
    const uint32_t ci = base + slot_of(r);
    const RankSum own = rsj[r];
    Cand c;
    memset(&c, 0, sizeof(c));
    c.rank = r;
    c.group = it.g;
    c.op = own.last_op;
    c.onset = own.onset;
    c.known = (own.flags & RS_PROG) ? 1 : 0;
    c.ready = own.ready;
    c.tx = own.tx;
    c.done = own.done;
    c.it_lo = 0;
    c.it_hi = -1;
    c.ev_off = ci * EV;
    c.ev_n = 0;
    csg_evidence* ev = cev + static_cast<uint64_t>(ci) * EV;
    // own progress_of(r, op) evidence, ascending channel (rca.cpp:593-594)
    const unsigned long long* ck = chan_key + (static_cast<uint64_t>(it.j) * s.R + r) * nch;
    if (c.known)
      for (int ch = 0; ch < nch; ++ch)
        if (ck[ch]) ev[c.ev_n++] = csg_evidence{r, ch, dkey_inv(ck[ch]), c.op};
    // ring successor members[(i+1) % n] on the suspect's op (rca.cpp:596-605)
    bool peer_known = false;
    uint64_t prd = 0, ptx = 0, pdn = 0;
    if (mm >= 2) {
      const uint32_t sq = mo + (i + 1) % mm;
      const int32_t succ = m.members[sq];
      const SuccProg p = sp[static_cast<uint64_t>(it.j) * M + sq];
      if (p.known) {
        peer_known = true;
        prd = p.ready;
        ptx = p.tx;
        pdn = p.done;
        const unsigned long long* sk = sp_key + (static_cast<uint64_t>(it.j) * M + sq) * nch;
        for (int ch = 0; ch < nch; ++ch)
          if (sk[ch]) ev[c.ev_n++] = csg_evidence{succ, ch, dkey_inv(sk[ch]), c.op};
      }
    }
    if (c.known) {
      int cat, side;
      if (!rc_table(c.ready, c.tx, c.done, peer_known, prd, ptx, pdn, &cat, &side))
        atomicOr(err, DEV_ERR_RC_TABLE);
      c.cat = static_cast<uint8_t>(cat);
      c.side = static_cast<uint8_t>(side);
    } else {
      c.cat = CSG_RC_UNINITIALIZED_OR_BLOCKED;
      c.side = CSG_SIDE_UNDETERMINED;
    }
    // no evidence: cite the last log (rca.cpp:615-622)
    if (c.ev_n == 0) ev[c.ev_n++] = csg_evidence{r, own.last_chan, own.last_ts, c.op};
    cand[ci] = c;
  }
}

struct ExoTrip {
  int32_t j;
  int32_t naff;
  uint32_t cand_base;   // first candidate of the trip
  uint32_t n_cand;      // filled on device from the scan (see k_exonerate)
  uint32_t first_item, n_items;
  uint64_t scratch_off;  // bytes into the scratch pool (16-aligned)
  uint32_t sus_off, ev_off;  // output regions (upper bounds from the host)
};

// Failure planning on the device (no host round trip after k_affected):
// per trip its candidate bound C = members of its affected groups, then in
// trip order the items, exoneration trips and output regions the host would
// otherwise lay out (same formulas as the host path in rca_batch).
struct FailPlan {
  unsigned n_items, pad;
  unsigned long long cand_ub, sus_fail, ev_fail, scratch_bytes;
};

__host__ __device__ inline uint64_t exo_scratch_need(uint64_t C, uint64_t Rs) {
  uint64_t P = 1;
  while (P < C) P <<= 1;
  const uint64_t need = ((P * 4 + 15) & ~15ull) + ((C * 8 + 15) & ~15ull) +
                        ((C * 4 + 15) & ~15ull) + ((C + 15) & ~15ull) +
                        4 * ((Rs + 3) & ~3ull) + 8 * (((Rs + 31) / 32 + 3) & ~3ull) +
                        32 * C + 64;
  return (need + 255) & ~255ull;
}

__global__ void __launch_bounds__(1024)
    k_fail_plan(int32_t J, int32_t G, const int32_t* __restrict__ kind,
                const int32_t* __restrict__ naff, const int32_t* __restrict__ aff,
                ModelView m, int32_t R, int EV, FailItem* __restrict__ items,
                ExoTrip* __restrict__ exo, FailPlan* __restrict__ plan,
                unsigned long long* __restrict__ used) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int32_t j = warp; j < J; j += nw) {
    const int32_t na = naff[j];
    const bool ok = kind[j] == CSG_TRIGGER_FAILURE && na > 0 && m.opn > 0;
    unsigned long long C = 0;
    if (ok)
      for (int32_t i = lane; i < na; i += 32) {
        const int32_t g = aff[static_cast<uint64_t>(j) * G + i];
        C += m.member_off[g + 1] - m.member_off[g];
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) C += __shfl_xor_sync(FULL, C, o);
    if (lane == 0) {
      ExoTrip e;
      memset(&e, 0, sizeof(e));
      e.j = ok ? j : -1;
      e.naff = na;
      e.n_cand = static_cast<uint32_t>(C);  // bound for the layout pass
      exo[j] = e;
    }
  }
  __syncthreads();
  __shared__ unsigned s_ni;
  if (threadIdx.x == 0) {
    unsigned ni = 0;
    unsigned long long sb = 0, sus = 0, ev = 0, cub = 0;
    const uint64_t Rs = R > 0 ? R : 1;
    for (int32_t j = 0; j < J; ++j) {
      ExoTrip& e = exo[j];
      if (e.j < 0) continue;
      const unsigned long long C = e.n_cand;
      e.n_cand = 0;
      e.first_item = ni;
      e.n_items = static_cast<uint32_t>(e.naff);
      e.scratch_off = sb;
      e.sus_off = static_cast<uint32_t>(sus);
      e.ev_off = static_cast<uint32_t>(ev);
      ni += e.naff;
      sb += exo_scratch_need(C, Rs);
      sus += 2 * C;
      ev += C * EV;
      cub += C;
    }
    plan->n_items = ni;
    plan->cand_ub = cub;
    plan->sus_fail = sus;
    plan->ev_fail = ev;
    plan->scratch_bytes = sb;
    for (int q = 0; q < 8; ++q) used[q] = 0;
    used[2] = sus;  // P_SUS: straggler bump allocations start after these
    used[3] = ev;   // P_EV
    s_ni = ni;
  }
  __syncthreads();
  for (int32_t j = warp; j < J; j += nw) {
    const ExoTrip e = exo[j];
    if (e.j < 0) continue;
    for (int32_t i = lane; i < e.naff; i += 32)
      items[e.first_item + i] = FailItem{j, aff[static_cast<uint64_t>(j) * G + i]};
  }
}

struct ExoArgs {
  int debug;
  StoreView s;
  ModelView m;
  const Cand* cand;
  const csg_evidence* cev;
  int32_t EV;
  const uint32_t* off;   // exclusive scan of item counts (n_items + 1)
  ExoTrip* trips;
  int32_t n_trips;
  unsigned char* scratch;
  unsigned long long* bits;
  unsigned long long bits_cap;
  unsigned long long* bits_used;
  csg_suspect* sus;
  csg_evidence* ev;
  TripOut* out;
  uint64_t N;
  uint32_t* err;
  int warp_sweep;  // CSG_EXO_WARP_SWEEP=1: the single-warp sweep only
};

// Block-wide inclusive scan (blockDim a multiple of 32, <= 1024) with an
// associative op; wtot: 32 words of shared scratch. Block-collective.
template <typename T, typename Op>
__device__ T block_incl_scan(T v, T* wtot, Op op) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v = op(y, v);
  }
  __syncthreads();
  if (lane == 31) wtot[warp] = v;
  __syncthreads();
  if (warp == 0) {
    T x = wtot[lane < nw ? lane : 0];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x = op(y, x);
    }
    if (lane < nw) wtot[lane] = x;
  }
  __syncthreads();
  if (warp > 0) v = op(wtot[warp - 1], v);
  return v;
}

// In-place block bitonic sort of idx[0, P) (P power of two) by `less`;
// entries >= n are padding (sort last).
template <typename L>
__device__ void block_bitonic(uint32_t* idx, uint32_t n, uint32_t P, L less) {
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) idx[i] = i < n ? i : 0xFFFFFFFFu;
  __syncthreads();
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
      for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
        const uint32_t l = i ^ jj;
        if (l > i) {
          const uint32_t a = idx[i], b = idx[l];
          const bool up = (i & k) == 0;
          bool a_lt_b;
          if (a == 0xFFFFFFFFu) a_lt_b = false;
          else if (b == 0xFFFFFFFFu) a_lt_b = true;
          else a_lt_b = less(a, b);
          const bool swap = up ? !a_lt_b : a_lt_b;
          if (swap && !(a == b)) {
            idx[i] = b;
            idx[l] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

__device__ inline uint32_t pow2_ceil(uint32_t x) {
  uint32_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

constexpr int kExoThreads = 512;
constexpr size_t kExoSmemMax = 192 * 1024;
// Trips with at most kExoStage candidates keep the exoneration keys, the
// (op, rank) order and the retained list in shared memory: the greedy sweep
// is O(C x retained) dependent lookups, latency-bound from global memory.
constexpr uint32_t kExoStage = 4096;
struct ExoKey {
  int64_t op;
  int32_t rank;
  uint32_t known;
  uint64_t done, tx, ready;
};
constexpr size_t kExoStageBytes = kExoStage * (sizeof(ExoKey) + 4);

__global__ void __launch_bounds__(kExoThreads, 1) k_exonerate(ExoArgs a) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned long long exo_dyn[];
  __shared__ int32_t sh_i[8];
  __shared__ unsigned long long sh_u[2];
  __shared__ uint32_t wsum[16];
  __shared__ uint32_t scan3[16][3];
  __shared__ int32_t s_rsum[kExoStage];
  __shared__ uint8_t s_keep[kExoStage];
  ExoTrip& tp = a.trips[blockIdx.x];
  if (tp.j < 0) {
    // device plan (one entry per trip, failure-only batch): no affected group
    // or no program -> FalseTrigger, as k_decide would write it
    if (threadIdx.x == 0) {
      TripOut o;
      memset(&o, 0, sizeof(o));
      o.verdict = CSG_VERDICT_FALSE_TRIGGER;
      o.n_aff = tp.naff;
      o.scanned = a.N;
      a.out[blockIdx.x] = o;
    }
    return;
  }
  const int tid = threadIdx.x;
  const uint32_t cbase = a.off[tp.first_item];
  const uint32_t C = a.off[tp.first_item + tp.n_items] - cbase;
  const Cand* cands = a.cand + cbase;
  TripOut o;
  memset(&o, 0, sizeof(o));
  o.n_aff = tp.naff;
  o.sus_off = tp.sus_off;
  o.ev_off = tp.ev_off;
  o.scanned = 2 * a.N;
  if (C == 0) {
    if (tid == 0) {
      o.verdict = CSG_VERDICT_UNDETERMINED;
      o.exo_off = tp.sus_off;
      a.out[tp.j] = o;
    }
    return;
  }
  // scratch layout (all 16-aligned)
  const uint32_t P = pow2_ceil(C);
  unsigned char* sp = a.scratch + tp.scratch_off;
  const bool staged = C <= kExoStage;
  unsigned char* dynb = reinterpret_cast<unsigned char*>(exo_dyn);
  ExoKey* sk = reinterpret_cast<ExoKey*>(dynb);
  uint32_t* ord = staged ? reinterpret_cast<uint32_t*>(dynb + kExoStage * sizeof(ExoKey))
                         : reinterpret_cast<uint32_t*>(sp);
  int64_t* U = reinterpret_cast<int64_t*>(sp + ((P * 4 + 15) & ~15u));
  uint32_t* ret_g = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(U) +
                                                ((C * 8 + 15) & ~15u));
  uint8_t* keep_g = reinterpret_cast<uint8_t*>(ret_g) + ((C * 4 + 15) & ~15u);
  const uint32_t Rs = static_cast<uint32_t>(a.s.R > 0 ? a.s.R : 1);
  uint32_t* minpos = reinterpret_cast<uint32_t*>(keep_g + ((C + 15) & ~15u));
  uint8_t* keep = staged ? s_keep : keep_g;
  uint32_t* rbits = minpos + ((Rs + 3) & ~3u);
  uint32_t* woff = rbits + (((Rs + 31) / 32 + 3) & ~3u);
  csg_suspect* stmp =
      reinterpret_cast<csg_suspect*>(woff + (((Rs + 31) / 32 + 3) & ~3u));
  if (staged) {
    for (uint32_t i = tid; i < C; i += blockDim.x) {
      const Cand& c = cands[i];
      sk[i] = ExoKey{c.op, c.rank, c.known, c.done, c.tx, c.ready};
    }
    __syncthreads();
  }
  auto key = [&](uint32_t i) -> ExoKey {
    if (staged) return sk[i];
    const Cand& c = cands[i];
    return ExoKey{c.op, c.rank, c.known, c.done, c.tx, c.ready};
  };
  long long clk0 = clock64(), clk1 = 0, clk2 = 0, clk3 = 0, clk4 = 0, clk5 = 0;
  long long cy_y = 0, cy_dd = 0, cy_walk = 0;
  // 1. stable (op, rank) order. When (op - min op, rank, index) packs into
  // 64 bits and P keys fit the free shared memory past the staged keys, the
  // bitonic network sorts the packed keys directly (no indirection through
  // the 40-byte key records per compare-exchange).
  bool packed = false;
  if (staged && P <= (kExoSmemMax - kExoStageBytes) / 8) {
    __shared__ long long s_opmin, s_opmax;
    __shared__ int s_rmax;
    if (tid == 0) {
      s_opmin = LLONG_MAX;
      s_opmax = LLONG_MIN;
      s_rmax = 0;
    }
    __syncthreads();
    long long mn = LLONG_MAX, mx = LLONG_MIN;
    int rm = 0;
    for (uint32_t i = tid; i < C; i += blockDim.x) {
      mn = min(mn, static_cast<long long>(sk[i].op));
      mx = max(mx, static_cast<long long>(sk[i].op));
      rm = max(rm, sk[i].rank);
    }
    atomicMin(&s_opmin, mn);
    atomicMax(&s_opmax, mx);
    atomicMax(&s_rmax, rm);
    __syncthreads();
    const unsigned long long span =
        static_cast<unsigned long long>(s_opmax) - static_cast<unsigned long long>(s_opmin);
    const int ib = 32 - __clz(static_cast<int>(P - 1) | 1);
    const int rb = 32 - __clz(s_rmax | 1);
    const int ob = 64 - __clzll(static_cast<long long>(span | 1));
    if (s_rmax >= 0 && ob + rb + ib <= 64 && (span >> 62) == 0) {
      packed = true;
      unsigned long long* pk =
          reinterpret_cast<unsigned long long*>(dynb + kExoStageBytes);
      const long long omin = s_opmin;
      for (uint32_t i = tid; i < P; i += blockDim.x)
        pk[i] = i < C ? ((static_cast<unsigned long long>(sk[i].op - omin) << (rb + ib)) |
                         (static_cast<unsigned long long>(sk[i].rank) << ib) | i)
                      : ~0ull;
      __syncthreads();
      for (uint32_t k = 2; k <= P; k <<= 1) {
        for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
          for (uint32_t i = tid; i < P; i += blockDim.x) {
            const uint32_t l = i ^ jj;
            if (l > i) {
              const unsigned long long x = pk[i], y = pk[l];
              if (((i & k) == 0) == (x > y)) {
                pk[i] = y;
                pk[l] = x;
              }
            }
          }
          __syncthreads();
        }
      }
      const unsigned long long im = (1ull << ib) - 1;
      for (uint32_t i = tid; i < P; i += blockDim.x)
        ord[i] = i < C ? static_cast<uint32_t>(pk[i] & im) : 0xFFFFFFFFu;
      __syncthreads();
    }
  }
  if (!packed) {
    // large trips: the same packed (op - min op, rank, index) keys, sorted
    // in the trip's global scratch (the report's staging area, free here)
    __shared__ long long g_opmin, g_opmax;
    __shared__ int g_rmax;
    if (tid == 0) {
      g_opmin = LLONG_MAX;
      g_opmax = LLONG_MIN;
      g_rmax = 0;
    }
    __syncthreads();
    long long mn = LLONG_MAX, mx = LLONG_MIN;
    int rm = 0;
    for (uint32_t i = tid; i < C; i += blockDim.x) {
      const ExoKey k2 = key(i);
      mn = min(mn, static_cast<long long>(k2.op));
      mx = max(mx, static_cast<long long>(k2.op));
      rm = max(rm, k2.rank);
    }
    atomicMin(&g_opmin, mn);
    atomicMax(&g_opmax, mx);
    atomicMax(&g_rmax, rm);
    __syncthreads();
    const unsigned long long span =
        static_cast<unsigned long long>(g_opmax) - static_cast<unsigned long long>(g_opmin);
    const int ib = 32 - __clz(static_cast<int>(P - 1) | 1);
    const int rb = 32 - __clz(g_rmax | 1);
    const int ob = 64 - __clzll(static_cast<long long>(span | 1));
    if (g_rmax >= 0 && ob + rb + ib <= 64 && (span >> 62) == 0) {
      packed = true;
      unsigned long long* pk = reinterpret_cast<unsigned long long*>(stmp);
      const long long omin = g_opmin;
      for (uint32_t i = tid; i < P; i += blockDim.x) {
        if (i < C) {
          const ExoKey k2 = key(i);
          pk[i] = (static_cast<unsigned long long>(k2.op - omin) << (rb + ib)) |
                  (static_cast<unsigned long long>(k2.rank) << ib) | i;
        } else {
          pk[i] = ~0ull;
        }
      }
      __syncthreads();
      for (uint32_t k = 2; k <= P; k <<= 1) {
        for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
          for (uint32_t i = tid; i < P; i += blockDim.x) {
            const uint32_t l = i ^ jj;
            if (l > i) {
              const unsigned long long x = pk[i], y = pk[l];
              if (((i & k) == 0) == (x > y)) {
                pk[i] = y;
                pk[l] = x;
              }
            }
          }
          __syncthreads();
        }
      }
      const unsigned long long im = (1ull << ib) - 1;
      for (uint32_t i = tid; i < P; i += blockDim.x)
        ord[i] = i < C ? static_cast<uint32_t>(pk[i] & im) : 0xFFFFFFFFu;
      __syncthreads();
    }
  }
  if (!packed)
    block_bitonic(ord, C, P, [&](uint32_t x, uint32_t y) {
      const ExoKey kx = key(x), ky = key(y);
      if (kx.op != ky.op) return kx.op < ky.op;
      if (kx.rank != ky.rank) return kx.rank < ky.rank;
      return x < y;
    });
  clk1 = clock64();
  // 2. distinct valid (>= 0) candidate ops, ascending (ordered compaction)
  {
    int Kc = 0;
    const int nw = blockDim.x >> 5;
    for (uint32_t base = 0; base < C; base += blockDim.x) {
      const uint32_t x = base + tid;
      int64_t op = -1, prev = -1;
      bool fl = false;
      if (x < C) {
        op = key(ord[x]).op;
        prev = x ? key(ord[x - 1]).op : -1;
        fl = op >= 0 && (x == 0 || prev != op);
      }
      const unsigned bm = __ballot_sync(FULL, fl);
      if ((tid & 31) == 0) wsum[tid >> 5] = __popc(bm);
      __syncthreads();
      int before = 0, total = 0;
      for (int q = 0; q < nw; ++q) {
        if (q < (tid >> 5)) before += wsum[q];
        total += wsum[q];
      }
      if (fl) U[Kc + before + __popc(bm & ((1u << (tid & 31)) - 1u))] = op;
      Kc += total;
      __syncthreads();
    }
    if (tid == 0) sh_i[0] = Kc;
  }
  __syncthreads();
  clk2 = clock64();
  const int K = sh_i[0];
  const int words = (K + 63) / 64;
  const int32_t opn = a.m.opn;
  int64_t lo = 0, hi = -1;
  unsigned long long* bits = nullptr;
  int32_t* cidx = nullptr;  // dense op -> candidate bit over [lo, hi], -1 if none
  if (K >= 2) {
    lo = U[0];
    hi = U[K - 1];
    const unsigned long long V = static_cast<unsigned long long>(hi - lo + 1);
    // + per candidate rank: the op groups whose only retained rank it is
    const unsigned long long want = V * words + (V + 1) / 2 + static_cast<unsigned long long>(C) * words;
    if (tid == 0) {
      const unsigned long long b0 = atomicAdd(a.bits_used, want);
      sh_u[0] = b0;
      sh_i[1] = b0 + want <= a.bits_cap;
      if (!sh_i[1]) atomicOr(a.err, DEV_ERR_DAG_SCRATCH);
    }
    __syncthreads();
    if (!sh_i[1]) return;
    const size_t stage_b = staged ? kExoStageBytes : 0;
    if ((V * words + (V + 1) / 2) * 8 <= kExoSmemMax - stage_b) {
      bits = exo_dyn + stage_b / 8;  // ancestor bitsets resident in shared memory
    } else {
      bits = a.bits + sh_u[0];
    }
    cidx = reinterpret_cast<int32_t*>(bits + V * words);
    for (unsigned long long i = tid; i < V * words; i += blockDim.x) bits[i] = 0;
    for (unsigned long long i = tid; i < V; i += blockDim.x) cidx[i] = -1;
    __syncthreads();
    for (int i = tid; i < K; i += blockDim.x) cidx[U[i] - lo] = i;
    __syncthreads();
    // ancestor bitsets over [lo, hi] in (iteration, level) order
    const bool in_smem = bits == exo_dyn + stage_b / 8;
    const size_t used_b = (V * words + (V + 1) / 2) * 8;
    const size_t small_b = V * 8 + 4 + V * static_cast<size_t>(a.m.max_deg) * 4;
    if (in_smem && V <= 4096 && used_b + small_b <= kExoSmemMax - stage_b) {
      // Small window: the parent lists of every op in [lo, hi] are gathered
      // into shared memory once (one round of independent global loads),
      // then the (iteration, level) wavefront runs on shared memory only.
      int32_t* vlv = cidx + ((V + 1) & ~1ull);
      uint32_t* vpo = reinterpret_cast<uint32_t*>(vlv + V);
      int32_t* vpl = reinterpret_cast<int32_t*>(vpo + V + 1);
      const uint32_t md = static_cast<uint32_t>(a.m.max_deg);
      for (unsigned long long v = tid; v < V; v += blockDim.x) {
        const int64_t gv = lo + static_cast<int64_t>(v);
        const int32_t sop = static_cast<int32_t>(gv - (gv / opn) * opn);
        vlv[v] = __ldg(a.m.op_level + sop);
        vpo[v] = __ldg(a.m.par_off + sop + 1) - __ldg(a.m.par_off + sop);
      }
      // one (op, parent slot) per thread: independent loads, one latency
      for (unsigned long long q = tid; q < V * md; q += blockDim.x) {
        const unsigned long long v = q / md;
        const uint32_t k = static_cast<uint32_t>(q % md);
        const int64_t gv = lo + static_cast<int64_t>(v);
        const int64_t it = gv / opn;
        const int32_t sop = static_cast<int32_t>(gv - it * opn);
        const uint32_t pe0 = __ldg(a.m.par_off + sop), pe1 = __ldg(a.m.par_off + sop + 1);
        int32_t lp = -1;
        if (pe0 + k < pe1) {
          const int64_t pit = it + __ldg(a.m.par_it + pe0 + k);
          const int64_t pv = pit * opn + __ldg(a.m.par_op + pe0 + k);
          if (pit >= 0 && pv >= lo) lp = static_cast<int32_t>(pv - lo);
        }
        vpl[q] = lp;
      }
      __syncthreads();
      // wavefront: one warp per (op, word), lanes over the parent slots
      const int lane = tid & 31, nwarps = blockDim.x >> 5;
      for (int64_t it = lo / opn; it <= hi / opn; ++it) {
        for (int32_t lv = 0; lv < a.m.n_levels; ++lv) {
          for (unsigned long long q = tid >> 5; q < V * words; q += nwarps) {
            const unsigned long long v = q / words;
            const int wd = static_cast<int>(q % words);
            if (vlv[v] != lv || (lo + static_cast<int64_t>(v)) / opn != it) continue;
            unsigned long long acc = 0;
            const uint32_t np = vpo[v];
            for (uint32_t k = lane; k < np; k += 32) {
              const int32_t lp = vpl[v * md + k];
              if (lp < 0) continue;
              acc |= bits[static_cast<uint64_t>(lp) * words + wd];
              const int l = cidx[lp];
              if (l >= 0 && (l >> 6) == wd) acc |= 1ull << (l & 63);
            }
            const uint32_t lo32 = __reduce_or_sync(FULL, static_cast<uint32_t>(acc));
            const uint32_t hi32 = __reduce_or_sync(FULL, static_cast<uint32_t>(acc >> 32));
            if (lane == 0) bits[v * words + wd] = (static_cast<unsigned long long>(hi32) << 32) | lo32;
          }
          __syncthreads();
        }
      }
    } else
    for (int64_t it = lo / opn; it <= hi / opn; ++it) {
      for (int32_t lv = 0; lv < a.m.n_levels; ++lv) {
        const uint32_t l0 = a.m.lvl_off[lv];
        const uint32_t nl = a.m.lvl_off[lv + 1] - l0;
        // a thread per (op, run of 8 words) for wide rows: the parent list
        // is read once per 8 words and the 8 parent words load
        // independently; narrow rows keep a thread per (op, word)
        constexpr int kWC = 8;
        if (words < 24) {
          for (uint32_t q = tid; q < nl * words; q += blockDim.x) {
            const int32_t sop = a.m.lvl_ops[l0 + q / words];
            const int wd = q % words;
            const int64_t v = it * opn + sop;
            if (v < lo || v > hi) continue;
            unsigned long long acc = 0;
            const uint32_t pe0 = __ldg(a.m.par_off + sop), pe1 = __ldg(a.m.par_off + sop + 1);
#pragma unroll 8
            for (uint32_t pe = pe0; pe < pe1; ++pe) {
              const int64_t pit = it + __ldg(a.m.par_it + pe);
              const int64_t pv = pit * opn + __ldg(a.m.par_op + pe);
              if (pit < 0 || pv < lo) continue;
              acc |= bits[(pv - lo) * words + wd];
              const int l = cidx[pv - lo];
              if (l >= 0 && (l >> 6) == wd) acc |= 1ull << (l & 63);
            }
            bits[(v - lo) * words + wd] = acc;
          }
          __syncthreads();
          continue;
        }
        const int wc = kWC;
        const uint32_t nwc = static_cast<uint32_t>(words + wc - 1) / wc;
        for (uint32_t q = tid; q < nl * nwc; q += blockDim.x) {
          const int32_t sop = a.m.lvl_ops[l0 + q / nwc];
          const int w0 = static_cast<int>(q % nwc) * wc;
          const int w1 = min(words, w0 + wc);
          const int64_t v = it * opn + sop;
          if (v < lo || v > hi) continue;
          unsigned long long acc[kWC];
#pragma unroll
          for (int k = 0; k < kWC; ++k) acc[k] = 0;
          const uint32_t pe0 = __ldg(a.m.par_off + sop), pe1 = __ldg(a.m.par_off + sop + 1);
          for (uint32_t pe = pe0; pe < pe1; ++pe) {
            const int64_t pit = it + __ldg(a.m.par_it + pe);
            const int64_t pv = pit * opn + __ldg(a.m.par_op + pe);
            if (pit < 0 || pv < lo) continue;
            const unsigned long long* prow = bits + (pv - lo) * words;
#pragma unroll
            for (int k = 0; k < kWC; ++k)
              if (w0 + k < w1) acc[k] |= prow[w0 + k];
            const int l = cidx[pv - lo];
            const int lw = l >> 6;
            if (l >= 0 && lw >= w0 && lw < w1) {
#pragma unroll
              for (int k = 0; k < kWC; ++k)
                if (lw == w0 + k) acc[k] |= 1ull << (l & 63);
            }
          }
          unsigned long long* vrow = bits + (v - lo) * words;
#pragma unroll
          for (int k = 0; k < kWC; ++k)
            if (w0 + k < w1) vrow[w0 + k] = acc[k];
        }
        __syncthreads();
      }
    }
  }
  __syncthreads();
  clk3 = clock64();
  // 3. greedy exoneration (rca.cpp:487-514). In (op, rank) order a
  //    candidate c is dropped by an already-retained u of another rank when
  //    u has the same op and strictly less progress (done, tx, ready), or
  //    when c's op depends on u's op. Both relations only look backwards in
  //    op order, so the sweep runs op group by op group (one warp):
  //    * dependency drops: a group's candidates test, in parallel, the
  //      ancestor bitset of their op against a summary of every earlier
  //      group's retained ranks (rsum[l]: -1 none, the single rank, or -2
  //      for two or more ranks; NE / MU bitsets of non-empty / multi-rank
  //      groups), i.e. "some retained u there has a rank != c.rank";
  //    * same-op drops: the group walks in rank order keeping the least
  //      retained progress m1 (rank rk1) and the least progress of a retained
  //      rank != rk1 (m2); c is dropped iff the least retained progress among
  //      OTHER ranks is below its own.
  //    Exactly the reference's O(C x retained) greedy, in O(C + K) steps.
  constexpr int kMaskWords = 128;  // op groups up to 8192 keep the group masks
  __shared__ unsigned long long NE[kMaskWords], MU[kMaskWords];
  // [K] retained-rank summary (K <= C)
  int32_t* rsum = staged ? s_rsum : reinterpret_cast<int32_t*>(ret_g);
  // dependency drops by rank: RB[rid(r)] = the op groups whose retained set
  // is exactly {r}; then c (rank r) is dropped iff its ancestors meet a
  // multi-rank group or a single-rank group outside RB[rid(r)] — a word scan
  // instead of one rsum lookup per retained ancestor group. rid: compact
  // ids of the candidate ranks (the report's minpos array, reset there).
  unsigned long long* RB = nullptr;
  __shared__ unsigned s_nrid;
  if (K >= 2 && words <= kMaskWords) {
    const unsigned long long V = static_cast<unsigned long long>(hi - lo + 1);
    RB = a.bits + sh_u[0] + V * words + (V + 1) / 2;
    for (unsigned long long i = tid; i < static_cast<unsigned long long>(C) * words; i += blockDim.x)
      RB[i] = 0;
    for (uint32_t r = tid; r < Rs; r += blockDim.x) minpos[r] = 0xFFFFFFFFu;
    if (tid == 0) s_nrid = 0;
    __syncthreads();
    for (uint32_t x2 = tid; x2 < C; x2 += blockDim.x) {
      const int32_t r = key(x2).rank;
      if (r >= 0 && static_cast<uint32_t>(r) < Rs &&
          atomicCAS(&minpos[r], 0xFFFFFFFFu, 0xFFFFFFFEu) == 0xFFFFFFFFu)
        minpos[r] = atomicAdd(&s_nrid, 1u);
    }
    __syncthreads();
  }
  // The whole block sweeps when the progress triples pack into one ordered
  // u64 (done, tx, ready each < 2^21: done << 42 | tx << 21 | ready orders
  // like prog_less): per op group, every candidate's dependency test runs on
  // its own thread, and the same-op rule's exclusive run minimum is two
  // block scans (a prefix minimum of the surviving known progress and a
  // prefix maximum of the run starts) — a few barriers per group instead of
  // a warp's chain of 64-bit shuffles per 32 candidates.
  __shared__ int s_pack;
  if (tid == 0) s_pack = a.warp_sweep ? 0 : 1;
  __syncthreads();
  for (uint32_t x2 = tid; x2 < C; x2 += blockDim.x) {
    const ExoKey k2 = key(x2);
    if (k2.known && (k2.done >= (1ull << 21) || k2.tx >= (1ull << 21) || k2.ready >= (1ull << 21)))
      s_pack = 0;
  }
  __syncthreads();
  if (s_pack) {
    const bool masks = words <= kMaskWords;
    __shared__ unsigned long long s_w64[32];
    __shared__ uint32_t s_w32[32];
    __shared__ unsigned long long s_pm[kExoThreads];
    __shared__ uint32_t s_rs[kExoThreads];
    __shared__ int32_t s_red[2][32];
    __shared__ uint32_t s_kg;
    uint32_t* gpos = reinterpret_cast<uint32_t*>(stmp);  // [K + 1] group starts
    // group starts in sorted order
    if (tid == 0) s_kg = 0;
    for (int l = tid; l < K; l += blockDim.x) rsum[l] = -1;
    for (int w = tid; w < kMaskWords; w += blockDim.x) NE[w] = MU[w] = 0;
    __syncthreads();
    for (uint32_t b0 = 0; b0 < C; b0 += blockDim.x) {
      const uint32_t i = b0 + tid;
      const uint32_t f = i < C && (i == 0 || key(ord[i]).op != key(ord[i - 1]).op) ? 1u : 0u;
      const uint32_t inc = block_incl_scan(f, s_w32, [](uint32_t u, uint32_t v2) { return u + v2; });
      const uint32_t base_g = s_kg;
      if (f) gpos[base_g + inc - 1] = i;
      __syncthreads();
      if (tid == blockDim.x - 1) s_kg = base_g + inc;
      __syncthreads();
    }
    const uint32_t KG = s_kg;
    if (tid == 0) gpos[KG] = C;
    __syncthreads();
    const unsigned long long INF = ~0ull;
    auto pk = [](const ExoKey& k2) {
      return (k2.done << 42) | (k2.tx << 21) | k2.ready;
    };
    __shared__ unsigned long long s_T[kMaskWords];  // row & single-rank groups
    __shared__ uint16_t s_nz[kMaskWords];           // words of s_T that are non-zero
    __shared__ int s_nnz, s_mu;
    for (uint32_t gi = 0; gi < KG; ++gi) {
      const uint32_t x = gpos[gi], y = gpos[gi + 1];
      const int64_t op = key(ord[x]).op;
      const bool dag = op >= 0 && K >= 2;
      const int g = dag ? cidx[op - lo] : -1;
      const unsigned long long* row = dag ? bits + (op - lo) * words : nullptr;
      // every candidate of the group shares its op's ancestor row: stage
      // row & single-rank groups once (and whether the row meets a
      // multi-rank group, which drops the whole group)
      const bool staged_row = dag && masks && RB;
      if (staged_row) {
        if (tid == 0) {
          s_nnz = 0;
          s_mu = 0;
        }
        __syncthreads();
        for (int w = tid; w < words; w += blockDim.x) {
          const unsigned long long rw = row[w];
          if (rw & MU[w]) s_mu = 1;
          const unsigned long long t = rw & NE[w] & ~MU[w];
          s_T[w] = t;
          if (t) s_nz[atomicAdd(&s_nnz, 1)] = static_cast<uint16_t>(w);
        }
        __syncthreads();
      }
      unsigned long long carry_all = INF;     // min over [x, base)
      unsigned long long carry_closed = INF;  // min over [x, start of the open run)
      int32_t open_rank = INT_MIN;
      int32_t kmin = INT_MAX, kmax = INT_MIN;
      for (uint32_t base = x; base < y; base += blockDim.x) {
        const uint32_t i = base + tid;
        const bool in = i < y;
        ExoKey mk{};
        if (in) mk = key(ord[i]);
        bool dd = false;
        if (in && dag && staged_row && mk.rank >= 0 && static_cast<uint32_t>(mk.rank) < Rs) {
          dd = s_mu != 0;
          const unsigned long long* rb = RB + static_cast<uint64_t>(minpos[mk.rank]) * words;
          const int nnz = s_nnz;
          for (int z0 = 0; z0 < nnz && !dd; z0 += 8) {
            unsigned long long rv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) rv[q] = z0 + q < nnz ? rb[s_nz[z0 + q]] : ~0ull;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (z0 + q < nnz) dd = dd || (s_T[s_nz[z0 + q]] & ~rv[q]);
          }
        } else if (in && dag) {
          const int32_t r = mk.rank;
          const unsigned long long* rb =
              RB && r >= 0 && static_cast<uint32_t>(r) < Rs ? RB + static_cast<uint64_t>(minpos[r]) * words
                                                          : nullptr;
          if (rb) {
            for (int w0 = 0; w0 < words && !dd; w0 += 8) {
              unsigned long long av[8], rv[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                av[q] = w0 + q < words ? row[w0 + q] : 0ull;
                rv[q] = w0 + q < words ? rb[w0 + q] : 0ull;
              }
#pragma unroll
              for (int q = 0; q < 8; ++q)
                if (w0 + q < words)
                  dd = dd || (av[q] & MU[w0 + q]) || (av[q] & NE[w0 + q] & ~MU[w0 + q] & ~rv[q]);
            }
          } else {
            for (int w = 0; w < words && !dd; ++w) {
              unsigned long long av2 = row[w];
              if (masks) {
                if (av2 & MU[w]) {
                  dd = true;
                  break;
                }
                av2 &= NE[w];
              }
              while (av2 && !dd) {
                const int l = w * 64 + __ffsll(av2) - 1;
                const int32_t q = rsum[l];
                dd = q != -1 && q != r;
                av2 &= av2 - 1;
              }
            }
          }
        }
        const int32_t rk = in ? mk.rank : INT_MAX;
        const unsigned long long v = in && !dd && mk.known ? pk(mk) : INF;
        int32_t prev_rk = INT_MIN;
        if (in && i > x) prev_rk = tid == 0 ? open_rank : key(ord[i - 1]).rank;
        const bool start = in && (i == x || rk != prev_rk);
        const unsigned long long pm = block_incl_scan(
            v, s_w64, [](unsigned long long u, unsigned long long w2) { return u < w2 ? u : w2; });
        const uint32_t rs = block_incl_scan(start ? i + 1 : 0u, s_w32,
                                            [](uint32_t u, uint32_t w2) { return u > w2 ? u : w2; });
        s_pm[tid] = pm;
        s_rs[tid] = rs;
        __syncthreads();
        // least surviving known progress before my run
        unsigned long long km;
        if (rs) {  // my run starts in this chunk, at rs - 1
          const uint32_t st0 = rs - 1;
          km = carry_all;
          if (st0 > base) {
            const unsigned long long b2 = s_pm[st0 - 1 - base];
            if (b2 < km) km = b2;
          }
        } else {
          km = carry_closed;
        }
        bool kept = in && !dd;
        if (kept && mk.known) kept = !(km < pk(mk));
        if (in) keep[i] = kept ? 1 : 0;
        if (kept) {
          kmin = min(kmin, rk);
          kmax = max(kmax, rk);
        }
        // carries: the chunk's last position
        const uint32_t L = min(y, base + blockDim.x) - 1 - base;
        const uint32_t rsL = s_rs[L];
        if (rsL) {
          const uint32_t st0 = rsL - 1;
          unsigned long long c2 = carry_all;
          if (st0 > base && s_pm[st0 - 1 - base] < c2) c2 = s_pm[st0 - 1 - base];
          carry_closed = c2;
        }
        if (s_pm[L] < carry_all) carry_all = s_pm[L];
        open_rank = key(ord[base + L]).rank;
        __syncthreads();
      }
      // retained-rank summary: -1 none, the single rank, -2 several
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(FULL, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(FULL, kmax, o));
      }
      if ((tid & 31) == 0) {
        s_red[0][tid >> 5] = kmin;
        s_red[1][tid >> 5] = kmax;
      }
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
          kmin = min(kmin, s_red[0][w]);
          kmax = max(kmax, s_red[1][w]);
        }
        const int32_t gs = kmin == INT_MAX ? -1 : (kmin == kmax ? kmin : -2);
        if (g >= 0) {
          rsum[g] = gs;
          if (masks && gs != -1) {
            NE[g >> 6] |= 1ull << (g & 63);
            if (gs == -2) MU[g >> 6] |= 1ull << (g & 63);
          }
          if (RB && gs >= 0 && static_cast<uint32_t>(gs) < Rs)
            RB[static_cast<uint64_t>(minpos[gs]) * words + (g >> 6)] |= 1ull << (g & 63);
        }
      }
      __syncthreads();
    }
  } else if (tid < 32) {
    const int lane = tid;
    const bool masks = words <= kMaskWords;
    for (int l = lane; l < K; l += 32) rsum[l] = -1;
    for (int w = lane; w < kMaskWords; w += 32) NE[w] = MU[w] = 0;
    __syncwarp();
    auto plt = [](uint64_t d0, uint64_t t0, uint64_t r0, uint64_t d1, uint64_t t1,
                  uint64_t r1) { return prog_less(d0, t0, r0, d1, t1, r1); };
    uint32_t x = 0;
    while (x < C) {
      long long c0 = clock64();
      const int64_t op = key(ord[x]).op;
      // group end: first sorted position with a different op
      uint32_t y = x + 1;
      for (uint32_t b0 = x + 1; b0 < C; b0 += 32) {
        const uint32_t i = b0 + lane;
        const unsigned mm = __ballot_sync(FULL, i < C && key(ord[i]).op != op);
        if (mm) {
          y = b0 + __ffs(mm) - 1;
          break;
        }
        y = min(C, b0 + 32);
      }
      cy_y += clock64() - c0;
      const bool dag = op >= 0 && K >= 2;
      const int g = dag ? cidx[op - lo] : -1;
      const unsigned long long* row = dag ? bits + (op - lo) * words : nullptr;
      // Same-op rule, in parallel. Inside a group the candidates run in rank
      // order and equal ranks are adjacent, so "retained u of another rank
      // before c" = retained candidates before c's rank run. A candidate
      // with progress above the least retained progress is dropped, so the
      // least RETAINED progress before a run equals the least progress of
      // ALL dependency-surviving known candidates before it (the minimum
      // itself is always retained). Hence c survives iff !dd and
      // !(KM(run start) < prog(c)), KM = exclusive prefix minimum over the
      // group at run granularity — no step depends on another's verdict.
      const uint64_t INF = ~0ull;
      uint64_t kcd = INF, kct = INF, kcr = INF;  // min before the open run
      uint64_t kod = INF, kot = INF, kor = INF;  // min inside the open run
      int32_t orank = INT_MIN;                   // rank of the open run
      int32_t kmin = INT_MAX, kmax = INT_MIN;    // retained ranks of the group
      for (uint32_t base = x; base < y; base += 32) {
        const uint32_t i = base + lane;
        bool dd = false;
        long long c1 = clock64();
        const int32_t rr = i < y ? key(ord[i]).rank : -1;
        const unsigned long long* rb =
            RB && rr >= 0 && static_cast<uint32_t>(rr) < Rs ? RB + static_cast<uint64_t>(minpos[rr]) * words
                                                            : nullptr;
        if (i < y && dag && rb) {
          // eight words of the ancestor row and of RB per round trip (the
          // rows of wide op windows live in global memory)
          for (int w0 = 0; w0 < words && !dd; w0 += 8) {
            unsigned long long av[8], rv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              av[q] = w0 + q < words ? row[w0 + q] : 0ull;
              rv[q] = w0 + q < words ? rb[w0 + q] : 0ull;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (w0 + q < words)
                dd = dd || (av[q] & MU[w0 + q]) || (av[q] & NE[w0 + q] & ~MU[w0 + q] & ~rv[q]);
          }
        } else if (i < y && dag) {
          const int32_t r = rr;
          for (int w = 0; w < words && !dd; ++w) {
            unsigned long long av = row[w];
            if (masks) {
              if (av & MU[w]) {
                dd = true;
                break;
              }
              av &= NE[w];
            }
            while (av && !dd) {
              const int l = w * 64 + __ffsll(av) - 1;
              const int32_t q = rsum[l];
              dd = q != -1 && q != r;
              av &= av - 1;
            }
          }
        }
        long long c2 = clock64();
        cy_dd += c2 - c1;
        const bool in = i < y;
        ExoKey mk{};
        if (in) mk = key(ord[i]);
        const int32_t rk = in ? mk.rank : INT_MAX;
        // this lane's contribution to the minimum
        uint64_t vd = INF, vt = INF, vr = INF;
        if (in && !dd && mk.known) {
          vd = mk.done;
          vt = mk.tx;
          vr = mk.ready;
        }
        // exclusive prefix minimum over lanes (lexicographic triples)
        uint64_t pd = vd, pt = vt, pr = vr;  // inclusive first
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint64_t qd = __shfl_up_sync(FULL, pd, o), qt = __shfl_up_sync(FULL, pt, o),
                         qr = __shfl_up_sync(FULL, pr, o);
          if (lane >= o && plt(qd, qt, qr, pd, pt, pr)) {
            pd = qd;
            pt = qt;
            pr = qr;
          }
        }
        // run starts inside the batch
        const int32_t prev_rank = __shfl_up_sync(FULL, rk, 1);
        const bool start = in && (lane == 0 ? rk != orank : rk != prev_rank);
        const unsigned sm = __ballot_sync(FULL, start);
        const unsigned upto = sm & (lane == 31 ? FULL : ((2u << lane) - 1u));
        // KM for this lane's run
        uint64_t md = kcd, mt = kct, mr = kcr;
        {
          const int s = upto ? 31 - __clz(upto) : -1;  // start of my run in batch
          // min over batch lanes [0, s) = inclusive prefix at s - 1
          const int src = s > 0 ? s - 1 : 0;
          const uint64_t bd = __shfl_sync(FULL, pd, src), bt = __shfl_sync(FULL, pt, src),
                         br = __shfl_sync(FULL, pr, src);
          if (s >= 0) {  // my run starts in this batch: closed + open run + lanes before s
            if (plt(kod, kot, kor, md, mt, mr)) {
              md = kod;
              mt = kot;
              mr = kor;
            }
            if (s > 0 && plt(bd, bt, br, md, mt, mr)) {
              md = bd;
              mt = bt;
              mr = br;
            }
          }
        }
        bool kept = in && !dd;
        if (kept && mk.known) kept = !plt(md, mt, mr, mk.done, mk.tx, mk.ready);
        if (in) keep[i] = kept ? 1 : 0;
        if (kept) {
          kmin = min(kmin, rk);
          kmax = max(kmax, rk);
        }
        // carry: the open run after this batch is the last lane's run
        const unsigned last = __ballot_sync(FULL, in);
        const int ll = 31 - __clz(last);
        const int ls = __shfl_sync(FULL, upto ? 31 - __clz(upto) : -1, ll);
        const uint64_t ad = __shfl_sync(FULL, pd, ll), at = __shfl_sync(FULL, pt, ll),
                       ar = __shfl_sync(FULL, pr, ll);  // min over the whole batch
        if (ls >= 0) {
          // closed = everything before the last run's start
          const int src = ls > 0 ? ls - 1 : 0;
          const uint64_t bd = __shfl_sync(FULL, pd, src), bt = __shfl_sync(FULL, pt, src),
                         br = __shfl_sync(FULL, pr, src);
          if (plt(kod, kot, kor, kcd, kct, kcr)) {
            kcd = kod;
            kct = kot;
            kcr = kor;
          }
          if (ls > 0 && plt(bd, bt, br, kcd, kct, kcr)) {
            kcd = bd;
            kct = bt;
            kcr = br;
          }
          // open run = lanes [ls, ll]: min of their values
          uint64_t od = INF, ot = INF, orr = INF;
          if (lane >= ls && lane <= ll) {
            od = vd;
            ot = vt;
            orr = vr;
          }
#pragma unroll
          for (int o = 16; o; o >>= 1) {
            const uint64_t qd = __shfl_xor_sync(FULL, od, o), qt = __shfl_xor_sync(FULL, ot, o),
                           qr = __shfl_xor_sync(FULL, orr, o);
            if (plt(qd, qt, qr, od, ot, orr)) {
              od = qd;
              ot = qt;
              orr = qr;
            }
          }
          kod = od;
          kot = ot;
          kor = orr;
        } else if (plt(ad, at, ar, kod, kot, kor)) {  // the open run continues
          kod = ad;
          kot = at;
          kor = ar;
        }
        orank = __shfl_sync(FULL, rk, ll);
        cy_walk += clock64() - c2;
      }
      // retained-rank summary: -1 none, the single rank, -2 several
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(FULL, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(FULL, kmax, o));
      }
      const int32_t gs = kmin == INT_MAX ? -1 : (kmin == kmax ? kmin : -2);
      if (g >= 0 && lane == 0) {
        rsum[g] = gs;
        if (masks && gs != -1) {
          NE[g >> 6] |= 1ull << (g & 63);
          if (gs == -2) MU[g >> 6] |= 1ull << (g & 63);
        }
        if (RB && gs >= 0 && static_cast<uint32_t>(gs) < Rs)
          RB[static_cast<uint64_t>(minpos[gs]) * words + (g >> 6)] |= 1ull << (g & 63);
      }
      __syncwarp();
      x = y;
    }
  }
  __syncthreads();
  clk4 = clock64();
  // 4. report: exonerated in sorted order; suspects = first retained entry
  //    per rank (its evidence in that order); suspects sorted by rank.
  const int32_t R = a.s.R > 0 ? a.s.R : 1;
  const uint32_t rw = static_cast<uint32_t>(R + 31) / 32;
  for (int32_t r = tid; r < R; r += blockDim.x) minpos[r] = 0xFFFFFFFFu;
  for (uint32_t w = tid; w < rw; w += blockDim.x) rbits[w] = 0;
  __syncthreads();
  for (uint32_t x = tid; x < C; x += blockDim.x)
    if (keep[x]) {
      const int32_t r = cands[ord[x]].rank;
      if (r >= 0 && r < R) atomicMin(&minpos[r], x);
    }
  __syncthreads();
  csg_suspect* sus = a.sus + tp.sus_off;  // [C] suspects, then [C] exonerated
  csg_suspect* exo = sus + C;
  csg_evidence* evo = a.ev + tp.ev_off;
  uint32_t run_e = 0, run_s = 0, run_v = 0;
  const int nwb = blockDim.x >> 5;
  for (uint32_t base = 0; base < C; base += blockDim.x) {
    const uint32_t x = base + tid;
    const bool valid = x < C;
    Cand c;
    if (valid) c = cands[ord[x]];
    const bool isexo = valid && !keep[x];
    const bool isfirst = valid && keep[x] && c.rank >= 0 && c.rank < R &&
                         minpos[c.rank] == x;
    const uint32_t evn = isfirst ? c.ev_n : 0;
    // block exclusive scan of (isexo, isfirst, evn)
    uint32_t e = isexo, f = isfirst, v = evn;
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t e2 = __shfl_up_sync(FULL, e, o), f2 = __shfl_up_sync(FULL, f, o),
                     v2 = __shfl_up_sync(FULL, v, o);
      if (lane >= o) {
        e += e2;
        f += f2;
        v += v2;
      }
    }
    if (lane == 31) {
      scan3[warp][0] = e;
      scan3[warp][1] = f;
      scan3[warp][2] = v;
    }
    __syncthreads();
    uint32_t be = 0, bf = 0, bv = 0, te = 0, tf = 0, tv = 0;
    for (int q = 0; q < nwb; ++q) {
      if (q < warp) {
        be += scan3[q][0];
        bf += scan3[q][1];
        bv += scan3[q][2];
      }
      te += scan3[q][0];
      tf += scan3[q][1];
      tv += scan3[q][2];
    }
    if (isexo) exo[run_e + be + e - 1] = to_suspect(c);
    if (isfirst) {
      sus[run_s + bf + f - 1] = to_suspect(c);
      atomicOr(&rbits[c.rank >> 5], 1u << (c.rank & 31));
      const uint32_t v0 = run_v + bv + v - evn;
      for (uint32_t q = 0; q < evn; ++q) evo[v0 + q] = a.cev[c.ev_off + q];
    }
    run_e += te;
    run_s += tf;
    run_v += tv;
    __syncthreads();
  }
  clk5 = clock64();
  // suspect ranks are unique: rank-sorted position = number of suspect ranks
  // below it (prefix popcount over the rank bitmap)
  if (tid == 0) {
    uint32_t acc = 0;
    for (uint32_t w = 0; w < rw; ++w) {
      const uint32_t c = __popc(rbits[w]);
      woff[w] = acc;
      acc += c;
    }
  }
  __syncthreads();
  for (uint32_t i = tid; i < run_s; i += blockDim.x) {
    const int32_t r = sus[i].rank;
    const uint32_t pos = woff[r >> 5] + __popc(rbits[r >> 5] & ((1u << (r & 31)) - 1u));
    stmp[pos] = sus[i];
  }
  __syncthreads();
  for (uint32_t i = tid; i < run_s; i += blockDim.x) sus[i] = stmp[i];
  if (tid == 0) {
    if (a.debug)
      printf("exo trip %d C=%u K=%d lo=%lld hi=%lld words=%d phases (cycles): sort %lld "
             "ops %lld dag %lld sweep %lld [y %lld dd %lld walk %lld] report %lld order %lld\n",
             tp.j, C, K, (long long)lo, (long long)hi, words, clk1 - clk0, clk2 - clk1,
             clk3 - clk2, clk4 - clk3, cy_y, cy_dd, cy_walk, clk5 - clk4,
             (long long)clock64() - clk5);
    o.verdict = run_s ? CSG_VERDICT_SUSPECTS : CSG_VERDICT_UNDETERMINED;
    o.n_sus = run_s;
    o.exo_off = tp.sus_off + C;
    o.n_exo = run_e;
    o.n_ev = run_v;
    a.out[tp.j] = o;
  }
}

// Dense packing of every trip's suspects, exonerated and evidence, copied
// on the device straight into mapped pinned host memory.
__global__ void k_pack(const TripOut* __restrict__ out, int32_t J,
                       const csg_suspect* __restrict__ sus,
                       const csg_evidence* __restrict__ ev,
                       csg_suspect* __restrict__ osus,
                       csg_evidence* __restrict__ oev, FetchArgs fa,
                       unsigned long long* flag, unsigned long long v,
                       unsigned* __restrict__ fdone) {
  pdl_wait();
  pdl_trigger();
  // block (j, kind, slice): its packed offset is the sum of the earlier
  // regions' counts in (trip, suspects / exonerated / evidence) order; the
  // host derives the same offsets from the fetched trip table. grid.y slices
  // each region (the PCIe writes into mapped memory of one block were the
  // kernel's time).
  const int32_t j = blockIdx.x / 3, kind = blockIdx.x % 3;
  __shared__ uint32_t s_dst;
  if (threadIdx.x == 0) {
    uint32_t d = 0;
    for (int32_t q = 0; q < j; ++q) d += kind < 2 ? out[q].n_sus + out[q].n_exo : out[q].n_ev;
    if (kind == 1) d += out[j].n_sus;
    s_dst = d;
  }
  __syncthreads();
  const TripOut& t = out[j];
  const uint32_t n = kind == 0 ? t.n_sus : kind == 1 ? t.n_exo : t.n_ev;
  const uint32_t s0 = kind == 0 ? t.sus_off : kind == 1 ? t.exo_off : t.ev_off;
  const uint32_t d0 = s_dst;
  for (uint32_t i = blockIdx.y * blockDim.x + threadIdx.x; i < n; i += gridDim.y * blockDim.x) {
    if (kind < 2) osus[d0 + i] = sus[s0 + i];
    else oev[d0 + i] = ev[s0 + i];
  }
  // the batch's tail (error word, pool usage, trip table) rides on the
  // last block: no k_fetch launch behind the pack
  fetch_tail(fa, flag, v, fdone);
}

__global__ void __launch_bounds__(kDecideThreads)
    k_decide(DecideArgs a) {
  extern __shared__ __align__(16) unsigned char dyn[];
  BlockShared& sh = *reinterpret_cast<BlockShared*>(dyn);
  const int32_t j = blockIdx.x;
  if (threadIdx.x == 0) {
    sh.abort = 0;
    sh.nsus = sh.nexo = 0;
    sh.nev = 0;
    sh.sus_base = sh.exo_base = sh.ev_base = 0;
  }
  __syncthreads();
  uint32_t* scratch = a.pools.u32 + (a.js_of[j] >= 0 ? static_cast<uint64_t>(j) * a.scratch_per_trip : 0);
  const int32_t naff = a.n_aff[j];
  if (naff == 0 || a.m.opn == 0) {
    write_trip(a, j, CSG_VERDICT_FALSE_TRIGGER, naff, a.N, sh);
    return;
  }
  if (a.trip_kind[j] == CSG_TRIGGER_FAILURE) return;  // k_exonerate
  if (a.phase == 1 && a.sl_par) return;  // k_sl_late .. k_sl_emit
  if (a.phase == 1) decide_straggler(a, j, sh, scratch);
  else decide_straggler_finish(a, j, sh, scratch);
}

// Cohort medians ahead of the self-evidence filter: block (j, q, nm)
// computes the cohort (op name nm, iteration it_lo(j) + q) of straggler
// trip j, where [it_lo(j), it_hi(j)] spans the iteration windows of the
// trip's candidates, and publishes it in the batch-wide table — every cohort
// a candidate can ask for is computed once, all in parallel, instead of by
// the first candidate block that needs it while others wait.
constexpr int kCohortNames = 4;  // AllGather, ReduceScatter, AllReduce, Send
__global__ void __launch_bounds__(kDecideThreads) k_cohorts(DecideArgs a) {
  extern __shared__ __align__(16) unsigned char dyn[];
  BlockShared& sh = *reinterpret_cast<BlockShared*>(dyn);
  const int32_t j = blockIdx.x;
  const int32_t q = blockIdx.y;
  const uint8_t nm = static_cast<uint8_t>(blockIdx.z);
  if (a.trip_kind[j] == CSG_TRIGGER_FAILURE) return;
  const StragState S = a.state[j];
  if (S.C <= 0) return;
  const Cand* cands = a.pools.cand + S.cand_base;
  long long lo = LLONG_MAX, hi = LLONG_MIN;
  for (int x = threadIdx.x; x < S.C; x += blockDim.x) {
    const Cand& c = cands[x];
    if (c.it_hi < c.it_lo) continue;
    lo = min(lo, static_cast<long long>(c.it_lo));
    hi = max(hi, static_cast<long long>(c.it_hi));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(FULL, lo, o));
    hi = max(hi, __shfl_xor_sync(FULL, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    sh.red_l[threadIdx.x >> 5] = lo;
    sh.red_l[16 + (threadIdx.x >> 5)] = hi;
  }
  __syncthreads();
  lo = LLONG_MAX;
  hi = LLONG_MIN;
  for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
    lo = min(lo, sh.red_l[w]);
    hi = max(hi, sh.red_l[16 + w]);
  }
  __syncthreads();
  // every iteration of the trip's candidate windows (grid.y strides them)
  for (long long it = lo + q; lo <= hi && it <= hi; it += gridDim.y) {
    const unsigned long long ckey =
        (static_cast<unsigned long long>(j) << 44) ^
        (static_cast<unsigned long long>(nm) << 36) ^
        (static_cast<unsigned long long>(it) & ((1ull << 36) - 1));
    __shared__ int s_slot;
    if (threadIdx.x == 0) {
      s_slot = -1;
      const uint32_t mask = a.coh_cap - 1;
      uint32_t h = static_cast<uint32_t>((ckey * 0x9E3779B97F4A7C15ull) >> 40) & mask;
      for (uint32_t probe = 0; probe < a.coh_cap; ++probe, h = (h + 1) & mask) {
        const unsigned long long k = atomicCAS(a.coh_key + h, ~0ull, ckey);
        if (k == ~0ull) {
          s_slot = static_cast<int>(h);
          break;
        }
        if (k == ckey) break;  // already there
      }
    }
    __syncthreads();
    if (s_slot >= 0) {
      const double med = cohort_median(a, it, nm, a.trip_t[j], sh);
      if (threadIdx.x == 0) {
        a.coh_val[s_slot] = med;
        __threadfence();
        atomicExch(a.coh_state + s_slot, 2u);
      }
    }
    __syncthreads();
  }
}

// The cohorts k_sf_fast claimed (state 0): one block per claimed slot.
__global__ void __launch_bounds__(kDecideThreads) k_cohorts_lazy(DecideArgs a) {
  extern __shared__ __align__(16) unsigned char dyn[];
  BlockShared& sh = *reinterpret_cast<BlockShared*>(dyn);
  __shared__ int s_mine, s_slot2;
  for (uint32_t h = blockIdx.x; h < a.coh_cap; h += gridDim.x) {
    if (a.coh_key[h] == ~0ull || a.coh_state[h] == 2u) continue;
    const longlong2 mt = a.coh_meta[h];
    const int32_t j = static_cast<int32_t>(mt.y >> 8);
    const uint8_t nm = static_cast<uint8_t>(mt.y & 0xff);
    const double t = a.trip_t[j];
    // The (op name, iteration) cohort over all of its entries, once per
    // batch: trips whose time follows every entry use it as is (the ts <= t
    // filter keeps everything); the claimer computes, the others wait.
    const unsigned long long key2 =
        (static_cast<unsigned long long>(nm) << 48) ^
        (static_cast<unsigned long long>(mt.x) & ((1ull << 48) - 1));
    if (threadIdx.x == 0) {
      s_mine = 0;
      s_slot2 = -1;
      const uint32_t mask = a.coh_cap - 1;
      uint32_t h2 = static_cast<uint32_t>((key2 * 0x9E3779B97F4A7C15ull) >> 40) & mask;
      for (uint32_t probe = 0; probe < a.coh_cap; ++probe, h2 = (h2 + 1) & mask) {
        const unsigned long long k2 = atomicCAS(a.coh2_key + h2, ~0ull, key2);
        if (k2 == ~0ull || k2 == key2) {
          s_mine = k2 == ~0ull;
          s_slot2 = static_cast<int>(h2);
          break;
        }
      }
    }
    __syncthreads();
    double med = 0;
    bool done = false;
    if (s_slot2 >= 0) {
      const int h2 = s_slot2;
      if (s_mine) {
        const double mall = cohort_median(a, mt.x, nm, INFINITY, sh);
        // latest timestamp of the cohort's entries
        int64_t olo, ohi;
        iter_ops(mt.x, a.m.opn, olo, ohi);
        const bool empty = ohi < a.min_op;
        const uint64_t k0 = olo < a.min_op ? 0 : static_cast<uint64_t>(olo - a.min_op);
        const uint64_t k1 = empty ? 0 : static_cast<uint64_t>(ohi - a.min_op);
        uint64_t cb, ce;
        op_segment(a, k0, k1, empty, sh, cb, ce);
        double mx = -INFINITY;
        for (uint64_t y = cb + threadIdx.x; y < ce; y += blockDim.x)
          if (a.op_nm[y] == nm) mx = fmax(mx, a.op_ts[y]);
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
        if ((threadIdx.x & 31) == 0) sh.red_u[0][threadIdx.x >> 5] = dkey(mx);
        __syncthreads();
        if (threadIdx.x == 0) {
          unsigned long long m2 = 0;
          for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) m2 = max(m2, sh.red_u[0][q]);
          a.coh2_val[h2] = mall;
          a.coh2_mx[h2] = dkey_inv(m2);
          __threadfence();
          atomicExch(a.coh2_state + h2, 2u);
        }
        __syncthreads();
      } else if (threadIdx.x == 0) {
        while (*reinterpret_cast<volatile unsigned*>(a.coh2_state + h2) != 2u) {
        }
        __threadfence();
      }
      __syncthreads();
      const double mx = *reinterpret_cast<volatile double*>(a.coh2_mx + h2);
      if (mx <= t) {
        med = *reinterpret_cast<volatile double*>(a.coh2_val + h2);
        done = true;
      }
    }
    if (!done) med = cohort_median(a, mt.x, nm, t, sh);
    if (threadIdx.x == 0) {
      a.coh_val[h] = med;
      __threadfence();
      atomicExch(a.coh_state + h, 2u);
    }
    __syncthreads();
  }
}

// The claimed cohorts as one multi-block radix select: every (trip, op name,
// iteration) slot k_sf_fast claimed becomes an item over its iteration's
// op-index range; eight 8-bit digit passes run over all
// items' entries at once (the top digit's pass also counts the entries;
// 4096-entry units spread over the whole GPU, block
// histograms merged into per-item global ones), a tiny pick kernel narrows
// each item's prefix between passes. The lower median of an item is element
// (m - 1) / 2 of its entries with op name nm and ts <= t; fewer than two
// entries give 0 (rca.cpp:833-840: the op is then skipped).
struct CohItem {
  uint32_t slot;
  uint32_t m;       // matching entries
  uint64_t cb, ce;  // op-index range of the iteration
  uint64_t unit0;   // first work unit
  uint64_t prefix;  // selected key bits so far
  uint64_t kth;     // rank still to find inside the prefix
  double t;
  int32_t nm;
  int32_t pad;
  uint64_t off;    // compacted keys of the item: ckeys[off, off + m2)
  uint64_t unit2;  // first work unit over the compacted keys
  uint32_t m2;     // entries left after the digits down to kCohCompactShift
  uint32_t fill;
};
struct CohPlan {
  unsigned n_items;
  unsigned compact;  // the compacted keys fit: the low digits' passes read them
  unsigned long long units;
  unsigned long long units2;
  unsigned long long total2;
};
static_assert(sizeof(CohPlan) <= 64, "CohPlan sits in the first 64 bytes of the items buffer");
constexpr int kCohUnit = 4096;
constexpr uint32_t kCohItemsCap = 8192;
// After the digits 63..40 the surviving entries of each item (a handful of
// durations sharing sign, exponent and 12 mantissa bits) are compacted, so
// the five low digits' passes stop rescanning the iterations' op ranges.
constexpr int kCohCompactShift = 40;

// Exclusive block scan of n values val(i) -> put(i, prefix); returns the total.
template <typename V, typename P>
__device__ unsigned long long block_excl_scan_n(uint32_t n, V val, P put,
                                                unsigned long long* s_w,
                                                unsigned long long* s_carry) {
  if (threadIdx.x == 0) *s_carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < n; base += blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const unsigned long long v = i < n ? val(i) : 0ull;
    const unsigned long long inc = block_incl_scan(
        v, s_w, [](unsigned long long x, unsigned long long y) { return x + y; });
    const unsigned long long c0 = *s_carry;
    if (i < n) put(i, c0 + inc - v);
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) *s_carry = c0 + inc;
    __syncthreads();
  }
  return *s_carry;
}

__global__ void __launch_bounds__(1024) k_coh_collect(DecideArgs a, CohItem* __restrict__ items,
                                                      CohPlan* __restrict__ plan,
                                                      uint32_t* __restrict__ hist) {
  __shared__ unsigned s_n;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (uint32_t b0 = 0; b0 < a.coh_cap; b0 += blockDim.x) {
    const uint32_t h = b0 + threadIdx.x;
    const bool want = h < a.coh_cap && a.coh_key[h] != ~0ull && a.coh_state[h] != 2u;
    const unsigned mm = __ballot_sync(FULL, want);
    unsigned at = 0;
    if (lane == 0 && mm) at = atomicAdd(&s_n, static_cast<unsigned>(__popc(mm)));
    at = __shfl_sync(FULL, at, 0) + __popc(mm & ((1u << lane) - 1u));
    if (want && at >= kCohItemsCap) atomicExch(a.coh_state + h, 3u);  // abandoned
    if (want && at < kCohItemsCap) {
      const longlong2 mt = a.coh_meta[h];
      const int32_t j = static_cast<int32_t>(mt.y >> 8);
      CohItem it;
      it.slot = h;
      it.m = 0;
      it.nm = static_cast<int32_t>(mt.y & 0xff);
      it.t = a.trip_t[j];
      int64_t olo, ohi;
      iter_ops(mt.x, a.m.opn, olo, ohi);
      olo = max(olo, a.min_op);
      ohi = min(ohi, a.max_op);
      if (olo <= ohi) {
        it.cb = a.opoff[olo - a.min_op];
        it.ce = a.opoff[ohi - a.min_op + 1];
      } else {
        it.cb = it.ce = 0;
      }
      it.prefix = 0;
      it.kth = 0;
      it.unit0 = 0;
      it.pad = 0;
      items[at] = it;
    }
  }
  __syncthreads();
  const unsigned n = min(s_n, kCohItemsCap);
  for (uint64_t i = threadIdx.x; i < static_cast<uint64_t>(n) * 256; i += blockDim.x) hist[i] = 0;
  __shared__ unsigned long long s_w[32], s_carry;
  const unsigned long long u = block_excl_scan_n(
      n, [&](uint32_t i) { return (items[i].ce - items[i].cb + kCohUnit - 1) / kCohUnit; },
      [&](uint32_t i, unsigned long long x) { items[i].unit0 = x; }, s_w, &s_carry);
  if (threadIdx.x == 0) {
    plan->n_items = n;
    plan->units = u;
    plan->compact = 0;
  }
}

// shift < 0: count pass only (unused); else the digit at `shift` of the keys matching the
// item's prefix above it
__global__ void __launch_bounds__(256) k_coh_pass(DecideArgs a, CohItem* __restrict__ items,
                                                  const CohPlan* __restrict__ plan,
                                                  uint32_t* __restrict__ hist, int shift,
                                                  const unsigned long long* __restrict__ ckeys) {
  __shared__ uint32_t sh[256];
  __shared__ uint32_t s_cnt;
  const unsigned n = plan->n_items;
  const int lane = threadIdx.x & 31;
  if (shift < kCohCompactShift && plan->compact) {
    // the low digits over the compacted keys (all pass the op-name / time
    // filters and match the prefix down to kCohCompactShift)
    const unsigned long long U2 = plan->units2;
    const uint64_t mask = ~0ull << (shift + 8);
    for (unsigned long long u = blockIdx.x; u < U2; u += gridDim.x) {
      unsigned lo = 0, hi = n;
      while (hi - lo > 1) {
        const unsigned mid = (lo + hi) >> 1;
        if (items[mid].unit2 <= u) lo = mid; else hi = mid;
      }
      const CohItem it = items[lo];
      const uint64_t y0 = it.off + (u - it.unit2) * kCohUnit;
      const uint64_t y1 = min(it.off + it.m2, y0 + kCohUnit);
      for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 0;
      __syncthreads();
      for (uint64_t b0 = y0; b0 < y1; b0 += blockDim.x) {
        const uint64_t y = b0 + threadIdx.x;
        uint32_t d = 256;
        if (y < y1) {
          const uint64_t key = ckeys[y];
          if ((key & mask) == (it.prefix & mask)) d = static_cast<uint32_t>((key >> shift) & 255);
        }
        const unsigned peers = __match_any_sync(FULL, d);
        if (d < 256 && lane == __ffs(peers) - 1) atomicAdd(&sh[d], static_cast<uint32_t>(__popc(peers)));
      }
      __syncthreads();
      for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[static_cast<uint64_t>(lo) * 256 + i], sh[i]);
      __syncthreads();
    }
    return;
  }
  const unsigned long long U = plan->units;
  for (unsigned long long u = blockIdx.x; u < U; u += gridDim.x) {
    unsigned lo = 0, hi = n;  // items[lo].unit0 <= u < items[hi].unit0
    while (hi - lo > 1) {
      const unsigned mid = (lo + hi) >> 1;
      if (items[mid].unit0 <= u) lo = mid; else hi = mid;
    }
    const CohItem it = items[lo];
    const uint64_t y0 = it.cb + (u - it.unit0) * kCohUnit;
    const uint64_t y1 = min(it.ce, y0 + kCohUnit);
    const uint64_t mask = shift >= 56 || shift < 0 ? 0ull : (~0ull << (shift + 8));
    if (shift >= 0) {
      for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 0;
    } else if (threadIdx.x == 0) {
      s_cnt = 0;
    }
    __syncthreads();
    uint32_t cnt = 0;
    const bool counting = shift < 0 || shift == 56;  // the top digit's pass counts too
    if (shift == 56 && threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    for (uint64_t b0 = y0; b0 < y1; b0 += blockDim.x) {
      const uint64_t y = b0 + threadIdx.x;
      uint32_t d = 256;
      if (y < y1 && a.op_nm[y] == it.nm && a.op_ts[y] <= it.t) {
        if (counting) ++cnt;
        if (shift >= 0) {
          const uint64_t key = dkey(a.op_dur[y]);
          if ((key & mask) == (it.prefix & mask)) d = static_cast<uint32_t>((key >> shift) & 255);
        }
      }
      if (shift >= 0) {
        const unsigned peers = __match_any_sync(FULL, d);
        if (d < 256 && lane == __ffs(peers) - 1) atomicAdd(&sh[d], static_cast<uint32_t>(__popc(peers)));
      }
    }
    if (counting) {
#pragma unroll
      for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
      if (lane == 0 && cnt) atomicAdd(&s_cnt, cnt);
    }
    __syncthreads();
    if (counting && threadIdx.x == 0 && s_cnt) atomicAdd(&items[lo].m, s_cnt);
    if (shift >= 0) {
      for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[static_cast<uint64_t>(lo) * 256 + i], sh[i]);
    }
    __syncthreads();
  }
}

// shift < 0: after the count pass (kth = (m - 1) / 2); else pick the digit
// bucket holding the kth key; last pass (shift == 0) publishes the medians.
__global__ void k_coh_pick(DecideArgs a, CohItem* __restrict__ items,
                           const CohPlan* __restrict__ plan, uint32_t* __restrict__ hist,
                           int shift) {
  const unsigned n = plan->n_items;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    CohItem& it = items[i];
    if (shift < 0 || shift == 56) {
      it.kth = it.m >= 1 ? (it.m - 1) / 2 : 0;
      if (shift < 0) continue;
    }
    uint32_t* hh = hist + static_cast<uint64_t>(i) * 256;
    uint64_t acc = 0;
    int bsel = 255;
    for (int b = 0; b < 256; ++b) {
      if (acc + hh[b] > it.kth) {
        bsel = b;
        break;
      }
      acc += hh[b];
    }
    if (shift == kCohCompactShift) it.m2 = hh[bsel];
    for (int b = 0; b < 256; ++b) hh[b] = 0;
    it.prefix |= static_cast<uint64_t>(bsel) << shift;
    it.kth -= acc;
    if (shift == 0) {
      a.coh_val[it.slot] = it.m < 2 ? 0.0 : dkey_inv(it.prefix);
      __threadfence();
      atomicExch(a.coh_state + it.slot, 2u);
    }
  }
}

// Offsets of the items' compacted keys; compaction only when they fit.
__global__ void __launch_bounds__(1024) k_coh_offsets(CohItem* __restrict__ items,
                                                      CohPlan* __restrict__ plan,
                                                      unsigned long long cap) {
  __shared__ unsigned long long s_w[32], s_carry;
  const unsigned n = plan->n_items;
  const unsigned long long tot = block_excl_scan_n(
      n, [&](uint32_t i) { return static_cast<unsigned long long>(items[i].m2); },
      [&](uint32_t i, unsigned long long x) {
        items[i].off = x;
        items[i].fill = 0;
      },
      s_w, &s_carry);
  const unsigned long long u2 = block_excl_scan_n(
      n, [&](uint32_t i) { return (static_cast<unsigned long long>(items[i].m2) + kCohUnit - 1) / kCohUnit; },
      [&](uint32_t i, unsigned long long x) { items[i].unit2 = x; }, s_w, &s_carry);
  if (threadIdx.x == 0) {
    plan->total2 = tot;
    plan->units2 = u2;
    plan->compact = tot <= cap ? 1u : 0u;
  }
}

// The entries of each item matching its prefix down to kCohCompactShift,
// copied (keys only, any order: a selection) into ckeys.
__global__ void __launch_bounds__(256) k_coh_compact(DecideArgs a, CohItem* __restrict__ items,
                                                     const CohPlan* __restrict__ plan,
                                                     unsigned long long* __restrict__ ckeys) {
  if (!plan->compact) return;
  const unsigned n = plan->n_items;
  const unsigned long long U = plan->units;
  const int lane = threadIdx.x & 31;
  const uint64_t mask = ~0ull << kCohCompactShift;
  for (unsigned long long u = blockIdx.x; u < U; u += gridDim.x) {
    unsigned lo = 0, hi = n;
    while (hi - lo > 1) {
      const unsigned mid = (lo + hi) >> 1;
      if (items[mid].unit0 <= u) lo = mid; else hi = mid;
    }
    const CohItem it = items[lo];
    const uint64_t y0 = it.cb + (u - it.unit0) * kCohUnit;
    const uint64_t y1 = min(it.ce, y0 + kCohUnit);
    for (uint64_t b0 = y0; b0 < y1; b0 += blockDim.x) {
      const uint64_t y = b0 + threadIdx.x;
      bool keep = false;
      uint64_t key = 0;
      if (y < y1 && a.op_nm[y] == it.nm && a.op_ts[y] <= it.t) {
        key = dkey(a.op_dur[y]);
        keep = (key & mask) == (it.prefix & mask);
      }
      const unsigned mm = __ballot_sync(FULL, keep);
      if (!mm) continue;
      unsigned base = 0;
      if (lane == __ffs(mm) - 1) base = atomicAdd(&items[lo].fill, static_cast<unsigned>(__popc(mm)));
      base = __shfl_sync(FULL, base, __ffs(mm) - 1);
      if (keep) ckeys[it.off + base + __popc(mm & ((1u << lane) - 1u))] = key;
    }
  }
}

// Self-evidence filter for every straggler candidate of the batch: a block
// per candidate (grid-stride over the candidates of all straggler trips,
// flattened from the per-trip counts left by k_decide phase 1). Marks
// cands[x].pad = self_faulted (rca.cpp:821-848); candidates without an
// iteration window (flow findings) are self-faulted by definition.
__global__ void __launch_bounds__(kDecideThreads) k_self_faulted(DecideArgs a) {
  extern __shared__ __align__(16) unsigned char dyn[];
  BlockShared& sh = *reinterpret_cast<BlockShared*>(dyn);
  __shared__ unsigned long long s_total;
  if (threadIdx.x == 0) {
    sh.coh_n = 0;
    unsigned long long tot = 0;
    for (int32_t j = 0; j < a.J; ++j)
      if (a.trip_kind[j] != CSG_TRIGGER_FAILURE && a.state[j].C > 0) tot += a.state[j].C;
    s_total = tot;
  }
  __syncthreads();
  const unsigned long long total = s_total;
  uint32_t* lst = a.sf_scratch + static_cast<uint64_t>(blockIdx.x) * a.sf_words;
  int32_t jcur = 0;
  unsigned long long jbase = 0;  // flattened index of trip jcur's first candidate
  for (unsigned long long w = blockIdx.x; w < total; w += gridDim.x) {
    // advance to the trip holding item w (w increases monotonically)
    while (true) {
      const bool strag = a.trip_kind[jcur] != CSG_TRIGGER_FAILURE && a.state[jcur].C > 0;
      const unsigned long long cj = strag ? static_cast<unsigned long long>(a.state[jcur].C) : 0;
      if (w < jbase + cj) break;
      jbase += cj;
      ++jcur;
    }
    const int32_t x = static_cast<int32_t>(w - jbase);
    Cand* cands = a.pools.cand + a.state[jcur].cand_base;
    const Cand c = cands[x];
    if (a.sf_fast && c.pad != 2) continue;  // decided by k_sf_fast
    const long long c0 = clock64();
    const bool sf = c.it_hi < c.it_lo ? true : self_faulted(a, jcur, c, sh, lst);
    if (threadIdx.x == 0) cands[x].pad = sf ? 1 : 0;
    if (a.debug && threadIdx.x == 0 && (w < 4 || (w >= 20000 && w < 20006)))
      printf("self_faulted item %llu trip %d cand %d rank %d it [%lld,%lld] sf %d: %lld cycles, "
             "n_mine %u distinct %u\n", w, jcur, x, c.rank, (long long)c.it_lo,
             (long long)c.it_hi, sf ? 1 : 0, (long long)clock64() - c0, sh.dbg_n, sh.dbg_d);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Straggler candidates (analyze_straggler, rca.cpp:654-789) for all trips and
// groups in parallel. The reference walks the affected groups in ascending
// order and, per group, appends (1) its late members in member order, (2)
// FlowSkewed findings of not-yet-candidate members in rank order, (3)
// FlowIncomplete findings likewise. "Not yet candidate" only depends on
// earlier groups: a rank is marked before group g's flow passes iff it is
// late in g, or late or flow-flagged in an earlier affected group with
// history (the first such group gives it a candidate either way). So every
// (trip, group) decides its candidates on its own:
//   k_sl_late   warp per (trip, affected group): window medians, late bits
//   k_sl_count  warp per (trip, affected group): flow-candidate types from
//               the member's earlier groups, candidate / evidence counts
//   k_sl_scan   block per trip: offsets in group order, pool allocation
//   k_sl_emit   warp per (trip, affected group): candidates + evidence
// ---------------------------------------------------------------------------
// Warp-collective ascending bitonic sort of n (<= cap, power-of-two P)
// ordered keys in shared memory.
__device__ void warp_bitonic_u64(unsigned long long* v, uint32_t P) {
  const int lane = threadIdx.x & 31;
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
      for (uint32_t i = lane; i < P; i += 32) {
        const uint32_t l = i ^ jj;
        if (l > i) {
          const unsigned long long x = v[i], y = v[l];
          if ((x > y) == ((i & k) == 0)) {
            v[i] = y;
            v[l] = x;
          }
        }
      }
      __syncwarp();
    }
  }
}

constexpr int kSlWarps = 4;
constexpr int kSlCap = 1024;  // members whose keys a warp sorts in shared memory
constexpr uint8_t kSlHist = 0x80;   // slot of an affected group with history
constexpr uint8_t kSlSkew = 0x10;   // FlowSkewed candidate
constexpr uint8_t kSlInc = 0x20;    // FlowIncomplete candidate

// lower median (element (m-1)/2) of m keys, warp-collective
template <typename V>
__device__ double warp_lower_median_sorted(int m, V val, unsigned long long* buf) {
  const int lane = threadIdx.x & 31;
  if (m > kSlCap) return warp_lower_median(m, [&](int i) { return dkey_inv(val(i)); });
  uint32_t P = 32;
  while (P < static_cast<uint32_t>(m)) P <<= 1;
  for (uint32_t i = lane; i < P; i += 32) buf[i] = i < static_cast<uint32_t>(m) ? val(i) : ~0ull;
  __syncwarp();
  warp_bitonic_u64(buf, P);
  const double r = dkey_inv(buf[(m - 1) / 2]);
  __syncwarp();
  return r;
}

__global__ void __launch_bounds__(kSlWarps * 32) k_sl_late(DecideArgs a, int32_t Js) {
  __shared__ unsigned long long buf[kSlWarps][kSlCap];
  __shared__ double smed[kSlWarps][2][kMaxK];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int32_t G = a.m.n_groups;
  const uint64_t w = blockIdx.x * (uint64_t)kSlWarps + wib;
  if (w >= static_cast<uint64_t>(Js) * G) return;
  const int32_t js = static_cast<int32_t>(w / G), i = static_cast<int32_t>(w % G);
  const int32_t j = a.strag_trip[js];
  if (i >= a.n_aff[j] || a.m.opn == 0) return;
  const int32_t g = a.aff[static_cast<uint64_t>(j) * G + i];
  const uint32_t mo = a.m.member_off[g];
  const int32_t m = static_cast<int32_t>(a.m.member_off[g + 1] - mo);
  if (m < 2) return;
  const uint64_t gidx = static_cast<uint64_t>(js) * G + g;
  if (a.gi[gidx].n_common < a.k) return;
  const uint64_t rowbase = static_cast<uint64_t>(js) * a.M;
  const int32_t k = a.k;
  // lower medians of the members' starts / ends per window iteration
  // (rca.cpp:670-681)
  for (int q = 0; q < k; ++q) {
    const int64_t it = a.gi_last[gidx * k + q] - a.it_min;
    const double ms = warp_lower_median_sorted(
        m, [&](int x) { return a.tbl_s[(rowbase + a.m.member_slot[mo + x]) * a.n_it + it]; },
        buf[wib]);
    const double me = warp_lower_median_sorted(
        m, [&](int x) { return a.tbl_e[(rowbase + a.m.member_slot[mo + x]) * a.n_it + it]; },
        buf[wib]);
    if (lane == 0) {
      smed[wib][0][q] = ms;
      smed[wib][1][q] = me;
    }
  }
  __syncwarp();
  for (int x = lane; x < m; x += 32) {
    uint32_t bits = 3;
    const uint64_t cell = (rowbase + a.m.member_slot[mo + x]) * a.n_it;
    for (int q = 0; q < k; ++q) {
      const int64_t it = a.gi_last[gidx * k + q] - a.it_min;
      if (dkey_inv(a.tbl_s[cell + it]) - smed[wib][0][q] < a.thr) bits &= ~1u;
      if (dkey_inv(a.tbl_e[cell + it]) - smed[wib][1][q] < a.thr) bits &= ~2u;
    }
    a.sl_late[rowbase + mo + x] = static_cast<uint8_t>(kSlHist | bits);
  }
}

__global__ void __launch_bounds__(kSlWarps * 32) k_sl_count(DecideArgs a, int32_t Js) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int32_t G = a.m.n_groups;
  const uint64_t w = blockIdx.x * (uint64_t)kSlWarps + wib;
  if (w >= static_cast<uint64_t>(Js) * G) return;
  const int32_t js = static_cast<int32_t>(w / G), i = static_cast<int32_t>(w % G);
  const int32_t j = a.strag_trip[js];
  uint2 cnt = make_uint2(0, 0);
  if (i < a.n_aff[j] && a.m.opn != 0) {
    const int32_t g = a.aff[static_cast<uint64_t>(j) * G + i];
    const uint32_t mo = a.m.member_off[g];
    const int32_t m = static_cast<int32_t>(a.m.member_off[g + 1] - mo);
    const uint64_t rowbase = static_cast<uint64_t>(js) * a.M;
    if (m >= 2 && (a.sl_late[rowbase + mo] & kSlHist)) {
      uint32_t nl = 0, nf = 0;
      for (int x = lane; x < m; x += 32) {
        const uint32_t slot = mo + x;
        uint8_t v = a.sl_late[rowbase + slot];
        const bool lt = (v & 3) != 0;
        const int32_t ff = a.fs[rowbase + slot].flags;
        uint8_t type = 0;
        if (!lt && (ff & 3)) {
          // marked by an earlier affected group with history?
          const int32_t r = a.m.members[slot];
          bool marked = false;
          if (r >= 0 && r < a.m.rank_space)
            for (uint32_t q = a.m.rg_off[r]; q < a.m.rg_off[r + 1] && !marked; ++q) {
              const int32_t g2 = a.m.rg_group[q];
              if (g2 >= g) continue;
              const uint32_t s2 = a.m.rg_slot[q];
              const uint8_t v2 = a.sl_late[rowbase + s2];
              if (!(v2 & kSlHist)) continue;
              marked = (v2 & 3) || (a.fs[rowbase + s2].flags & 3);
            }
          if (!marked) type = (ff & 1) ? kSlSkew : kSlInc;
        }
        if (type) a.sl_late[rowbase + slot] = static_cast<uint8_t>(v | type);
        nl += lt ? 1u : 0u;
        nf += type ? 1u : 0u;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        nl += __shfl_xor_sync(FULL, nl, o);
        nf += __shfl_xor_sync(FULL, nf, o);
      }
      cnt = make_uint2(nl + nf, nl * static_cast<uint32_t>(a.k) + nf);
    }
  }
  if (lane == 0) a.sl_cnt[static_cast<uint64_t>(js) * G + i] = cnt;
}

// Per straggler trip: exclusive scan of the groups' (candidates, evidence)
// counts in affected-group order (in place), pool allocation, trip state.
__global__ void __launch_bounds__(1024) k_sl_scan(DecideArgs a) {
  __shared__ uint32_t wc[32], we[32];
  __shared__ uint32_t run_c, run_e;
  __shared__ int s_hist;
  const int32_t js = blockIdx.x;
  const int32_t j = a.strag_trip[js];
  const int32_t G = a.m.n_groups;
  const int32_t naff = a.n_aff[j];
  if (naff == 0 || a.m.opn == 0) return;  // false trigger: k_decide
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    run_c = 0;
    run_e = 0;
    s_hist = 0;
  }
  __syncthreads();
  uint2* cnt = a.sl_cnt + static_cast<uint64_t>(js) * G;
  const uint64_t rowbase = static_cast<uint64_t>(js) * a.M;
  int hist = 0;
  for (int32_t b0 = 0; b0 < naff; b0 += blockDim.x) {
    const int32_t i = b0 + threadIdx.x;
    uint2 v = i < naff ? cnt[i] : make_uint2(0, 0);
    if (i < naff) {
      const int32_t g = a.aff[static_cast<uint64_t>(j) * G + i];
      if (a.m.member_off[g + 1] - a.m.member_off[g] >= 2 &&
          (a.sl_late[rowbase + a.m.member_off[g]] & kSlHist))
        hist = 1;
    }
    uint32_t c = v.x, e = v.y;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t c2 = __shfl_up_sync(FULL, c, o), e2 = __shfl_up_sync(FULL, e, o);
      if (lane >= o) {
        c += c2;
        e += e2;
      }
    }
    if (lane == 31) {
      wc[warp] = c;
      we[warp] = e;
    }
    __syncthreads();
    uint32_t bc = run_c, be = run_e, tc = 0, te = 0;
    for (int q = 0; q < nw; ++q) {
      if (q < warp) {
        bc += wc[q];
        be += we[q];
      }
      tc += wc[q];
      te += we[q];
    }
    if (i < naff) cnt[i] = make_uint2(bc + c - v.x, be + e - v.y);
    __syncthreads();
    if (threadIdx.x == 0) {
      run_c += tc;
      run_e += te;
    }
    __syncthreads();
  }
  if (hist) s_hist = 1;
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t C = run_c, CE = run_e;
  StragState S;
  memset(&S, 0, sizeof(S));
  S.any_history = s_hist;
  TripOut o;
  memset(&o, 0, sizeof(o));
  o.n_aff = naff;
  if (C == 0) {
    o.verdict = s_hist ? CSG_VERDICT_NO_STRAGGLER : CSG_VERDICT_INSUFFICIENT_HISTORY;
    o.scanned = 2 * a.N;
    a.out[j] = o;
    a.state[j] = S;
    return;
  }
  bool ok1, ok2, ok3, ok4;
  S.cap_cand = C;
  S.cap_cev = CE;
  S.cand_base = pool_alloc(a.pools.used, P_CAND, C, a.pools.cand_cap, a.err, DEV_ERR_POOL, &ok1);
  S.cev_base = pool_alloc(a.pools.used, P_CEV, CE, a.pools.cev_cap, a.err, DEV_ERR_POOL, &ok2);
  S.sus_base = pool_alloc(a.pools.used, P_SUS, 3ull * C, a.pools.sus_cap, a.err, DEV_ERR_POOL,
                          &ok3);
  S.exo_base = S.sus_base + C;
  S.ev_base = pool_alloc(a.pools.used, P_EV, CE, a.pools.ev_cap, a.err, DEV_ERR_POOL, &ok4);
  if (!(ok1 && ok2 && ok3 && ok4)) {
    S.C = 0;  // the host retries with larger pools (DEV_ERR_POOL)
    a.state[j] = S;
    return;
  }
  S.C = static_cast<int32_t>(C);
  S.cev_used = CE;
  a.state[j] = S;
}

__device__ inline void sl_cev(const DecideArgs& a, const StragState& S, uint32_t at,
                              int32_t rank, int32_t ch, double tms, int64_t op) {
  csg_evidence e;
  e.rank = rank;
  e.channel = ch;
  e.time_ms = tms;
  e.op_seq = op;
  a.pools.cev[S.cev_base + at] = e;
}

__global__ void __launch_bounds__(kSlWarps * 32) k_sl_emit(DecideArgs a, int32_t Js) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int32_t G = a.m.n_groups;
  const uint64_t w = blockIdx.x * (uint64_t)kSlWarps + wib;
  if (w >= static_cast<uint64_t>(Js) * G) return;
  const int32_t js = static_cast<int32_t>(w / G), i = static_cast<int32_t>(w % G);
  const int32_t j = a.strag_trip[js];
  if (i >= a.n_aff[j] || a.m.opn == 0) return;
  const StragState S = a.state[j];
  if (S.C <= 0) return;
  const int32_t g = a.aff[static_cast<uint64_t>(j) * G + i];
  const uint32_t mo = a.m.member_off[g];
  const int32_t m = static_cast<int32_t>(a.m.member_off[g + 1] - mo);
  const uint64_t rowbase = static_cast<uint64_t>(js) * a.M;
  if (m < 2 || !(a.sl_late[rowbase + mo] & kSlHist)) return;
  const uint2 off = a.sl_cnt[static_cast<uint64_t>(js) * G + i];
  const uint64_t gidx = static_cast<uint64_t>(js) * G + g;
  const int32_t k = a.k, opn = a.m.opn;
  const int64_t gfo = a.m.group_first_op[g];
  const int64_t wlo = a.gi_last[gidx * k], whi = a.gi_last[gidx * k + k - 1];
  Cand* cands = a.pools.cand + S.cand_base;
  // (1) late members in member order
  uint32_t nl = 0;
  for (int b0 = 0; b0 < m; b0 += 32) {
    const int x = b0 + lane;
    const uint8_t v = x < m ? a.sl_late[rowbase + mo + x] : 0;
    const bool lt = (v & 3) != 0;
    const unsigned mm = __ballot_sync(FULL, lt);
    if (lt) {
      const uint32_t pos = nl + __popc(mm & ((1u << lane) - 1u));
      const int32_t r = a.m.members[mo + x];
      const uint64_t cell = (rowbase + a.m.member_slot[mo + x]) * a.n_it;
      Cand c;
      memset(&c, 0, sizeof(c));
      c.rank = r;
      c.cat = (v & 1) ? CSG_RC_STRAGGLER_LATE_START : CSG_RC_STRAGGLER_LATE_END;
      c.side = CSG_SIDE_LOCAL;
      c.group = g;
      c.op = whi * opn + gfo;
      c.onset = dkey_inv(a.tbl_s[cell + (wlo - a.it_min)]);
      c.it_lo = wlo;
      c.it_hi = whi;
      c.ev_off = off.y + pos * k;
      c.ev_n = k;
      for (int q = 0; q < k; ++q) {
        const int64_t it = a.gi_last[gidx * k + q];
        sl_cev(a, S, c.ev_off + q, r, -1, dkey_inv(a.tbl_s[cell + (it - a.it_min)]),
               it * opn + gfo);
      }
      cands[off.x + pos] = c;
    }
    nl += __popc(mm);
  }
  // (2) FlowSkewed then (3) FlowIncomplete, each in ascending rank order
  uint32_t base_c = off.x + nl, base_e = off.y + nl * static_cast<uint32_t>(k);
  for (int pass = 0; pass < 2; ++pass) {
    const uint8_t want = pass == 0 ? kSlSkew : kSlInc;
    uint32_t nt = 0;
    for (int b0 = 0; b0 < m; b0 += 32) {
      const int x = b0 + lane;
      const bool is = x < m && (a.sl_late[rowbase + mo + x] & want);
      if (is) {
        const int32_t r = a.m.members[mo + x];
        uint32_t pos = 0;  // rank-order position among this pass's findings
        for (int y = 0; y < m; ++y)
          if ((a.sl_late[rowbase + mo + y] & want) && a.m.members[mo + y] < r) ++pos;
        const FlowSum f = a.fs[rowbase + mo + x];
        Cand c;
        memset(&c, 0, sizeof(c));
        c.rank = r;
        c.side = CSG_SIDE_LOCAL;
        c.group = g;
        c.it_lo = 0;
        c.it_hi = -1;
        c.ev_off = base_e + pos;
        c.ev_n = 1;
        if (pass == 0) {
          c.cat = CSG_RC_FLOW_SKEWED;
          c.op = f.skew_op;
          c.onset = f.skew_start;
          sl_cev(a, S, c.ev_off, r, f.skew_chan, f.skew_end, f.skew_op);
        } else {
          c.cat = CSG_RC_FLOW_INCOMPLETE;
          c.op = f.inc_op;
          c.onset = a.trip_t[j];
          sl_cev(a, S, c.ev_off, r, f.inc_chan, a.trip_t[j], f.inc_op);
        }
        cands[base_c + pos] = c;
      }
      nt += __popc(__ballot_sync(FULL, is));
    }
    base_c += nt;
    base_e += nt;
  }
}

// ---------------------------------------------------------------------------
// Sorted self-evidence path. self_faulted (rca.cpp:821-848) asks, for a
// candidate rank r and each op o of its iteration window that r completed,
// whether r's longest duration of o exceeds skew x the lower median of every
// other rank's durations of o (ts <= t). The sibling multiset is the op's
// whole op-index segment minus r's own entries, so with the segment sorted
// once (k_opsort) the median is a lookup: element q = (m - k_r - 1) / 2 of
// the segment with r's k_r values skipped lies in [q, q + k_r] and follows
// from one window load and a merge against r's sorted values. A warp per
// candidate (k_sf_fast) does that for every op of the window; candidates it
// cannot decide this way (sharded store, a segment with entries after t or
// too long to sort, more than 32 completions of one op, a cohort the table
// does not hold) are left to k_self_faulted (Cand::pad = 2).
// ---------------------------------------------------------------------------
struct SfPlan {
  unsigned long long k0, k1;  // op keys covered by the candidates' windows
  unsigned long long total;   // straggler candidates in the batch
  int32_t any;
  int32_t pad;
  unsigned long long cstart[1];  // [J + 1] flattened candidate offsets
};

constexpr int kOpSortWarpCap = 512;    // entries a warp sorts in shared memory
constexpr int kOpSortBlockCap = 8192;  // entries a block sorts (64 KB)
constexpr int kSfWarps = 4;
constexpr int kSfPend = 8;

__global__ void __launch_bounds__(1024) k_sf_prep(DecideArgs a) {
  SfPlan* pl = a.plan;
  __shared__ long long s_lo[32], s_hi[32];
  long long lo = LLONG_MAX, hi = LLONG_MIN;
  for (int32_t j = 0; j < a.J; ++j) {
    if (a.trip_kind[j] == CSG_TRIGGER_FAILURE) continue;
    const StragState S = a.state[j];
    if (S.C <= 0) continue;
    const Cand* cands = a.pools.cand + S.cand_base;
    for (int x = threadIdx.x; x < S.C; x += blockDim.x) {
      const Cand& c = cands[x];
      if (c.it_hi < c.it_lo) continue;
      lo = min(lo, static_cast<long long>(c.it_lo));
      hi = max(hi, static_cast<long long>(c.it_hi));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(FULL, lo, o));
    hi = max(hi, __shfl_xor_sync(FULL, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    s_lo[threadIdx.x >> 5] = lo;
    s_hi[threadIdx.x >> 5] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
      lo = min(lo, s_lo[w]);
      hi = max(hi, s_hi[w]);
    }
    unsigned long long tot = 0;
    for (int32_t j = 0; j < a.J; ++j) {
      pl->cstart[j] = tot;
      if (a.trip_kind[j] != CSG_TRIGGER_FAILURE && a.state[j].C > 0) tot += a.state[j].C;
    }
    pl->cstart[a.J] = tot;
    pl->total = tot;
    pl->any = 0;
    if (lo <= hi && a.m.opn > 0) {
      int64_t olo, ohi, x0, x1;
      iter_ops(lo, a.m.opn, olo, x1);
      iter_ops(hi, a.m.opn, x0, ohi);
      // keys of ops inside the store's op range
      const long long mo = a.min_op;
      const long long k0 = max(0ll, static_cast<long long>(olo) - mo);
      const long long k1 = min(static_cast<long long>(ohi), static_cast<long long>(a.max_op)) - mo;
      if (k1 >= k0) {
        pl->k0 = static_cast<unsigned long long>(k0);
        pl->k1 = static_cast<unsigned long long>(k1);
        pl->any = 1;
      }
    }
  }
}

// Per op key in the plan's range: sort the op-index segment's entries by
// duration (warp per op up to kOpSortWarpCap entries; longer segments go to
// k_opsort_large) into sdur / sts / srank, and record the segment's latest
// timestamp.
__device__ void warp_bitonic_kv(unsigned long long* v, uint16_t* ix, uint32_t P) {
  const int lane = threadIdx.x & 31;
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
      for (uint32_t i = lane; i < P; i += 32) {
        const uint32_t l = i ^ jj;
        if (l > i) {
          const unsigned long long x = v[i], y = v[l];
          if ((x > y) == ((i & k) == 0)) {
            v[i] = y;
            v[l] = x;
            const uint16_t t = ix[i];
            ix[i] = ix[l];
            ix[l] = t;
          }
        }
      }
      __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(256) k_opsort(DecideArgs a, unsigned* __restrict__ large,
                                                unsigned* __restrict__ n_large,
                                                uint32_t large_cap) {
  __shared__ unsigned long long buf[8][kOpSortWarpCap];
  __shared__ uint16_t ibuf[8][kOpSortWarpCap];
  const SfPlan* pl = a.plan;
  if (!pl->any) return;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned long long* v = buf[wib];
  uint16_t* ix = ibuf[wib];
  const unsigned long long k0 = pl->k0, k1 = pl->k1;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t kk = k0 + (blockIdx.x * (uint64_t)(blockDim.x >> 5) + wib); kk <= k1; kk += nw) {
    const uint32_t sb = a.opoff[kk], se = a.opoff[kk + 1];
    const uint32_t m = se - sb;
    if (m == 0) continue;
    if (m > kOpSortWarpCap) {
      if (lane == 0) {
        const unsigned at = atomicAdd(n_large, 1u);
        if (at < large_cap) large[at] = static_cast<unsigned>(kk - k0);
        else a.opmax[kk] = __longlong_as_double(0x7FF8000000000000ll);  // unsorted
      }
      continue;
    }
    uint32_t P = 32;
    while (P < m) P <<= 1;
    double mx = -INFINITY;
    for (uint32_t i = lane; i < P; i += 32) {
      if (i < m) {
        v[i] = dkey(a.op_dur[sb + i]);
        mx = fmax(mx, a.op_ts[sb + i]);
      } else {
        v[i] = ~0ull;
      }
      ix[i] = static_cast<uint16_t>(i);
    }
    __syncwarp();
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
    warp_bitonic_kv(v, ix, P);
    for (uint32_t i = lane; i < m; i += 32) {
      a.sdur[sb + i] = v[i];
      a.sts[sb + i] = a.op_ts[sb + ix[i]];
      a.srank[sb + i] = a.oprank[sb + ix[i]];
    }
    if (lane == 0) a.opmax[kk] = mx;
    __syncwarp();
  }
}

__global__ void __launch_bounds__(1024) k_opsort_large(DecideArgs a,
                                                       const unsigned* __restrict__ large,
                                                       const unsigned* __restrict__ n_large,
                                                       uint32_t large_cap) {
  extern __shared__ __align__(16) unsigned long long sv[];  // [kOpSortBlockCap] + u16 idx
  uint16_t* si = reinterpret_cast<uint16_t*>(sv + kOpSortBlockCap);
  __shared__ double s_mx[32];
  const SfPlan* pl = a.plan;
  if (!pl->any) return;
  const uint32_t nl = min(*n_large, large_cap);
  for (uint32_t w = blockIdx.x; w < nl; w += gridDim.x) {
    const unsigned long long kk = pl->k0 + large[w];
    const uint32_t sb = a.opoff[kk], se = a.opoff[kk + 1];
    const uint32_t m = se - sb;
    if (m > kOpSortBlockCap) {
      if (threadIdx.x == 0) a.opmax[kk] = __longlong_as_double(0x7FF8000000000000ll);
      continue;
    }
    uint32_t P = 32;
    while (P < m) P <<= 1;
    double mx = -INFINITY;
    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
      if (i < m) {
        sv[i] = dkey(a.op_dur[sb + i]);
        mx = fmax(mx, a.op_ts[sb + i]);
      } else {
        sv[i] = ~0ull;
      }
      si[i] = static_cast<uint16_t>(i);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
    if ((threadIdx.x & 31) == 0) s_mx[threadIdx.x >> 5] = mx;
    __syncthreads();
    for (uint32_t k = 2; k <= P; k <<= 1) {
      for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
        for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
          const uint32_t l = i ^ jj;
          if (l > i) {
            const unsigned long long x = sv[i], y = sv[l];
            if ((x > y) == ((i & k) == 0)) {
              sv[i] = y;
              sv[l] = x;
              const uint16_t t = si[i];
              si[i] = si[l];
              si[l] = t;
            }
          }
        }
        __syncthreads();
      }
    }
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
      a.sdur[sb + i] = sv[i];
      a.sts[sb + i] = a.op_ts[sb + si[i]];
      a.srank[sb + i] = a.oprank[sb + si[i]];
    }
    if (threadIdx.x == 0) {
      double t = -INFINITY;
      for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) t = fmax(t, s_mx[q]);
      a.opmax[kk] = t;
    }
    __syncthreads();
  }
}

// Sharded stores: every shard decided its own ranks' candidates (0 for the
// others); the verdicts travel as one byte per flattened candidate through a
// MAX all-reduce (dir 0: pack, dir 1: unpack).
__global__ void k_sf_pads(DecideArgs a, uint8_t* __restrict__ flat, int dir) {
  const SfPlan* pl = a.plan;
  const unsigned long long total = pl->total;
  for (unsigned long long w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < total;
       w += (uint64_t)gridDim.x * blockDim.x) {
    int32_t lo = 0, hi = a.J;
    while (hi - lo > 1) {
      const int32_t mid = (lo + hi) >> 1;
      if (pl->cstart[mid] <= w) lo = mid; else hi = mid;
    }
    Cand& c = a.pools.cand[a.state[lo].cand_base + (w - pl->cstart[lo])];
    if (dir == 0) flat[w] = c.pad;
    else c.pad = flat[w];
  }
}

// Warp-collective ascending sort of one u64 key per lane.
__device__ inline unsigned long long warp_sort32(unsigned long long v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      const unsigned long long o = __shfl_xor_sync(FULL, v, jj);
      const bool up = (lane & k) == 0;
      const bool lower = (lane & jj) == 0;
      v = (lower == up) ? min(v, o) : max(v, o);
    }
  }
  return v;
}

__global__ void __launch_bounds__(kSfWarps * 32) k_sf_fast(DecideArgs a,
                                                           unsigned* __restrict__ why,
                                                           int pass) {
  const SfPlan* pl = a.plan;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const unsigned long long total = pl->total;
  const uint64_t nw = (uint64_t)gridDim.x * kSfWarps;
  const int32_t opn = a.m.opn;
  for (unsigned long long w = blockIdx.x * (uint64_t)kSfWarps + wib; w < total; w += nw) {
    // trip of flattened candidate w
    int32_t lo = 0, hi = a.J;  // cstart[lo] <= w < cstart[hi]
    while (hi - lo > 1) {
      const int32_t mid = (lo + hi) >> 1;
      if (pl->cstart[mid] <= w) lo = mid; else hi = mid;
    }
    const int32_t j = lo;
    Cand* cands = a.pools.cand + a.state[j].cand_base;
    const uint32_t x = static_cast<uint32_t>(w - pl->cstart[j]);
    const Cand c = cands[x];
    if (pass == 1 && c.pad != 3) continue;  // second pass: waited for cohorts only
    // 0 not self-faulted, 1 self-faulted, 2 deferred to k_self_faulted,
    // 3 needs a cohort median (claimed for k_cohorts_lazy; second pass)
    int verdict = 0;
    int reason = 0;
    const int32_t r = c.rank;
    const double t = a.trip_t[j];
    if (c.it_hi < c.it_lo) {
      verdict = 1;
    } else if (a.f.n == 0 || opn <= 0) {
      verdict = 2;
      reason = 1;
    } else if (a.sharded && !(r >= 0 && r < a.s.R && a.s.rank_off[r + 1] > a.s.rank_off[r])) {
      verdict = 0;  // another shard's rank: its owner decides (k_sf_pads MAX-combines)
    } else if (r >= 0 && r < a.s.R) {
      const uint32_t b = a.s.rank_off[r], e = a.s.rank_off[r + 1];
      const bool uns = a.f.unsorted[r] != 0;
      auto opat = [&](uint32_t i) { return a.s.op[a.f.at(uns, i)]; };
      int64_t olo, ohi, x0, x1;
      iter_ops(c.it_lo, opn, olo, x1);
      iter_ops(c.it_hi, opn, x0, ohi);
      // the window's ops in ascending order: each op's run of the flow
      // order, found by a partition point from the run start. The second
      // pass revisits only the ops whose cohort the first pass waited for
      // (up to kSfPend of them, listed by the first pass).
      const uint32_t np = pass == 1 ? a.pend_n[w] : 0u;
      const bool listed = pass == 1 && np <= static_cast<uint32_t>(kSfPend);
      uint32_t fo = b, fe = e;
      if (!listed) {
        fo = warp_partition_point(b, e, [&](uint32_t i) { return opat(i) >= olo; });
        fe = warp_partition_point(fo, e, [&](uint32_t i) { return opat(i) > ohi; });
      }
      bool pending = false;
      uint32_t npend = 0, pi = 0;
      for (uint32_t p0 = fo; verdict == 0;) {
        int64_t o;
        uint32_t p1;
        if (listed) {
          if (pi >= np) break;
          o = a.pend_ops[w * kSfPend + pi++];
          p0 = warp_partition_point(b, e, [&](uint32_t i) { return opat(i) >= o; });
          p1 = warp_partition_point(p0, e, [&](uint32_t i) { return opat(i) > o; });
        } else {
          if (p0 >= fe) break;
          o = opat(p0);
          p1 = warp_partition_point(p0, fe, [&](uint32_t i) { return opat(i) > o; });
        }
        // r's completions of o (non-Recv, ts <= t): value k of the run on lane k
        int kr = 0;
        unsigned long long mv = 0;
        for (uint32_t base = p0; base < p1 && kr <= 32; base += 32) {
          const uint32_t i = base + lane;
          bool ok = false;
          unsigned long long dk = 0;
          if (i < p1) {
            const uint32_t p = a.f.at(uns, i);
            const uint8_t ko = a.s.ko[p];
            ok = ko_kind(ko) == CSG_KIND_COMPLETION && ko_opname(ko) != CSG_OP_RECV &&
                 a.s.ts[p] <= t;
            if (ok) dk = dkey(a.s.ts[p] - as_double(a.s.pa[p]));
          }
          const unsigned mm = __ballot_sync(FULL, ok);
          for (unsigned q = mm; q; q &= q - 1) {
            const int src = __ffs(q) - 1;
            const unsigned long long v = __shfl_sync(FULL, dk, src);
            if (lane == kr + __popc(mm & ((1u << src) - 1u))) mv = v;
          }
          kr += __popc(mm);
        }
        p0 = p1;
        if (kr == 0) continue;
        if (kr > 32) {
          verdict = 2;
          reason = 2;
          break;
        }
        unsigned long long mine = lane < kr ? mv : 0ull;
#pragma unroll
        for (int s2 = 16; s2; s2 >>= 1) mine = max(mine, __shfl_xor_sync(FULL, mine, s2));
        const uint64_t key = static_cast<uint64_t>(o - a.min_op);
        const uint32_t sb = a.opoff[key], se = a.opoff[key + 1];
        const uint32_t m = se - sb;
        const double omx = a.opmax[key];
        if (omx != omx || m < static_cast<uint32_t>(kr)) {
          verdict = 2;
          reason = 3;
          break;
        }
        // entries after t: siblings = the sorted entries with ts <= t of
        // other ranks; order statistic by two counting passes
        const bool filtered = !(omx <= t);
        uint32_t nsib = m - kr;
        if (filtered) {
          uint32_t cnt = 0;
          for (uint32_t base = 0; base < m; base += 32) {
            const uint32_t i = base + lane;
            const bool keep = i < m && a.sts[sb + i] <= t && a.srank[sb + i] != r;
            cnt += __popc(__ballot_sync(FULL, keep));
          }
          nsib = cnt;
        }
        double med;
        if (nsib == 0) {
          // no siblings: the (op name, iteration) cohort of k_cohorts
          const int64_t it = iter_of(o, opn);
          const uint8_t nm = a.m.op_name[static_cast<uint64_t>(o % opn)];
          const unsigned long long ckey =
              (static_cast<unsigned long long>(j) << 44) ^
              (static_cast<unsigned long long>(nm) << 36) ^
              (static_cast<unsigned long long>(it) & ((1ull << 36) - 1));
          // 1 published, 2 claimed / pending (first pass only: the second
          // pass and k_self_faulted must not leave claims nobody computes)
          int found = 0;
          double cv = 0;
          if (lane == 0 && a.coh_cap) {
            const uint32_t mask = a.coh_cap - 1;
            uint32_t h = static_cast<uint32_t>((ckey * 0x9E3779B97F4A7C15ull) >> 40) & mask;
            for (uint32_t probe = 0; probe < a.coh_cap; ++probe, h = (h + 1) & mask) {
              const unsigned long long kk2 =
                  pass == 0 ? atomicCAS(a.coh_key + h, ~0ull, ckey) : a.coh_key[h];
              if (kk2 == ~0ull) {
                if (pass == 0) {  // claimed: k_cohorts_lazy computes it
                  a.coh_meta[h] = make_longlong2(it, (static_cast<long long>(j) << 8) | nm);
                  found = 2;
                }
                break;
              }
              if (kk2 == ckey) {
                if (*reinterpret_cast<volatile unsigned*>(a.coh_state + h) == 2u) {
                  found = 1;
                  cv = a.coh_val[h];
                } else {
                  found = 2;
                }
                break;
              }
            }
          }
          found = __shfl_sync(FULL, found, 0);
          if (found == 2 && pass == 0) {  // decide the other ops, then wait for it
            pending = true;
            if (npend < static_cast<uint32_t>(kSfPend) && lane == 0)
              a.pend_ops[w * kSfPend + npend] = o;
            ++npend;
            continue;
          }
          if (found != 1) {
            verdict = 2;
            reason = 5;
            break;
          }
          med = __shfl_sync(FULL, cv, 0);
        } else if (filtered) {
          const uint32_t q = (nsib - 1) / 2;
          uint32_t cnt = 0, at = 0;
          for (uint32_t base = 0; base < m; base += 32) {
            const uint32_t i = base + lane;
            const bool keep = i < m && a.sts[sb + i] <= t && a.srank[sb + i] != r;
            const unsigned mm = __ballot_sync(FULL, keep);
            const uint32_t c2 = __popc(mm);
            if (cnt + c2 > q) {  // the q-th kept entry is in this chunk
              unsigned x2 = mm;
              for (uint32_t z = cnt; z < q; ++z) x2 &= x2 - 1;
              at = base + __ffs(x2) - 1;
              break;
            }
            cnt += c2;
          }
          med = dkey_inv(a.sdur[sb + at]);
        } else {
          // element q of the sorted segment with r's kr values skipped
          const uint32_t qm = (m - kr - 1) / 2;
          const unsigned long long sorted_mine = warp_sort32(lane < kr ? mv : ~0ull);
          const unsigned long long win = lane <= kr ? a.sdur[sb + qm + lane] : ~0ull;
          int pos = 0;
          for (int i = 0; i < kr; ++i) {
            const unsigned long long vi = __shfl_sync(FULL, sorted_mine, i);
            const unsigned long long lp = __shfl_sync(FULL, win, pos);
            if (vi <= lp) ++pos; else break;
          }
          med = dkey_inv(__shfl_sync(FULL, win, pos));
        }
        if (med > 0 && dkey_inv(mine) > __dmul_rn(a.skew, med)) verdict = 1;
      }
      if (verdict == 0 && pending) {
        verdict = 3;
        if (lane == 0) a.pend_n[w] = static_cast<uint8_t>(min(npend, 255u));
      }
    }
    if (lane == 0) {
      cands[x].pad = static_cast<uint8_t>(verdict);
      if (why) atomicAdd(why + reason, 1u);
    }
    __syncwarp();
  }
}

}  // namespace
}  // namespace csg

namespace csg {

namespace {

// Host vector -> device buffer through the buffer's pinned staging area
// (a truly asynchronous copy; the staging area is only rewritten by the
// next call, after the stream has been synchronised in between).
template <typename T>
T* upload(DevBuf& b, const std::vector<T>& v, cudaStream_t st) {
  b.ensure(v.size() * sizeof(T) + sizeof(T));
  if (!v.empty()) {
    b.stage.ensure(v.size() * sizeof(T));
    std::memcpy(b.stage.p, v.data(), v.size() * sizeof(T));
    CSG_CUDA(cudaMemcpyAsync(b.p, b.stage.p, v.size() * sizeof(T),
                             cudaMemcpyHostToDevice, st));
  }
  return b.as<T>();
}

void validate_analysis(const csg_analysis_config& c) {
  // AnalysisConfig::validate (proj/src/rca.cpp:63-71)
  if (!(c.straggler_threshold_ms > 0))
    throw Error(CSG_ERR_CONFIG, "analysis: straggler_threshold_ms must be > 0");
  if (c.consecutive_iterations_k < 1)
    throw Error(CSG_ERR_CONFIG,
                "analysis: consecutive_iterations_k must be >= 1");
  if (!(c.delta_ms > 0))
    throw Error(CSG_ERR_CONFIG, "analysis: delta_ms must be > 0");
  if (!(c.flow_skew_factor > 1))
    throw Error(CSG_ERR_CONFIG, "analysis: flow_skew_factor must be > 1");
}

}  // namespace

void rca_batch(csg_store* s, const csg_model* m, const csg_analysis_config& cfg,
               const csg_trigger_event* trips, int32_t J, bool affected_only,
               RcaResult& out) {
  out = RcaResult();
  out.G = m->n_groups;
  if (J <= 0) return;
  if (!affected_only) validate_analysis(cfg);
  if (cfg.consecutive_iterations_k > kMaxK)
    throw Error(CSG_ERR_RUNTIME,
                "engine: consecutive_iterations_k > 64 is not supported");
  tl_mark("rca_batch entry");
  store_build_index(s);
  store_resolve_max_seg(s);
  csg_ctx* c = s->ctx;
  cudaStream_t st = c->stream;
  const StoreView sv = s->view();
  const ModelView mv = m->view();
  const int32_t R = s->R;
  const int32_t nch = std::max(s->nch, 1);
  const int32_t G = m->n_groups;
  const int32_t opn = m->opn;
  const int32_t k = cfg.consecutive_iterations_k;
  const uint32_t M = G ? m->h_member_off[G] : 0;

  std::vector<double> h_t(J);
  std::vector<int32_t> h_kind(J), h_rank(J), h_js(J, -1), h_strag;
  for (int32_t j = 0; j < J; ++j) {
    h_t[j] = trips[j].time_ms;
    h_kind[j] = trips[j].kind;
    h_rank[j] = trips[j].suspect_rank;
    if (trips[j].kind == CSG_TRIGGER_STRAGGLER) {
      h_js[j] = static_cast<int32_t>(h_strag.size());
      h_strag.push_back(j);
    }
  }
  const int32_t Js = static_cast<int32_t>(h_strag.size());
  // the five per-trip arrays go up in one pinned copy (each API call costs
  // microseconds of host time on the critical path)
  DevBuf& targ = c->buf("rca.trip_args");
  const size_t nb_t = static_cast<size_t>(J) * 8, nb_i = static_cast<size_t>(J) * 4;
  const size_t o_kind = nb_t, o_rank = o_kind + nb_i, o_js = o_rank + nb_i,
               o_strag = o_js + nb_i, tbytes = o_strag + static_cast<size_t>(Js) * 4 + 8;
  targ.ensure(tbytes);
  targ.stage.ensure(tbytes);
  {
    unsigned char* h = targ.stage.as<unsigned char>();
    std::memcpy(h, h_t.data(), nb_t);
    std::memcpy(h + o_kind, h_kind.data(), nb_i);
    std::memcpy(h + o_rank, h_rank.data(), nb_i);
    std::memcpy(h + o_js, h_js.data(), nb_i);
    if (Js) std::memcpy(h + o_strag, h_strag.data(), static_cast<size_t>(Js) * 4);
    CSG_CUDA(cudaMemcpyAsync(targ.p, h, tbytes, cudaMemcpyHostToDevice, st));
  }
  tl_mark("rca trip args uploaded");
  unsigned char* tb = targ.as<unsigned char>();
  const double* dt = reinterpret_cast<const double*>(tb);
  const int32_t* dkind = reinterpret_cast<const int32_t*>(tb + o_kind);
  const int32_t* drank = reinterpret_cast<const int32_t*>(tb + o_rank);
  const int32_t* djs = reinterpret_cast<const int32_t*>(tb + o_js);
  const int32_t* dstrag = reinterpret_cast<const int32_t*>(tb + o_strag);

  // K1: per (trip, rank) prefix summaries
  DevBuf& rs = c->buf("rca.rs");
  DevBuf& chan_key = c->buf("rca.chan_key");
  rs.ensure(static_cast<size_t>(J) * std::max(R, 1) * sizeof(RankSum));
  chan_key.ensure(static_cast<size_t>(J) * std::max(R, 1) * nch * 8);
  // Sharded: only this shard's ranks are summarised; the other entries are
  // zero so a sum all-reduce assembles the global tables.
  const bool sharded = comm_active(c);
  const int32_t r0 = sharded ? std::max(s->own_lo, 0) : 0;
  const int32_t nr = sharded ? std::max(0, std::min(s->own_hi, R - 1) - r0 + 1) : R;
  if (sharded) {
    CSG_CUDA(cudaMemsetAsync(rs.p, 0, static_cast<size_t>(J) * std::max(R, 1) * sizeof(RankSum),
                             st));
    CSG_CUDA(cudaMemsetAsync(chan_key.p, 0,
                             static_cast<size_t>(J) * std::max(R, 1) * nch * 8, st));
  }
  if (R > 0 && nr > 0) {
    int wpb = 32768 / (nch * 4);
    wpb = std::max(1, std::min(8, wpb));
    const uint64_t warps = static_cast<uint64_t>(nr) * J;
    static const bool no_fi = std::getenv("CSG_DISABLE_FLOW_INDEX") != nullptr;
    if (!no_fi && store_build_flow_index(s)) {
      ProfScope ps_(c->lc, "k_rank_summary_fi", st);
      launch_pdl(k_rank_summary_fi, dim3(static_cast<unsigned>((warps + wpb - 1) / wpb)), dim3(wpb * 32), wpb * nch * 4, st, sv, s->flow_view(), J, dt, cfg.delta_ms,
                                               rs.as<RankSum>(),
                                               chan_key.as<unsigned long long>(), nch, r0, nr);
    } else {
      ProfScope ps_(c->lc, "k_rank_summary", st);
      k_rank_summary<<<static_cast<unsigned>((warps + wpb - 1) / wpb), wpb * 32,
                       wpb * nch * 4, st>>>(sv, J, dt, cfg.delta_ms,
                                            rs.as<RankSum>(),
                                            chan_key.as<unsigned long long>(), nch, r0, nr);
    }
  }
  // sharded: every rank's summary lives on exactly one shard (zeros
  // elsewhere), so a sum all-reduce assembles the global tables
  comm_group_start(c);
  comm_allreduce(c, rs.p, static_cast<size_t>(J) * std::max(R, 1) * sizeof(RankSum) / 8,
                 ncclUint64, ncclSum);
  comm_allreduce(c, chan_key.p, static_cast<size_t>(J) * std::max(R, 1) * nch,
                 ncclUint64, ncclSum);
  comm_group_end(c);
  // K1b: ring-successor progress per membership slot
  DevBuf& slot_group = c->buf("rca.slot_group");
  DevBuf& succ = c->buf("rca.succ");
  DevBuf& succ_key = c->buf("rca.succ_key");
  if (c->slot_group_uid != m->uid) {  // group of every membership slot
    std::vector<uint32_t> h_sg(std::max<uint32_t>(M, 1));
    for (int32_t g = 0; g < G; ++g)
      for (uint32_t q = m->h_member_off[g]; q < m->h_member_off[g + 1]; ++q)
        h_sg[q] = static_cast<uint32_t>(g);
    upload(slot_group, h_sg, st);
    c->slot_group_uid = m->uid;
  }
  succ.ensure(static_cast<size_t>(J) * std::max<uint32_t>(M, 1) * sizeof(SuccProg));
  succ_key.ensure(static_cast<size_t>(J) * std::max<uint32_t>(M, 1) * nch * 8);
  if (!affected_only && M > 0) {
    // sharded: the membership slots of owned ranks (contiguous in the
    // model's rank -> slot CSR), zeros elsewhere
    const uint32_t* slots = nullptr;
    uint32_t E = M;
    if (sharded) {
      CSG_CUDA(cudaMemsetAsync(succ.p, 0, static_cast<size_t>(J) * M * sizeof(SuccProg), st));
      CSG_CUDA(cudaMemsetAsync(succ_key.p, 0, static_cast<size_t>(J) * M * nch * 8, st));
      const int32_t RS = m->rank_space;
      const int32_t lo = std::min(r0, RS), hi = std::min(r0 + nr, RS);
      const uint32_t e0 = m->h_rg_off[lo], e1 = m->h_rg_off[hi];
      slots = m->rg_slot.as<uint32_t>() + e0;
      E = e1 - e0;
    }
    int wpb = 32768 / (nch * 4);
    wpb = std::max(1, std::min(8, wpb));
    const uint64_t warps = static_cast<uint64_t>(E) * J;
    if (warps) {
      ProfScope ps_(c->lc, "k_succ_prog", st);
      launch_pdl(k_succ_prog, dim3(static_cast<unsigned>((warps + wpb - 1) / wpb)), dim3(wpb * 32), wpb * nch * 4, st, sv, s->flow_view(), mv, J, M,
                                         slot_group.as<uint32_t>(), rs.as<RankSum>(),
                                         succ.as<SuccProg>(),
                                         succ_key.as<unsigned long long>(), nch, slots, E,
                                         dkind);
    }
  }
  if (!affected_only && M > 0) {
    comm_group_start(c);
    comm_allreduce(c, succ.p, static_cast<size_t>(J) * M * sizeof(SuccProg) / 8,
                   ncclUint64, ncclSum);
    comm_allreduce(c, succ_key.p, static_cast<size_t>(J) * M * nch, ncclUint64, ncclSum);
    comm_group_end(c);
  }
  // K2/K3: straggler iteration tables
  DevBuf& tbl_s = c->buf("rca.tbl_s");
  DevBuf& tbl_e = c->buf("rca.tbl_e");
  DevBuf& gi = c->buf("rca.gi");
  DevBuf& gi_last = c->buf("rca.gi_last");
  int64_t it_min = 0;
  int32_t n_it = 1;
  gi.ensure(static_cast<size_t>(std::max(Js, 1)) * std::max(G, 1) * sizeof(GroupIter));
  gi_last.ensure(static_cast<size_t>(std::max(Js, 1)) * std::max(G, 1) * k * 8);
  tbl_s.ensure(8);
  tbl_e.ensure(8);
  if (Js > 0) {
    CSG_CUDA(cudaMemsetAsync(gi.p, 0, gi.bytes, st));
    if (opn > 0 && M > 0) {
      it_min = iter_of(s->min_op, opn);
      const int64_t it_max = iter_of(s->max_op, opn);
      const int64_t span = s->n ? it_max - it_min + 1 : 1;
      const double bytes = 16.0 * Js * M * static_cast<double>(span);
      if (span > (1ll << 30) || bytes > 24e9)
        throw Error(CSG_ERR_RUNTIME,
                    "engine: straggler iteration tables exceed the device budget");
      n_it = static_cast<int32_t>(span);
      const size_t cells = static_cast<size_t>(Js) * M * n_it;
      tbl_s.ensure(cells * 8);
      tbl_e.ensure(cells * 8);
      CSG_CUDA(cudaMemsetAsync(tbl_s.p, 0xff, cells * 8, st));
      CSG_CUDA(cudaMemsetAsync(tbl_e.p, 0, cells * 8, st));
      // straggler trips in time order (every run_detection batch): one pass
      // over the store, then a running min/max over the trips' tables
      bool ordered = true;
      for (int32_t x = 1; x < Js; ++x)
        ordered = ordered && h_t[h_strag[x]] >= h_t[h_strag[x - 1]];
      static const bool inc_off = std::getenv("CSG_ITER_PER_TRIP") != nullptr;
      DevBuf& pc = c->buf("rca.iter_pc");
      const uint64_t per = static_cast<uint64_t>(M) * n_it;
      const uint64_t pcells = static_cast<uint64_t>(G) * n_it;
      pc.ensure(static_cast<size_t>(Js) * std::max<uint64_t>(pcells, 1) * 4);
      CSG_CUDA(cudaMemsetAsync(pc.p, 0, static_cast<size_t>(Js) * pcells * 4, st));
      auto grid_for = [](uint64_t n) {
        return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 16)));
      };
      const bool inc = R > 0 && ordered && !inc_off;
      if (inc) {
        {
          const int32_t cached = std::min(Js, 8192);
          ProfScope ps_(c->lc, "k_iter_tables", st);
          // one block of kIterParts warps per rank
          k_iter_tables_inc<<<static_cast<unsigned>(R), 32 * kIterParts,
                              static_cast<size_t>(cached) * 4, st>>>(
              sv, mv, Js, dstrag, rs.as<RankSum>(), it_min, n_it, M, cached,
              tbl_s.as<unsigned long long>(), tbl_e.as<unsigned long long>());
        }
        ProfScope ps_(c->lc, "k_iter_prefix", st);
        k_iter_prefix<<<grid_for(per), 256, 0, st>>>(
            Js, per, n_it, G, slot_group.as<uint32_t>(), mv.members,
            sharded ? r0 : INT_MIN, sharded ? r0 + nr - 1 : INT_MAX, tbl_s.as<unsigned long long>(),
            tbl_e.as<unsigned long long>(), pc.as<uint32_t>());
      } else {
        if (R > 0) {
          const uint64_t warps = static_cast<uint64_t>(R) * Js;
          ProfScope ps_(c->lc, "k_iter_tables", st);
          k_iter_tables<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0,
                          st>>>(sv, mv, Js, dstrag, rs.as<RankSum>(), it_min, n_it,
                                M, tbl_s.as<unsigned long long>(),
                                tbl_e.as<unsigned long long>());
        }
        ProfScope ps_(c->lc, "k_iter_count", st);
        k_iter_count<<<grid_for(static_cast<uint64_t>(Js) * per), 256, 0, st>>>(
            Js, per, n_it, G, slot_group.as<uint32_t>(), tbl_s.as<unsigned long long>(),
            pc.as<uint32_t>());
      }
      // sharded: a slot's cells live on the shard owning its rank, so the
      // member counts sum across shards; the tables themselves are only
      // exchanged at the cells read from here on (k_win_xfer)
      comm_allreduce(c, pc.p, static_cast<size_t>(Js) * pcells, ncclUint32, ncclSum);
      if (inc && Js > 1) {
        ProfScope ps_(c->lc, "k_pc_prefix", st);
        k_pc_prefix<<<grid_for(pcells), 256, 0, st>>>(Js, pcells, pc.as<uint32_t>());
      }
      const uint64_t gw = static_cast<uint64_t>(G) * Js;
      const unsigned gblocks = static_cast<unsigned>((gw * 32 + 255) / 256);
      if (sharded) {
        {
          ProfScope ps_(c->lc, "k_group_iters", st);
          k_group_iters<<<gblocks, 256, 0, st>>>(
              mv, Js, it_min, n_it, M, k, cfg.straggler_threshold_ms,
              tbl_s.as<unsigned long long>(), tbl_e.as<unsigned long long>(),
              pc.as<uint32_t>(), 1, gi.as<GroupIter>(), gi_last.as<int64_t>());
        }
        DevBuf& pk_s = c->buf("rca.win_s");
        DevBuf& pk_e = c->buf("rca.win_e");
        const size_t pn = static_cast<size_t>(Js) * M * k;
        pk_s.ensure(pn * 8);
        pk_e.ensure(pn * 8);
        CSG_CUDA(cudaMemsetAsync(pk_s.p, 0xff, pn * 8, st));
        CSG_CUDA(cudaMemsetAsync(pk_e.p, 0, pn * 8, st));
        {
          ProfScope ps_(c->lc, "k_win_xfer", st);
          k_win_xfer<<<gblocks, 256, 0, st>>>(mv, Js, it_min, n_it, M, k, gi.as<GroupIter>(),
                                              gi_last.as<int64_t>(),
                                              tbl_s.as<unsigned long long>(),
                                              tbl_e.as<unsigned long long>(),
                                              pk_s.as<unsigned long long>(),
                                              pk_e.as<unsigned long long>(), 0);
        }
        comm_group_start(c);
        comm_allreduce(c, pk_s.p, pn, ncclUint64, ncclMin);
        comm_allreduce(c, pk_e.p, pn, ncclUint64, ncclMax);
        comm_group_end(c);
        {
          ProfScope ps_(c->lc, "k_win_xfer", st);
          k_win_xfer<<<gblocks, 256, 0, st>>>(mv, Js, it_min, n_it, M, k, gi.as<GroupIter>(),
                                              gi_last.as<int64_t>(),
                                              tbl_s.as<unsigned long long>(),
                                              tbl_e.as<unsigned long long>(),
                                              pk_s.as<unsigned long long>(),
                                              pk_e.as<unsigned long long>(), 1);
        }
      }
      ProfScope ps_(c->lc, "k_group_iters", st);
      k_group_iters<<<gblocks, 256, 0, st>>>(
          mv, Js, it_min, n_it, M, k, cfg.straggler_threshold_ms,
          tbl_s.as<unsigned long long>(), tbl_e.as<unsigned long long>(),
          pc.as<uint32_t>(), sharded ? 2 : 3, gi.as<GroupIter>(), gi_last.as<int64_t>());
    }
  }
  // K4: affected groups
  DevBuf& aff = c->buf("rca.aff");
  DevBuf& aff_flag = c->buf("rca.aff_flag");
  DevBuf& n_aff = c->buf("rca.n_aff");
  aff.ensure(static_cast<size_t>(J) * std::max(G, 1) * 4);
  aff_flag.ensure(static_cast<size_t>(J) * std::max(G, 1));
  n_aff.ensure(static_cast<size_t>(J) * 4);
  {
    // per-trip slice counters: zeroed once, reset by the last slice
    DevBuf& sdone = c->buf("rca.aff_slices");
    if (sdone.bytes < static_cast<size_t>(J) * 4) {
      sdone.ensure(static_cast<size_t>(J) * 4);
      CSG_CUDA(cudaMemsetAsync(sdone.p, 0, sdone.bytes, st));
    }
    ProfScope ps_(c->lc, "k_affected", st);
    launch_pdl(k_affected, dim3(dim3(J, kAffSlices)), dim3(1024), 0, st, 
        sv, mv, J, dkind, drank, djs, rs.as<RankSum>(), gi.as<GroupIter>(), aff.as<int32_t>(),
        aff_flag.as<uint8_t>(), n_aff.as<int32_t>(), sdone.as<unsigned>());
  }
  HostBuf& h_affb = c->hbuf("rca.aff");
  h_affb.ensure(static_cast<size_t>(J) * (static_cast<size_t>(G) + 1) * 4 + 16);
  int32_t* h_na = h_affb.as<int32_t>();
  int32_t* h_ag = h_na + J;
  // Failure-only batches are planned on the device (k_fail_plan) when the
  // upper-bound layout (every failure trip affecting every group) is small:
  // no host round trip between k_affected and the candidate kernels; the
  // affected groups come back with the final results.
  const int EV = kEvSlots(nch);
  int32_t Jf = 0;
  for (int32_t j = 0; j < J; ++j) Jf += h_kind[j] == CSG_TRIGGER_FAILURE ? 1 : 0;
  const uint64_t ub_items = static_cast<uint64_t>(Jf) * G;
  const uint64_t ub_cand = static_cast<uint64_t>(Jf) * M;
  const uint64_t ub_scratch =
      static_cast<uint64_t>(Jf) * exo_scratch_need(M, static_cast<uint64_t>(std::max(R, 1)));
  const uint64_t ub_bytes = ub_cand * (sizeof(Cand) + 2 * EV * sizeof(csg_evidence) +
                                       2 * sizeof(csg_suspect)) +
                            ub_scratch + ub_items * (sizeof(FailItem) + sizeof(GroupPick) + 4);
  static const bool no_dev_plan = std::getenv("CSG_HOST_FAIL_PLAN") != nullptr;
  const bool dev_plan = !no_dev_plan && !affected_only && Js == 0 && Jf > 0 && opn > 0 &&
                        M > 0 && ub_bytes <= (512ull << 20) && ub_items < (1ull << 30) &&
                        2 * ub_cand < 0xF0000000ull && ub_cand * EV < 0xF0000000ull;
  if (!dev_plan) {
    FetchArgs fa{};
    fa.add(n_aff.p, h_na, static_cast<size_t>(J) * 4);
    // only each trip's affected groups cross PCIe, not the J x G matrix
    if (G) fa.add_rows(aff.p, h_ag, static_cast<size_t>(G) * 4, n_aff.as<int32_t>(), J);
    ctx_sync(c, &fa);
  }
  tl_mark("affected sync returned");
  std::vector<int32_t> h_naff(J, 0);
  if (!dev_plan) h_naff.assign(h_na, h_na + J);
  out.aff = h_ag;
  CSG_CUDA(cudaGetLastError());
  c->d2h_bytes += static_cast<uint64_t>(J) * 4 + static_cast<uint64_t>(J) * G * 4;
  out.trips.assign(J, TripOut{});
  for (int32_t j = 0; j < J; ++j) out.trips[j].n_aff = h_naff[j];
  if (affected_only) return;

  DevBuf& err = c->buf("rca.err");
  err.ensure(4);
  CSG_CUDA(cudaMemsetAsync(err.p, 0, 4, st));
  // K5: straggler flow rules
  DevBuf& fs = c->buf("rca.fs");
  fs.ensure(static_cast<size_t>(std::max(Js, 1)) * std::max<uint32_t>(M, 1) * sizeof(FlowSum));
  if (Js > 0 && opn > 0 && M > 0) {
    store_build_op_index(s, opn);
    const uint64_t warps = static_cast<uint64_t>(M) * Js;
    static const bool flow_scan = std::getenv("CSG_FLOW_SCAN") != nullptr;
    if (!flow_scan && s->flow_indexed) {
      DevBuf& spill = c->buf("rca.flow_spill");
      spill.ensure(warps * 4 + 16);
      unsigned* nsp = spill.as<unsigned>();
      CSG_CUDA(cudaMemsetAsync(nsp, 0, 16, st));
      {
        ProfScope ps_(c->lc, "k_flow_fi", st);
        k_flow_fi<<<static_cast<unsigned>((warps * 32 + kFlow2Warps * 32 - 1) / (kFlow2Warps * 32)),
                    kFlow2Warps * 32, 0, st>>>(
            sv, s->flow_view(), mv, Js, dstrag, dt, cfg.delta_ms, cfg.flow_skew_factor, k, M,
            slot_group.as<uint32_t>(), rs.as<RankSum>(), gi.as<GroupIter>(),
            aff_flag.as<uint8_t>(), fs.as<FlowSum>(), err.as<uint32_t>(),
            spill.as<uint32_t>() + 4, nsp);
      }
      ProfScope ps_(c->lc, "k_flow", st);
      k_flow<<<148 * 2, kFlowWarps * 32, 0, st>>>(
          sv, mv, Js, dstrag, dt, cfg.delta_ms, cfg.flow_skew_factor, k, M,
          slot_group.as<uint32_t>(), rs.as<RankSum>(), gi.as<GroupIter>(),
          aff_flag.as<uint8_t>(), fs.as<FlowSum>(), err.as<uint32_t>(),
          spill.as<uint32_t>() + 4, nsp);
    } else {
      ProfScope ps_(c->lc, "k_flow", st);
      k_flow<<<static_cast<unsigned>((warps * 32 + 127) / 128), 128, 0, st>>>(
          sv, mv, Js, dstrag, dt, cfg.delta_ms, cfg.flow_skew_factor, k, M,
          slot_group.as<uint32_t>(), rs.as<RankSum>(), gi.as<GroupIter>(),
          aff_flag.as<uint8_t>(), fs.as<FlowSum>(), err.as<uint32_t>(), nullptr, nullptr);
    }
    comm_allreduce(c, fs.p, static_cast<size_t>(Js) * M * sizeof(FlowSum) / 8,
                   ncclUint64, ncclSum);
  }

  // ---- failure trips: per-group candidates + per-trip exoneration ----
  std::vector<FailItem> items;
  std::vector<ExoTrip> exo;
  std::vector<uint64_t> item_m;  // members per item (upper bound of its cands)
  uint64_t cand_ub = 0, sus_fail = 0, ev_fail = 0, scratch_bytes = 0;
  uint64_t tot_all = 0, tot_max = 0;
  int32_t m_max = 1;
  for (int32_t g = 0; g < G; ++g)
    m_max = std::max<int32_t>(m_max, m->h_member_off[g + 1] - m->h_member_off[g]);
  for (int32_t j = 0; j < J && !dev_plan; ++j) {
    uint64_t tot = 0;
    for (int32_t i = 0; i < h_naff[j]; ++i) {
      const int32_t g = out.aff[static_cast<size_t>(j) * G + i];
      tot += m->h_member_off[g + 1] - m->h_member_off[g];
    }
    tot_all += tot;
    tot_max = std::max(tot_max, tot);
    if (h_kind[j] != CSG_TRIGGER_FAILURE || h_naff[j] == 0 || opn == 0) continue;
    ExoTrip e;
    std::memset(&e, 0, sizeof(e));
    e.j = j;
    e.naff = h_naff[j];
    e.first_item = static_cast<uint32_t>(items.size());
    e.n_items = static_cast<uint32_t>(h_naff[j]);
    for (int32_t i = 0; i < h_naff[j]; ++i)
      items.push_back(FailItem{j, out.aff[static_cast<size_t>(j) * G + i]});
    const uint64_t C = tot;
    uint64_t P = 1;
    while (P < C) P <<= 1;
    const uint64_t Rs = std::max<int32_t>(R, 1);
    const uint64_t need = ((P * 4 + 15) & ~15ull) + ((C * 8 + 15) & ~15ull) +
                          ((C * 4 + 15) & ~15ull) + ((C + 15) & ~15ull) +
                          4 * ((Rs + 3) & ~3ull) + 8 * (((Rs + 31) / 32 + 3) & ~3ull) +
                          32 * C + 64;
    e.scratch_off = scratch_bytes;
    scratch_bytes += (need + 255) & ~255ull;
    e.sus_off = static_cast<uint32_t>(sus_fail);
    sus_fail += 2 * C;
    e.ev_off = static_cast<uint32_t>(ev_fail);
    ev_fail += C * EV;
    cand_ub += C;
    exo.push_back(e);
  }
  if (sus_fail > 0xF0000000ull || ev_fail > 0xF0000000ull || cand_ub * EV > 0xF0000000ull)
    throw Error(CSG_ERR_RUNTIME, "engine: failure analysis outputs exceed 2^32 entries");
  const int32_t n_items = static_cast<int32_t>(items.size());
  DevBuf& d_items = c->buf("rca.items");
  DevBuf& d_pick = c->buf("rca.pick");
  DevBuf& d_off = c->buf("rca.off");
  DevBuf& d_cand = c->buf("rca.cand");
  DevBuf& d_cev = c->buf("rca.cev");
  ExoTrip* d_exo_ptr = nullptr;
  DevBuf& d_exs = c->buf("rca.exo_scratch");
  tl_mark("fail items planned");
  DevBuf& d_plan = c->buf("rca.fail_plan");
  d_plan.ensure(sizeof(FailPlan) + 16);
  int32_t n_exo_grid = static_cast<int32_t>(exo.size());
  if (dev_plan) {
    d_items.ensure(ub_items * sizeof(FailItem) + 16);
    d_exo_ptr = reinterpret_cast<ExoTrip*>(c->buf("rca.exo_dev").p);
    {
      DevBuf& dx = c->buf("rca.exo_dev");
      dx.ensure(static_cast<size_t>(J) * sizeof(ExoTrip) + 16);
      d_exo_ptr = dx.as<ExoTrip>();
    }
    d_pick.ensure(ub_items * sizeof(GroupPick) + 16);
    d_off.ensure((ub_items + 1) * 4);
    d_cand.ensure(ub_cand * sizeof(Cand) + sizeof(Cand));
    d_cev.ensure(ub_cand * EV * sizeof(csg_evidence) + sizeof(csg_evidence));
    d_exs.ensure(ub_scratch + 256);
    DevBuf& p_used0 = c->buf("rca.p_used");
    p_used0.ensure(8 * 8);
    {
      ProfScope ps_(c->lc, "k_fail_plan", st);
      k_fail_plan<<<1, 1024, 0, st>>>(J, G, dkind, n_aff.as<int32_t>(), aff.as<int32_t>(), mv,
                                      R, EV, d_items.as<FailItem>(), d_exo_ptr,
                                      d_plan.as<FailPlan>(),
                                      p_used0.as<unsigned long long>());
    }
    const unsigned* n_dev = &d_plan.as<FailPlan>()->n_items;
    {
      ProfScope ps_(c->lc, "k_fail_count", st);
      launch_pdl(k_fail_count, dim3(static_cast<unsigned>((ub_items * 32 + 255) / 256)), dim3(256), 0, st, 
          sv, mv, d_items.as<FailItem>(), static_cast<int32_t>(ub_items), rs.as<RankSum>(),
          d_pick.as<GroupPick>(), d_off.as<uint32_t>(), n_dev);
    }
    exclusive_scan_u32(d_off.as<uint32_t>(), ub_items + 1, c->buf("rca.scan_tmp"), st, c->lc);
    {
      ProfScope ps_(c->lc, "k_fail_cands", st);
      launch_pdl(k_fail_cands, dim3(static_cast<unsigned>((ub_items * 32 + 127) / 128)), dim3(128), 0, st, 
          sv, mv, d_items.as<FailItem>(), static_cast<int32_t>(ub_items), rs.as<RankSum>(),
          chan_key.as<unsigned long long>(), succ.as<SuccProg>(),
          succ_key.as<unsigned long long>(), M, nch, d_pick.as<GroupPick>(),
          d_off.as<uint32_t>(), d_cand.as<Cand>(), d_cev.as<csg_evidence>(),
          err.as<uint32_t>(), n_dev);
    }
    // pool regions sized by the bounds; the exact values come back with the
    // results (needed only if a retry re-initialises the pools)
    sus_fail = 2 * ub_cand;
    ev_fail = ub_cand * EV;
    n_exo_grid = J;
  }
  if (n_items > 0) {
    // items, exoneration trips and the zero closing the offset scan: one
    // pinned upload
    const size_t ib = items.size() * sizeof(FailItem), xb = exo.size() * sizeof(ExoTrip);
    const size_t xo = (ib + 15) & ~size_t(15), zo = (xo + xb + 15) & ~size_t(15);
    d_items.ensure(zo + 16);
    d_items.stage.ensure(zo + 16);
    std::memcpy(d_items.stage.p, items.data(), ib);
    std::memcpy(d_items.stage.as<unsigned char>() + xo, exo.data(), xb);
    std::memset(d_items.stage.as<unsigned char>() + zo, 0, 4);
    CSG_CUDA(cudaMemcpyAsync(d_items.p, d_items.stage.p, zo + 4, cudaMemcpyHostToDevice, st));
    d_pick.ensure(static_cast<size_t>(n_items) * sizeof(GroupPick));
    d_off.ensure(static_cast<size_t>(n_items + 1) * 4);  // [n_items] zeroed by k_fail_count
    d_cand.ensure(cand_ub * sizeof(Cand) + sizeof(Cand));
    d_cev.ensure(cand_ub * EV * sizeof(csg_evidence) + sizeof(csg_evidence));
    d_exo_ptr = reinterpret_cast<ExoTrip*>(d_items.as<unsigned char>() + xo);
    d_exs.ensure(scratch_bytes + 256);
    {
      ProfScope ps_(c->lc, "k_fail_count", st);
      launch_pdl(k_fail_count, dim3(static_cast<unsigned>((static_cast<uint64_t>(n_items) * 32 + 255) / 256)), dim3(256), 0, st, sv, mv, d_items.as<FailItem>(), n_items,
                                   rs.as<RankSum>(), d_pick.as<GroupPick>(),
                                   d_off.as<uint32_t>(), nullptr);
    }
    exclusive_scan_u32(d_off.as<uint32_t>(), static_cast<uint64_t>(n_items) + 1,
                       c->buf("rca.scan_tmp"), st, c->lc);
    {
      ProfScope ps_(c->lc, "k_fail_cands", st);
      launch_pdl(k_fail_cands, dim3(static_cast<unsigned>((static_cast<uint64_t>(n_items) * 32 + 127) / 128)), dim3(128), 0, st, sv, mv, d_items.as<FailItem>(), n_items,
                                   rs.as<RankSum>(), chan_key.as<unsigned long long>(),
                                   succ.as<SuccProg>(), succ_key.as<unsigned long long>(),
                                   M, nch,
                                   d_pick.as<GroupPick>(), d_off.as<uint32_t>(),
                                   d_cand.as<Cand>(), d_cev.as<csg_evidence>(),
                                   err.as<uint32_t>(), nullptr);
    }
  }

  // ---- output pools: failure regions first, straggler bump allocations after
  const uint64_t C2 = 2 * tot_max + 8;
  const uint64_t per_ev = std::max<uint64_t>(2 * nch + 1, k + 1);
  const uint64_t pm = std::max<uint64_t>(1, c->rca_pool_mult);  // grown last time
  uint64_t cand_cap = Js ? (2 * tot_all + 16) * pm : 16;
  uint64_t cev_cap = Js ? (tot_all * per_ev + 16) * pm : 16;
  uint64_t sus_cap = sus_fail + (Js ? 6 * tot_all * pm : 0) + 16;
  uint64_t ev_cap = ev_fail + (Js ? tot_all * per_ev * pm : 0) + 16;
  // grow-only across calls: a replay of the same store does not pay the
  // DAG-scratch retry again
  uint64_t bits_cap = std::max<uint64_t>(1ull << 22, c->rca_bits_cap);
  const uint64_t mwords = (static_cast<uint64_t>(R) + 31) / 32 + 1;
  uint64_t spt = 16;
  if (Js) {
    spt = std::max<uint64_t>(12 * C2, 4 * static_cast<uint64_t>(m_max));
    spt = std::max<uint64_t>(spt, mwords + 2 * std::max<uint64_t>(
                                                  std::max<uint64_t>(m_max, s->max_seg),
                                                  8 * C2));
  }
  spt = (spt + 64 + 3) & ~3ull;  // 16-byte aligned per-trip slices
  if (spt > 0xFFFFFFF0ull)
    throw Error(CSG_ERR_RUNTIME, "engine: per-trip scratch exceeds 2^32 words");
  DevBuf& p_cand = c->buf("rca.p_cand");
  DevBuf& p_cev = c->buf("rca.p_cev");
  DevBuf& p_sus = c->buf("rca.p_sus");
  DevBuf& p_ev = c->buf("rca.p_ev");
  DevBuf& p_bits = c->buf("rca.p_bits");
  DevBuf& p_u32 = c->buf("rca.p_u32");
  DevBuf& p_used = c->buf("rca.p_used");
  DevBuf& d_out = c->buf("rca.out");
  d_out.ensure(static_cast<size_t>(J) * sizeof(TripOut));
  p_used.ensure(8 * 8);
  p_u32.ensure(static_cast<size_t>(Js ? J : 1) * spt * 4);
  DecideArgs a;
  a.s = sv;
  a.m = mv;
  a.J = J;
  a.trip_t = dt;
  a.trip_kind = dkind;
  a.trip_rank = drank;
  a.js_of = djs;
  a.rs = rs.as<RankSum>();
  a.chan_key = chan_key.as<unsigned long long>();
  a.nch = nch;
  a.aff = aff.as<int32_t>();
  a.n_aff = n_aff.as<int32_t>();
  a.gi = gi.as<GroupIter>();
  a.gi_last = gi_last.as<int64_t>();
  a.k = k;
  a.fs = fs.as<FlowSum>();
  a.tbl_s = tbl_s.as<unsigned long long>();
  a.tbl_e = tbl_e.as<unsigned long long>();
  a.it_min = it_min;
  a.n_it = n_it;
  a.M = M;
  a.delta_a = cfg.delta_ms;
  a.thr = cfg.straggler_threshold_ms;
  a.skew = cfg.flow_skew_factor;
  a.N = s->n_global;
  a.opk = s->opidx_keys.as<uint64_t>();
  a.oprank = s->opidx_rank.as<int32_t>();
  a.op_ts = s->opidx_ts.as<double>();
  a.op_dur = s->opidx_dur.as<double>();
  a.op_nm = s->opidx_nm.as<uint8_t>();
  a.sharded = comm_active(c) ? 1 : 0;
  a.n_opidx = s->op_indexed ? s->n_opidx : 0;
  a.min_op = s->min_op;
  a.max_op = s->max_op;
  a.sf_fast = 0;
  a.f = FlowView();
  a.opoff = nullptr;
  a.sdur = nullptr;
  a.sts = nullptr;
  a.srank = nullptr;
  a.opmax = nullptr;
  a.plan = nullptr;
  static const bool sf_slow = std::getenv("CSG_SF_SLOW") != nullptr;
  DevBuf& d_sfl = c->buf("rca.sf_large");
  constexpr uint32_t kLargeCap = 1u << 16;
  if (Js > 0 && !sf_slow && s->op_indexed && s->flow_indexed) {
    a.sf_fast = 1;
    a.f = s->flow_view();
    a.opoff = s->op_seg_off.as<uint32_t>();
    DevBuf& d_sdur = c->buf("rca.sdur");
    d_sdur.ensure(s->n_opidx * 8 + 16);
    a.sdur = d_sdur.as<unsigned long long>();
    DevBuf& d_sts = c->buf("rca.sts");
    d_sts.ensure(s->n_opidx * 8 + 16);
    a.sts = d_sts.as<double>();
    DevBuf& d_srk = c->buf("rca.srank");
    d_srk.ensure(s->n_opidx * 4 + 16);
    a.srank = d_srk.as<int32_t>();
    DevBuf& d_opmax = c->buf("rca.opmax");
    const uint64_t range = s->max_op >= s->min_op ? static_cast<uint64_t>(s->max_op - s->min_op) : 0;
    d_opmax.ensure((range + 2) * 8 + 16);
    a.opmax = d_opmax.as<double>();
    DevBuf& d_plan2 = c->buf("rca.sf_plan");
    d_plan2.ensure(sizeof(SfPlan) + static_cast<size_t>(J + 1) * 8 + 16);
    a.plan = d_plan2.as<SfPlan>();
    d_sfl.ensure(static_cast<size_t>(kLargeCap) * 4 + 64);
  }
  DevBuf& d_pend = c->buf("rca.sf_pend");
  a.pend_ops = nullptr;
  a.pend_n = nullptr;
  static const bool sl_serial = std::getenv("CSG_SL_SERIAL") != nullptr;
  a.sl_par = (Js > 0 && !sl_serial && M > 0 && opn > 0) ? 1 : 0;
  a.strag_trip = dstrag;
  DevBuf& d_sll = c->buf("rca.sl_late");
  DevBuf& d_slc = c->buf("rca.sl_cnt");
  if (a.sl_par) {
    d_sll.ensure(static_cast<size_t>(Js) * M + 16);
    d_slc.ensure(static_cast<size_t>(Js) * std::max(G, 1) * sizeof(uint2) + 16);
    CSG_CUDA(cudaMemsetAsync(d_sll.p, 0, static_cast<size_t>(Js) * M, st));
  }
  a.sl_late = d_sll.as<uint8_t>();
  a.emit_rank = nullptr;
  a.emit_stride = 0;
  static const bool emit_serial = std::getenv("CSG_SL_SERIAL") != nullptr;
  if (Js > 0 && !emit_serial) {
    const uint64_t RS = static_cast<uint64_t>(std::max(m->view().rank_space, 1));
    a.emit_stride = RS + 2 * ((RS + 31) / 32) + 8;
    DevBuf& d_er = c->buf("rca.emit_rank");
    d_er.ensure(static_cast<size_t>(J) * a.emit_stride * 4 + 16);
    a.emit_rank = d_er.as<uint32_t>();
  }
  a.sl_cnt = d_slc.as<uint2>();
  a.scratch_per_trip = static_cast<uint32_t>(spt);
  DevBuf& d_state = c->buf("rca.strag_state");
  d_state.ensure(static_cast<size_t>(J) * sizeof(StragState) + 16);
  CSG_CUDA(cudaMemsetAsync(d_state.p, 0, static_cast<size_t>(J) * sizeof(StragState), st));
  a.state = d_state.as<StragState>();
  {  // self_faulted's list + first-occurrence bitmap behind it
    const uint64_t base =
        std::max<uint64_t>(16, (spt - ((static_cast<uint64_t>(R) + 31) / 32 + 1)) / 2);
    a.sf_words = static_cast<uint32_t>(base + base / 32 + 2);
  }
  DevBuf& d_sf = c->buf("rca.sf_scratch");
  if (Js > 0) d_sf.ensure(static_cast<size_t>(kSfBlocks) * a.sf_words * 4);
  a.sf_scratch = d_sf.as<uint32_t>();
  DevBuf& d_coh = c->buf("rca.cohort");
  a.coh_cap = 0;
  if (Js > 0) {  // (trip, op name, iteration) cohorts: room for 32 iterations per trip
    uint32_t cap = 4096;
    while (cap < static_cast<uint64_t>(J) * kCohortNames * 64) cap <<= 1;
    a.coh_cap = cap;
  }
  if (Js > 0) {
    d_coh.ensure(static_cast<size_t>(a.coh_cap) * 64 + 64);
    a.coh_key = d_coh.as<unsigned long long>();
    a.coh_val = reinterpret_cast<double*>(a.coh_key + a.coh_cap);
    a.coh_meta = reinterpret_cast<longlong2*>(a.coh_val + a.coh_cap);
    a.coh2_key = reinterpret_cast<unsigned long long*>(a.coh_meta + a.coh_cap);
    a.coh2_val = reinterpret_cast<double*>(a.coh2_key + a.coh_cap);
    a.coh2_mx = a.coh2_val + a.coh_cap;
    a.coh_state = reinterpret_cast<unsigned*>(a.coh2_mx + a.coh_cap);
    a.coh2_state = a.coh_state + a.coh_cap;
  }
  a.phase = 1;
  a.debug = std::getenv("CSG_DEBUG_EXO") != nullptr;
  a.out = d_out.as<TripOut>();
  a.err = err.as<uint32_t>();
  const size_t shm = sizeof(BlockShared);
  smem_optin(k_decide, shm);
  uint32_t h_err = 0;
  unsigned long long used[8];
  std::vector<TripOut> to(J);
  HostBuf& h_sus = c->hbuf("rca.packed_sus");
  HostBuf& h_ev = c->hbuf("rca.packed_ev");
  for (int attempt = 0;; ++attempt) {
    p_cand.ensure(cand_cap * sizeof(Cand));
    p_cev.ensure(cev_cap * sizeof(csg_evidence));
    p_sus.ensure(sus_cap * sizeof(csg_suspect));
    p_ev.ensure(ev_cap * sizeof(csg_evidence));
    p_bits.ensure(bits_cap * 8);
    a.pools.cand = p_cand.as<Cand>();
    a.pools.cand_cap = cand_cap;
    a.pools.cev = p_cev.as<csg_evidence>();
    a.pools.cev_cap = cev_cap;
    a.pools.sus = p_sus.as<csg_suspect>();
    a.pools.sus_cap = sus_cap;
    a.pools.ev = p_ev.as<csg_evidence>();
    a.pools.ev_cap = ev_cap;
    a.pools.bits = p_bits.as<unsigned long long>();
    a.pools.bits_cap = bits_cap;
    a.pools.u32 = p_u32.as<uint32_t>();
    a.pools.u32_cap = static_cast<unsigned long long>(J) * spt;
    a.pools.used = p_used.as<unsigned long long>();
    // device-planned batches: k_fail_plan initialised the pool usage on the
    // first attempt; a retry uses the exact region sizes it reported
    if (!dev_plan || attempt > 0) {
      unsigned long long init_used[8] = {0, 0, sus_fail, ev_fail, 0, 0, 0, 0};
      CSG_CUDA(cudaMemcpyAsync(p_used.p, init_used, 8 * 8, cudaMemcpyHostToDevice, st));
    }
    if (n_exo_grid > 0) {
      ExoArgs ea;
      ea.debug = std::getenv("CSG_DEBUG_EXO") != nullptr;
      ea.warp_sweep = std::getenv("CSG_EXO_WARP_SWEEP") != nullptr;
      ea.s = sv;
      ea.m = mv;
      ea.cand = d_cand.as<Cand>();
      ea.cev = d_cev.as<csg_evidence>();
      ea.EV = EV;
      ea.off = d_off.as<uint32_t>();
      ea.trips = d_exo_ptr;
      ea.n_trips = n_exo_grid;
      ea.scratch = d_exs.as<unsigned char>();
      ea.bits = p_bits.as<unsigned long long>();
      ea.bits_cap = bits_cap;
      ea.bits_used = p_used.as<unsigned long long>() + P_BITS;
      ea.sus = p_sus.as<csg_suspect>();
      ea.ev = p_ev.as<csg_evidence>();
      ea.out = d_out.as<TripOut>();
      ea.N = s->n_global;
      ea.err = err.as<uint32_t>();
      smem_optin(k_exonerate, kExoSmemMax);
      ProfScope ps_(c->lc, "k_exonerate", st);
      launch_pdl(k_exonerate, dim3(static_cast<unsigned>(n_exo_grid)), dim3(kExoThreads), kExoSmemMax, st, ea);
    }
    if (a.sl_par) {  // straggler candidates, every (trip, group) in parallel
      const uint64_t wg = static_cast<uint64_t>(Js) * G;
      const unsigned gb = static_cast<unsigned>((wg + kSlWarps - 1) / kSlWarps);
      {  // every attempt: k_sl_scan turns the counts into offsets in place
        ProfScope ps_(c->lc, "k_sl_late", st);
        k_sl_late<<<gb, kSlWarps * 32, 0, st>>>(a, Js);
      }
      {
        ProfScope ps_(c->lc, "k_sl_count", st);
        k_sl_count<<<gb, kSlWarps * 32, 0, st>>>(a, Js);
      }
      {
        ProfScope ps_(c->lc, "k_sl_scan", st);
        k_sl_scan<<<Js, 1024, 0, st>>>(a);
      }
      {
        ProfScope ps_(c->lc, "k_sl_emit", st);
        k_sl_emit<<<gb, kSlWarps * 32, 0, st>>>(a, Js);
      }
    }
    if (!dev_plan) {  // device-planned batches are failure-only: k_exonerate wrote every trip
      ProfScope ps_(c->lc, "k_decide", st);
      a.phase = 1;
      k_decide<<<J, kDecideThreads, shm, st>>>(a);
    }
    if (Js > 0) {
      // straggler self-evidence over every candidate in parallel, then the
      // per-trip filter + report
      CSG_CUDA(cudaMemsetAsync(a.coh_key, 0xff, static_cast<size_t>(a.coh_cap) * 8, st));
      CSG_CUDA(cudaMemsetAsync(a.coh_state, 0, static_cast<size_t>(a.coh_cap) * 8, st));
      CSG_CUDA(cudaMemsetAsync(a.coh2_key, 0xff, static_cast<size_t>(a.coh_cap) * 8, st));
      if (!a.sf_fast) {  // every cohort of the candidates' windows, up front
        ProfScope ps_(c->lc, "k_cohorts", st);
        k_cohorts<<<dim3(J, static_cast<unsigned>(std::max(k, 1) + 1), kCohortNames),
                    kDecideThreads, shm, st>>>(a);
      }
      if (a.sf_fast) {
        d_pend.ensure(cand_cap * (kSfPend * 8 + 1) + 64);
        a.pend_ops = d_pend.as<int64_t>();
        a.pend_n = reinterpret_cast<uint8_t*>(a.pend_ops + cand_cap * kSfPend);
        unsigned* nl = d_sfl.as<unsigned>();
        unsigned* large = nl + 16;
        CSG_CUDA(cudaMemsetAsync(nl, 0, 16, st));
        {
          ProfScope ps_(c->lc, "k_sf_prep", st);
          k_sf_prep<<<1, 1024, 0, st>>>(a);
        }
        {
          ProfScope ps_(c->lc, "k_opsort", st);
          k_opsort<<<148 * 4, 256, 0, st>>>(a, large, nl, kLargeCap);
        }
        {
          const size_t lsm = static_cast<size_t>(kOpSortBlockCap) * 10;
          smem_optin(k_opsort_large, lsm);
          ProfScope ps_(c->lc, "k_opsort_large", st);
          k_opsort_large<<<148, 1024, lsm, st>>>(a, large, nl, kLargeCap);
        }
        static const bool dbg_sf = std::getenv("CSG_DEBUG_SF") != nullptr;
        unsigned* why = dbg_sf ? nl + 8 : nullptr;
        if (why) CSG_CUDA(cudaMemsetAsync(why, 0, 8 * 4, st));
        {
          ProfScope ps_(c->lc, "k_sf_fast", st);
          k_sf_fast<<<148 * 16, kSfWarps * 32, 0, st>>>(a, why, 0);
        }
        {  // the cohorts the first pass asked for, then their candidates again
          ProfScope ps_(c->lc, "k_cohorts", st);
          static const bool coh_block = std::getenv("CSG_COHORT_BLOCK") != nullptr;
          if (coh_block) {
            k_cohorts_lazy<<<148 * 2, kDecideThreads, shm, st>>>(a);
          } else {
            DevBuf& d_ci = c->buf("rca.coh_items");
            d_ci.ensure(sizeof(CohPlan) + static_cast<size_t>(kCohItemsCap) * sizeof(CohItem) +
                        static_cast<size_t>(kCohItemsCap) * 256 * 4 + 64);
            CohPlan* cplan = d_ci.as<CohPlan>();
            CohItem* citems = reinterpret_cast<CohItem*>(d_ci.as<unsigned char>() + 64);
            uint32_t* chist = reinterpret_cast<uint32_t*>(citems + kCohItemsCap);
            DevBuf& d_ck = c->buf("rca.coh_ckeys");
            const uint64_t ccap = std::max<uint64_t>(1u << 16, std::min<uint64_t>(a.n_opidx, 1u << 24));
            d_ck.ensure(ccap * 8);
            unsigned long long* ck = d_ck.as<unsigned long long>();
            k_coh_collect<<<1, 1024, 0, st>>>(a, citems, cplan, chist);
            // the top digit's pass also counts each item's entries
            for (int sh2 = 56; sh2 >= 0; sh2 -= 8) {
              k_coh_pass<<<148 * 8, 256, 0, st>>>(a, citems, cplan, chist, sh2, ck);
              k_coh_pick<<<8, 256, 0, st>>>(a, citems, cplan, chist, sh2);
              if (sh2 == kCohCompactShift && !std::getenv("CSG_COH_NO_COMPACT")) {
                k_coh_offsets<<<1, 1024, 0, st>>>(citems, cplan, ccap);
                k_coh_compact<<<148 * 8, 256, 0, st>>>(a, citems, cplan, ck);
              }
            }
          }
        }
        {
          ProfScope ps_(c->lc, "k_sf_fast_p2", st);
          k_sf_fast<<<148 * 16, kSfWarps * 32, 0, st>>>(a, nullptr, 1);
        }
        if (a.sharded) {  // owners' verdicts to every shard
          DevBuf& d_fl = c->buf("rca.sf_flat");
          d_fl.ensure(cand_cap + 16);
          CSG_CUDA(cudaMemsetAsync(d_fl.p, 0, cand_cap, st));
          k_sf_pads<<<148 * 4, 256, 0, st>>>(a, d_fl.as<uint8_t>(), 0);
          comm_allreduce(c, d_fl.p, cand_cap, ncclUint8, ncclMax);
          k_sf_pads<<<148 * 4, 256, 0, st>>>(a, d_fl.as<uint8_t>(), 1);
        }
        if (why) {
          unsigned hw[8];
          CSG_CUDA(cudaMemcpyAsync(hw, why, sizeof(hw), cudaMemcpyDeviceToHost, st));
          CSG_CUDA(cudaStreamSynchronize(st));
          fprintf(stderr, "k_sf_fast: decided %u, deferred: no index %u, >32 completions %u, "
                  "unsorted segment %u, -- %u, cohort missing %u\n",
                  hw[0], hw[1], hw[2], hw[3], hw[4], hw[5]);
        }
      }
      {
        ProfScope ps_(c->lc, "k_self_faulted", st);
        k_self_faulted<<<kSfBlocks, kDecideThreads, shm, st>>>(a);
      }
      ProfScope ps_(c->lc, "k_decide", st);
      a.phase = 2;
      k_decide<<<J, kDecideThreads, shm, st>>>(a);
    }
    // pack straight into mapped host memory; the results, the trip table,
    // the pool usage and the error word all come back in ONE round trip
    h_sus.ensure(sus_cap * sizeof(csg_suspect) + 64);
    h_ev.ensure(ev_cap * sizeof(csg_evidence) + 64);
    // pinned: [0] error word, [16] pool usage, [80] packed totals, [96..) trips
    HostBuf& hr = c->hbuf("rca.tail");
    hr.ensure(96 + static_cast<size_t>(J) * sizeof(TripOut));
    unsigned char* hrp = hr.as<unsigned char>();
    {
      FetchArgs fa{};
      fa.add(err.p, hrp, 4);
      fa.add(p_used.p, hrp + 16, 8 * 8);
      fa.add(d_out.p, hrp + 96, static_cast<size_t>(J) * sizeof(TripOut));
      if (dev_plan) {  // the affected groups and the plan ride on this trip
        fa.add(n_aff.p, h_na, static_cast<size_t>(J) * 4);
        if (G) fa.add_rows(aff.p, h_ag, static_cast<size_t>(G) * 4, n_aff.as<int32_t>(), J);
        fa.add(d_plan.p, d_plan.stage.p ? d_plan.stage.p : (d_plan.stage.ensure(64), d_plan.stage.p),
               sizeof(FailPlan));
      }
      static const bool pack_fetch = std::getenv("CSG_PACK_FETCH") != nullptr;
      if (J > 0 && !pack_fetch) {
        // k_pack's last block copies the tail and raises the completion word
        c->sig.ensure(64);
        DevBuf& fdn = c->buf("fetch.done");
        if (fdn.bytes < 16) {
          fdn.ensure(16);
          CSG_CUDA(cudaMemsetAsync(fdn.p, 0, 16, st));
        }
        const unsigned long long v = ++c->sig_seq;
        {
          ProfScope ps_(c->lc, "k_pack", st);
          launch_pdl(k_pack, dim3(dim3(static_cast<unsigned>(3 * J), 8)), dim3(128), 0, st,
                     d_out.as<TripOut>(), J, p_sus.as<csg_suspect>(), p_ev.as<csg_evidence>(),
                     h_sus.as<csg_suspect>(), h_ev.as<csg_evidence>(), fa,
                     c->sig.as<unsigned long long>(), v, fdn.as<unsigned>());
        }
        CSG_CUDA(cudaGetLastError());
        if (!c->ev_fetch) CSG_CUDA(cudaEventCreateWithFlags(&c->ev_fetch, cudaEventDisableTiming));
        CSG_CUDA(cudaEventRecord(c->ev_fetch, st));
        ctx_fetch_wait(c, FetchTicket{v});
        // as ctx_sync: the stream is idle on return
        const cudaError_t e = cudaStreamQuery(st);
        if (e != cudaSuccess && e != cudaErrorNotReady) CSG_CUDA(e);
        if (e == cudaErrorNotReady) CSG_CUDA(cudaStreamSynchronize(st));
      } else {
        if (J > 0) {
          // unfused: the pack's own tail is a no-op (a null flag never fires
          // because fa is empty and the counter is private)
          DevBuf& pdn = c->buf("rca.pack_done");
          if (pdn.bytes < 16) {
            pdn.ensure(16);
            CSG_CUDA(cudaMemsetAsync(pdn.p, 0, 16, st));
          }
          DevBuf& pfl = c->buf("rca.pack_flag");
          pfl.ensure(16);
          ProfScope ps_(c->lc, "k_pack", st);
          launch_pdl(k_pack, dim3(dim3(static_cast<unsigned>(3 * J), 8)), dim3(128), 0, st,
                     d_out.as<TripOut>(), J, p_sus.as<csg_suspect>(), p_ev.as<csg_evidence>(),
                     h_sus.as<csg_suspect>(), h_ev.as<csg_evidence>(), FetchArgs{},
                     pfl.as<unsigned long long>(), 0ull, pdn.as<unsigned>());
        }
        ctx_sync(c, &fa);
      }
    }
    if (dev_plan) {
      const FailPlan* fp = d_plan.stage.as<FailPlan>();
      sus_fail = fp->sus_fail;
      ev_fail = fp->ev_fail;
    }
    std::memcpy(&h_err, hrp, 4);
    std::memcpy(used, hrp + 16, 8 * 8);
    std::memcpy(to.data(), hrp + 96, J * sizeof(TripOut));
    CSG_CUDA(cudaGetLastError());
    if (h_err & DEV_ERR_RC_TABLE)
      throw Error(CSG_ERR_RUNTIME,
                  "check_rc_table: counters violate the pipeline invariant");
    if (h_err & DEV_ERR_TOO_MANY_COMPS)
      throw Error(CSG_ERR_RUNTIME,
                  "engine: more than 256 completions of one (rank, op) in the "
                  "analysis window");
    if (!(h_err & (DEV_ERR_POOL | DEV_ERR_DAG_SCRATCH))) break;
    if (attempt >= 6)
      throw Error(CSG_ERR_RUNTIME, "engine: RCA output pools exhausted");
    static const bool dbg_retry = std::getenv("CSG_DEBUG_RETRY") != nullptr;
    if (a.debug || dbg_retry)
      fprintf(stderr, "rca retry %d: %s%s used cand %llu/%llu cev %llu/%llu sus %llu/%llu ev %llu/%llu\n",
              attempt, (h_err & DEV_ERR_POOL) ? "pools " : "",
              (h_err & DEV_ERR_DAG_SCRATCH) ? "dag-scratch" : "",
              (unsigned long long)used[P_CAND], (unsigned long long)cand_cap,
              (unsigned long long)used[P_CEV], (unsigned long long)cev_cap,
              (unsigned long long)used[P_SUS], (unsigned long long)sus_cap,
              (unsigned long long)used[P_EV], (unsigned long long)ev_cap);
    if (h_err & DEV_ERR_DAG_SCRATCH) {
      bits_cap = std::max<uint64_t>(bits_cap * 4, used[P_BITS] * 2);
      c->rca_bits_cap = bits_cap;
    }
    if (h_err & DEV_ERR_POOL) {
      c->rca_pool_mult = pm * 4;
      cand_cap *= 4;
      cev_cap *= 4;
      sus_cap = sus_fail + (sus_cap - sus_fail) * 4;
      ev_cap = ev_fail + (ev_cap - ev_fail) * 4;
    }
    h_err &= ~(DEV_ERR_POOL | DEV_ERR_DAG_SCRATCH);
    CSG_CUDA(cudaMemcpyAsync(err.p, &h_err, 4, cudaMemcpyHostToDevice, st));
  }
  // packed offsets, in the order k_pack wrote them
  uint64_t ns_tot = 0, ne_tot = 0;
  for (int32_t j = 0; j < J; ++j) {
    TripOut& t = to[j];
    t.sus_off = static_cast<uint32_t>(ns_tot);
    ns_tot += t.n_sus;
    t.exo_off = static_cast<uint32_t>(ns_tot);
    ns_tot += t.n_exo;
    t.ev_off = static_cast<uint32_t>(ne_tot);
    ne_tot += t.n_ev;
  }
  out.sus.assign(h_sus.as<csg_suspect>(), h_sus.as<csg_suspect>() + ns_tot);
  out.ev.assign(h_ev.as<csg_evidence>(), h_ev.as<csg_evidence>() + ne_tot);
  c->d2h_bytes += J * sizeof(TripOut) + ns_tot * sizeof(csg_suspect) +
                  ne_tot * sizeof(csg_evidence) + 8 * 8 + 4;
  out.trips = to;
}

}  // namespace csg
