// synth_flow.h — the synthetic generator's per-flow record expansion, shared
// verbatim by the host generator (host/synth.cpp) and the device generator
// (synth_gpu.cu) so both emit the same bytes.
//
// The host schedules op instances (dependencies, rank availability, faults)
// and produces one Flow per (instance, executing rank); each Flow expands,
// per channel, into the simulator's record pattern (sim.cpp:687-706, see
// synth.cpp): a state snapshot at every state-log window boundary inside the
// flow, then a flush snapshot and the completion at the flow's end. Both
// sides compile this with IEEE double arithmetic and no FMA contraction
// (g++ without -march on x86-64; nvcc -fmad=false), and use the <algorithm>
// forms of min / max / clamp written out below.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

#include "csg_engine.h"

#ifdef __CUDACC__
#define CSG_HD __host__ __device__
#else
#define CSG_HD
#endif
#ifdef __CUDA_ARCH__
#define CSG_FLOOR floor
#define CSG_ISFINITE isfinite
#else
#define CSG_FLOOR std::floor
#define CSG_ISFINITE std::isfinite
#endif

namespace csg_synth {

struct Flow {  // one (op instance, executing rank)
  double rs;      // the rank's start
  double rend;    // the rank's end (also when the instance stalls)
  int64_t gop;    // global op_seq
  uint64_t total; // chunks of the flow
  int32_t r;
  int32_t comm;
  uint8_t name;   // CSG_OP_*
  uint8_t stalls;
  uint8_t pad[6];
};

struct Params {
  double window, t_end, ack, hang_at, stop_logs_at;
  uint64_t msg_bytes;
  int32_t cpp, rank_lo, rank_hi, ranks_per_node, hang_node, hang_nic, nics_per_node, pad;
};

// std::min / std::max / std::clamp exactly as <algorithm> defines them
CSG_HD inline double dmin(double a, double b) { return b < a ? b : a; }
CSG_HD inline double dmax(double a, double b) { return a < b ? b : a; }
CSG_HD inline uint64_t umin(uint64_t a, uint64_t b) { return b < a ? b : a; }
CSG_HD inline double dclamp(double v, double lo, double hi) {
  return v < lo ? lo : (hi < v ? hi : v);
}

CSG_HD inline bool on_dead_nic(const Params& P, int32_t r, int ch) {
  return r / P.ranks_per_node == P.hang_node &&
         (P.hang_nic < 0 || ch % P.nics_per_node == P.hang_nic);
}

// The emit filter: the shard's ranks, logs of the failed node stop, the
// simulated horizon.
CSG_HD inline bool keep(const Params& P, double key, int32_t r) {
  if (r < P.rank_lo || r >= P.rank_hi) return false;
  if (CSG_ISFINITE(P.stop_logs_at) && key > P.stop_logs_at && r / P.ranks_per_node == P.hang_node)
    return false;
  return !(key > P.t_end);
}

CSG_HD inline csg_packed_record state_rec(const Flow& f, int ch, double ts, uint64_t rd,
                                          uint64_t tx, uint64_t dn) {
  csg_packed_record x;
  memset(&x, 0, sizeof(x));
  x.ts = ts;
  x.op_seq = f.gop;
  x.rank = f.r;
  x.comm_id = f.comm;
  x.channel = ch;
  x.kind = CSG_KIND_STATE;
  x.u.s.gpu_ready = static_cast<uint32_t>(rd);
  x.u.s.rdma_transmitted = static_cast<uint32_t>(tx);
  x.u.s.rdma_done = static_cast<uint32_t>(dn);
  return x;
}

// visit(key, record) for every record of channel ch of the flow, in the
// simulator's emission order.
template <class V>
CSG_HD inline void expand(const Params& P, const Flow& f, int ch, V&& visit) {
  const double cs = f.rs + 0.002 * ch;
  const double ce = f.stalls ? INFINITY : f.rend - 0.003 * (P.cpp - 1 - ch);
  const double span = dmax(1e-6, f.rend - cs);
  const uint64_t total = f.total;
  auto counters = [&](double t, uint64_t& rd, uint64_t& tx, uint64_t& dn) {
    double fr = (dmin(t, f.stalls ? P.hang_at : t) - cs) / span;
    fr = dclamp(fr, 0.0, 1.0);
    rd = umin(total, static_cast<uint64_t>(total * dmin(1.0, fr + 0.25)));
    tx = umin(rd, static_cast<uint64_t>(total * fr));
    dn = umin(tx, static_cast<uint64_t>(total * dmax(0.0, fr - 0.1)));
    if (f.stalls && on_dead_nic(P, f.r, ch) && tx > 0 && dn == tx) dn = tx - 1;
  };
  // periodic snapshots at window boundaries inside the flow
  const double stop = dmin(ce, P.t_end);
  for (double w = CSG_FLOOR(cs / P.window + 1) * P.window; w < stop; w += P.window) {
    uint64_t rd, tx, dn;
    counters(w, rd, tx, dn);
    visit(w, state_rec(f, ch, w, rd, tx, dn));
  }
  if (!f.stalls) {
    // flush snapshot at flow end, then the completion (end <= flush)
    const double flush = ce + P.ack;
    visit(flush, state_rec(f, ch, flush, total, total, total));
    csg_packed_record c;
    memset(&c, 0, sizeof(c));
    c.ts = ce;
    c.op_seq = f.gop;
    c.rank = f.r;
    c.comm_id = f.comm;
    c.channel = ch;
    c.kind = CSG_KIND_COMPLETION;
    c.op_name = f.name;
    c.u.c.start_ms = cs;
    c.u.c.msg_bytes = P.msg_bytes / P.cpp > 1 ? P.msg_bytes / P.cpp : 1;
    visit(flush, c);
  }
}

}  // namespace csg_synth

namespace csg {
// Device generator (synth_gpu.cu): expands the flows into records on the
// store's device, orders them by (emission time, emission sequence) and
// appends the first `target` (all when 0). Returns the records appended.
uint64_t synth_append_device(csg_store* store, const csg_synth::Flow* flows, size_t n_flows,
                             const csg_synth::Params& params, uint64_t target);
}  // namespace csg
