// synth.cpp — fast synthetic trace generator for the benchmark shapes.
//
// The reference's discrete-event simulator (proj/src/sim.cpp, out of scope
// here) produces ~2e5 records/s single-threaded, too slow for the 1e7-1e9
// record benchmark traces. This generator reproduces the record PATTERN the
// analyzer consumes, not the simulator's timing algebra:
//   * the scenario's layout + default program, iterated;
//   * every op instance starts when its dependencies and each executing
//     rank's previous op have ended (the DepIndex DAG, rca.cpp:99-119), and
//     lasts a ring-algorithm transfer time at the configured bandwidth, with
//     a small deterministic per-rank jitter (counter-based mix64 hash);
//   * per executing rank and channel: one state record per state-log window
//     boundary the flow spans, a flush state record at the flow's end and
//     then the completion record whose end_ms precedes the flush (the
//     simulator's emission pattern, sim.cpp:687-706, which makes per-rank
//     store order non-monotone in time);
//   * faults: nic_shutdown stalls every instance in flight on the node at
//     onset (and everything downstream of it); members of a stalled instance
//     keep logging frozen counters, the failed node stops logging after
//     stop_logs_after_ms; bandwidth/pcie/power faults slow the target's
//     transfers by their factor after onset.
// Records are emitted in global event-time order. Deterministic per seed.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <unordered_map>
#include <vector>

#include "host.h"
#include "synth_flow.h"

namespace csh {

namespace {

inline uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
inline double unit(uint64_t a, uint64_t b, uint64_t c) {
  return static_cast<double>(mix(a ^ mix(b ^ mix(c))) >> 11) * 0x1.0p-53;
}

struct Rec {
  double key;      // emission time
  uint64_t seq;    // tie-break: emission sequence
  csg_packed_record r;
};

}  // namespace

SynthPlan synth_plan(const Scenario& sc, uint64_t target, int32_t rank_lo, int32_t rank_hi) {
  const Layout l = sc.layout();
  const Program p = sc.program(l);
  const int opn = static_cast<int>(p.ops.size());
  const int W = l.world();
  const int cpp = l.channels_per_pair;
  const double window = sc.state_log_window_ms;
  const double t_end = sc.max_sim_ms;
  const double bw = sc.link_bandwidth;
  const double intra = sc.intra_bandwidth > 0 ? sc.intra_bandwidth : 10.0 * bw;
  // executing ranks per op
  std::vector<std::vector<int32_t>> ex(opn);
  for (int s = 0; s < opn; ++s) {
    const Op& op = p.ops[s];
    if (op.name == CSG_OP_SEND) ex[s] = {op.src};
    else if (op.name == CSG_OP_RECV) ex[s] = {op.dst};
    else ex[s] = l.members[op.group];
  }
  // per-op transfer time (ring algorithm), ms
  std::vector<double> base_dur(opn);
  std::vector<uint64_t> chunks(opn);
  for (int s = 0; s < opn; ++s) {
    const Op& op = p.ops[s];
    const auto& m = l.members[op.group];
    const double n = static_cast<double>(m.size());
    const bool intra_node = op.name != CSG_OP_SEND && op.name != CSG_OP_RECV &&
                            m.front() / l.ranks_per_node == m.back() / l.ranks_per_node;
    const double b = intra_node ? intra : bw;
    double steps = 1, bytes = static_cast<double>(sc.msg_bytes);
    if (op.name == CSG_OP_ALLREDUCE) {
      steps = 2 * (n - 1);
      bytes /= n;
    } else if (op.name != CSG_OP_SEND && op.name != CSG_OP_RECV) {
      steps = n - 1;
      bytes /= n;
    }
    base_dur[s] = steps * (bytes / b + sc.link_latency_ms);
    const double per_flow = bytes / cpp;
    chunks[s] = std::max<uint64_t>(
        1, static_cast<uint64_t>(std::ceil(per_flow / static_cast<double>(sc.chunk_bytes)))) *
                static_cast<uint64_t>(std::max(1.0, steps));
  }
  // faults
  double hang_at = INFINITY, stop_logs_at = INFINITY;
  int hang_node = -1, hang_nic = -1;
  std::vector<double> slow_onset(W, INFINITY), slow_factor(W, 1.0);
  for (const Fault& f : sc.faults) {
    if (f.kind == 0) {  // nic_shutdown
      if (f.onset_ms < hang_at) {
        hang_at = f.onset_ms;
        hang_node = f.target == 2 ? f.rank / l.ranks_per_node : f.node;
        hang_nic = f.target == 1 ? f.nic : -1;
        if (f.stop_logs_after_ms > 0) stop_logs_at = f.onset_ms + f.stop_logs_after_ms;
      }
    } else if (f.kind >= 1 && f.kind <= 5) {  // slowdowns
      // The reference simulator (sim.cpp:770-792) slows copies for
      // pcie_downgrade / gpu_power_limit / background_compute (copy_factor)
      // and flows for the NIC kinds (bandwidth_factor); this schedule has
      // one per-rank slowdown, so it takes whichever factor was set.
      const double fac = std::min(f.copy_factor, f.bandwidth_factor);
      for (int r = 0; r < W; ++r) {
        const bool hit = f.target == 2 ? r == f.rank : r / l.ranks_per_node == f.node;
        if (hit) {
          slow_onset[r] = std::min(slow_onset[r], f.onset_ms);
          slow_factor[r] = std::min(slow_factor[r], fac);
        }
      }
    }
  }
  auto on_dead_nic = [&](int32_t r, int ch) {
    return r / l.ranks_per_node == hang_node &&
           (hang_nic < 0 || ch % l.nics_per_node == hang_nic);
  };
  std::vector<double> ready(W, 0.0);      // rank free at
  std::vector<char> blocked(W, 0);        // rank waits forever
  std::vector<double> op_end(opn, 0.0);   // this iteration's end per op
  std::vector<char> op_stalled(opn, 0);
  SynthPlan plan;
  csg_synth::Params& P = plan.params;
  P.window = window;
  P.t_end = t_end;
  P.ack = sc.ack_latency_ms;
  P.hang_at = hang_at;
  P.stop_logs_at = stop_logs_at;
  P.msg_bytes = sc.msg_bytes;
  P.cpp = cpp;
  P.rank_lo = rank_lo;
  P.rank_hi = rank_hi;
  P.ranks_per_node = l.ranks_per_node;
  P.hang_node = hang_node;
  P.hang_nic = hang_nic;
  P.nics_per_node = l.nics_per_node;
  P.pad = 0;
  plan.target = target;
  uint64_t emitted = 0;  // records that pass the emit filter (the target cut)
  auto count = [&](const csg_synth::Flow& f) {
    for (int ch = 0; ch < cpp; ++ch)
      csg_synth::expand(P, f, ch, [&](double key, const csg_packed_record& r) {
        if (csg_synth::keep(P, key, r.rank)) ++emitted;
      });
  };
  const int iters = sc.iterations > 0 ? sc.iterations : 1;
  for (int it = 0; it < iters; ++it) {
    bool any_started = false;
    for (int s = 0; s < opn; ++s) {
      const Op& op = p.ops[s];
      const int64_t gop = static_cast<int64_t>(it) * opn + s;
      // start: deps end + executing ranks free
      double start = 0;
      bool blk = false;
      for (int64_t d : op.deps) {
        start = std::max(start, op_end[d]);
        blk |= op_stalled[d] != 0;
      }
      for (int32_t r : ex[s]) {
        start = std::max(start, ready[r]);
        blk |= blocked[r] != 0;
      }
      // Rendezvous: a send starts only once its receiver is free for the
      // matching receive (which depends on this send), so no stage runs
      // ahead of the pipeline, and a receiver that waits forever blocks it.
      if (op.name == CSG_OP_SEND && op.dst >= 0 && op.dst < W) {
        start = std::max(start, ready[op.dst]);
        blk |= blocked[op.dst] != 0;
      }
      if (blk || start > t_end) {
        op_stalled[s] = 1;
        for (int32_t r : ex[s]) blocked[r] = 1;
        op_end[s] = INFINITY;
        continue;
      }
      any_started = true;
      // does this instance hang?
      bool touches_dead = false;
      if (hang_node >= 0)
        for (int32_t r : ex[s])
          for (int ch = 0; ch < cpp; ++ch) touches_dead |= on_dead_nic(r, ch);
      double dur = base_dur[s];
      double inst_end = start;
      std::vector<double> rend(ex[s].size());
      for (size_t i = 0; i < ex[s].size(); ++i) {
        const int32_t r = ex[s][i];
        double d = dur * (1.0 + 0.04 * unit(sc.seed, gop, r));
        if (start >= slow_onset[r]) d /= slow_factor[r];
        rend[i] = start + d;
        inst_end = std::max(inst_end, rend[i]);
      }
      const bool stalls = touches_dead && inst_end > hang_at;
      for (size_t i = 0; i < ex[s].size(); ++i) {
        const int32_t r = ex[s][i];
        csg_synth::Flow f;
        std::memset(&f, 0, sizeof(f));
        f.rs = start + 0.01 * unit(sc.seed ^ 7, gop, r);
        f.rend = rend[i];
        f.gop = gop;
        f.total = chunks[s];
        f.r = r;
        f.comm = op.group;
        f.name = op.name;
        f.stalls = stalls ? 1 : 0;
        // flows of other shards' ranks emit nothing: not kept
        if (r >= rank_lo && r < rank_hi) {
          plan.flows.push_back(f);
          if (target) count(f);
        }
        ready[r] = stalls ? INFINITY : rend[i];
        if (stalls) blocked[r] = 1;
      }
      op_stalled[s] = stalls ? 1 : 0;
      op_end[s] = stalls ? INFINITY : inst_end;
    }
    if (!any_started) break;
    if (target && emitted >= target + target / 16) break;
  }
  return plan;
}

std::vector<csg_packed_record> synthesize(const Scenario& sc, uint64_t target,
                                          int32_t rank_lo, int32_t rank_hi) {
  const SynthPlan plan = synth_plan(sc, target, rank_lo, rank_hi);
  const csg_synth::Params& P = plan.params;
  std::vector<Rec> out;
  out.reserve(target ? target + target / 8 : 1 << 20);
  uint64_t seq = 0;
  for (const csg_synth::Flow& f : plan.flows)
    for (int ch = 0; ch < P.cpp; ++ch)
      csg_synth::expand(P, f, ch, [&](double key, const csg_packed_record& r) {
        if (csg_synth::keep(P, key, r.rank)) out.push_back(Rec{key, seq++, r});
      });
  std::sort(out.begin(), out.end(), [](const Rec& a, const Rec& b) {
    return a.key != b.key ? a.key < b.key : a.seq < b.seq;
  });
  if (target && out.size() > target) out.resize(target);
  std::vector<csg_packed_record> recs(out.size());
  for (size_t i = 0; i < out.size(); ++i) recs[i] = out[i].r;
  return recs;
}

}  // namespace csh
