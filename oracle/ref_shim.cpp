// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (oracle). Never linked into the
// product. A thin extern "C" adapter over the UNMODIFIED reference collsight
// library (built from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libcollsight_ref.so) so the parity tests and bench.py's CPU
// baseline leg can drive the reference C++ API with the same packed records
// and tables the B200 engine receives.
//
// Reference entry points driven here:
//   run_detection      proj/src/runner.cpp:47-81
//   reports_to_jsonl   proj/src/runner.cpp:103-169
//   evaluate           proj/src/trigger.cpp:57-136
//   sample_ranks       proj/src/trigger.cpp:29-55
//   analyze*           proj/src/rca.cpp:540-884
//   affected_groups    proj/src/rca.cpp:400-461
//   TraceStore::query / last_log_per_rank  proj/src/trace.cpp:101-144
//   run_simulation (trace generator for fixtures) proj/src/sim.cpp:919-924
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <charconv>
#include <string>
#include <vector>

#include "collsight/collsight.h"
#include "collsight/rca.hpp"
#include "collsight/runner.hpp"
#include "collsight/scenario.hpp"
#include "collsight/sim.hpp"
#include "collsight/trace.hpp"
#include "collsight/trigger.hpp"
#include "csg_engine.h"

using namespace collsight;

namespace {

thread_local std::string g_err;

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

template <typename Fn>
int guard(Fn&& fn) {
  try {
    return fn();
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const TraceParseError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

// Packed -> reference record. `node` carries the store index so query()
// results (which return copies) can be mapped back to indices.
TraceRecord unpack(const csg_packed_record& p, std::size_t idx) {
  TraceRecord rec;
  if (p.kind == CSG_KIND_COMPLETION) {
    CompletionRecord c;
    c.node = static_cast<NodeId>(idx);
    c.comm_id = p.comm_id;
    c.rank = p.rank;
    c.channel = p.channel;
    c.op_seq = p.op_seq;
    c.op_name = static_cast<OpName>(p.op_name);
    c.msg_bytes = p.u.c.msg_bytes;
    c.start_ms = p.u.c.start_ms;
    c.end_ms = p.ts;
    rec.body = c;
  } else {
    StateRecord s;
    s.node = static_cast<NodeId>(idx);
    s.comm_id = p.comm_id;
    s.rank = p.rank;
    s.channel = p.channel;
    s.op_seq = p.op_seq;
    s.window_end_ms = p.ts;
    s.stuck_ms = 0;
    s.gpu_ready = p.u.s.gpu_ready;
    s.rdma_transmitted = p.u.s.rdma_transmitted;
    s.rdma_done = p.u.s.rdma_done;
    s.total_chunks = s.gpu_ready;
    rec.body = s;
  }
  return rec;
}

csg_packed_record pack(const TraceRecord& rec) {
  csg_packed_record p;
  std::memset(&p, 0, sizeof(p));
  if (const CompletionRecord* c = rec.completion()) {
    p.ts = c->end_ms;
    p.op_seq = c->op_seq;
    p.rank = c->rank;
    p.comm_id = c->comm_id;
    p.channel = c->channel;
    p.kind = CSG_KIND_COMPLETION;
    p.op_name = static_cast<uint8_t>(c->op_name);
    p.u.c.start_ms = c->start_ms;
    p.u.c.msg_bytes = c->msg_bytes;
  } else {
    const StateRecord* s = rec.state();
    p.ts = s->window_end_ms;
    p.op_seq = s->op_seq;
    p.rank = s->rank;
    p.comm_id = s->comm_id;
    p.channel = s->channel;
    p.kind = CSG_KIND_STATE;
    p.u.s.gpu_ready = static_cast<uint32_t>(s->gpu_ready);
    p.u.s.rdma_transmitted = static_cast<uint32_t>(s->rdma_transmitted);
    p.u.s.rdma_done = static_cast<uint32_t>(s->rdma_done);
  }
  return p;
}

TraceStore make_store(const csg_packed_record* recs, std::size_t n) {
  TraceStore store;
  for (std::size_t i = 0; i < n; ++i) store.append(unpack(recs[i], i));
  return store;
}

Topology make_topo(const csg_topology_desc* d) {
  Topology t;
  t.tp = d->world_size;
  t.pp = 1;
  t.dp = 1;
  t.ranks_per_node = 1;
  for (int32_t g = 0; g < d->n_groups; ++g) {
    CommGroup grp;
    grp.comm_id = g;
    grp.kind = static_cast<GroupKind>(d->group_kind[g]);
    for (int64_t i = d->member_off[g]; i < d->member_off[g + 1]; ++i)
      grp.members.push_back(d->members[i]);
    t.groups.push_back(std::move(grp));
  }
  return t;
}

OpProgram make_program(const csg_program_desc* d) {
  OpProgram p;
  for (int32_t i = 0; i < d->n_ops; ++i) {
    CollOpSpec op;
    op.op_seq = i;
    op.op_name = static_cast<OpName>(d->op_name[i]);
    op.group = d->group[i];
    op.msg_bytes = 1;
    op.src = d->src[i];
    op.dst = d->dst[i];
    for (int64_t k = d->dep_off[i]; k < d->dep_off[i + 1]; ++k)
      op.depends_on.push_back(d->deps[k]);
    p.ops.push_back(std::move(op));
  }
  return p;
}

TriggerConfig make_tcfg(const csg_trigger_config* c) {
  TriggerConfig t;
  t.delta_ms = c->delta_ms;
  t.detect_interval_ms = c->detect_interval_ms;
  t.throughput_drop_factor = c->throughput_drop_factor;
  t.interval_inflation_factor = c->interval_inflation_factor;
  t.max_sampled_ranks = c->max_sampled_ranks;
  t.ema_alpha = c->ema_alpha;
  t.warmup_windows = c->warmup_windows;
  return t;
}

AnalysisConfig make_acfg(const csg_analysis_config* c) {
  AnalysisConfig a;
  a.straggler_threshold_ms = c->straggler_threshold_ms;
  a.consecutive_iterations_k = c->consecutive_iterations_k;
  a.delta_ms = c->delta_ms;
  a.flow_skew_factor = c->flow_skew_factor;
  return a;
}

void num(std::string& out, double v) {
  char tmp[64];
  auto [p, ec] = std::to_chars(tmp, tmp + sizeof(tmp), v);
  (void)ec;
  out.append(tmp, p);
}

void entry(std::string& out, const SuspectEntry& s) {
  out += "{\"rank\":" + std::to_string(s.rank);
  out += ",\"category\":" + std::to_string(static_cast<int>(s.category));
  out += ",\"side\":" + std::to_string(static_cast<int>(s.side));
  out += ",\"group\":" + std::to_string(s.group);
  out += ",\"op_seq\":" + std::to_string(s.stuck_op);
  out += ",\"onset_ms\":";
  num(out, s.onset_ms);
  out += "}";
}

// Full structured report (exonerated included), one JSON object per line.
std::string full_report(const RootCauseReport& r) {
  std::string out = "{\"verdict\":" + std::to_string(static_cast<int>(r.verdict));
  out += ",\"kind\":" + std::to_string(static_cast<int>(r.trigger.kind));
  out += ",\"suspect_rank\":" + std::to_string(r.trigger.suspect_rank);
  out += ",\"time_ms\":";
  num(out, r.trigger.time_ms);
  out += ",\"suspects\":[";
  for (std::size_t i = 0; i < r.suspects.size(); ++i) {
    if (i) out += ",";
    entry(out, r.suspects[i]);
  }
  out += "],\"exonerated\":[";
  for (std::size_t i = 0; i < r.exonerated.size(); ++i) {
    if (i) out += ",";
    entry(out, r.exonerated[i]);
  }
  out += "],\"affected_groups\":[";
  for (std::size_t i = 0; i < r.affected_groups.size(); ++i) {
    if (i) out += ",";
    out += std::to_string(r.affected_groups[i]);
  }
  out += "],\"evidence\":[";
  for (std::size_t i = 0; i < r.evidence.size(); ++i) {
    const EvidenceRef& e = r.evidence[i];
    if (i) out += ",";
    out += "{\"rank\":" + std::to_string(e.rank) +
           ",\"channel\":" + std::to_string(e.channel) + ",\"time_ms\":";
    num(out, e.time_ms);
    out += ",\"op_seq\":" + std::to_string(e.op_seq) + "}";
  }
  out += "],\"records_scanned\":" + std::to_string(r.records_scanned) + "}\n";
  return out;
}

ScenarioConfig onset_cfg(int has_onset, double onset) {
  ScenarioConfig cfg;
  if (has_onset) {
    FaultSpec f;
    f.onset_ms = onset;
    cfg.faults.push_back(f);
  }
  return cfg;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

// Scenario-driven simulate: packed records in emission order (malloc'd).
int ref_simulate(const char* cfg_json, csg_packed_record** out, size_t* n,
                 char** jsonl) {
  return guard([&] {
    const ScenarioConfig cfg = parse_scenario(cfg_json);
    const RunResult run = run_simulate(cfg);
    *n = run.records.size();
    *out = static_cast<csg_packed_record*>(
        std::malloc(sizeof(csg_packed_record) * (run.records.size() + 1)));
    for (std::size_t i = 0; i < run.records.size(); ++i)
      (*out)[i] = pack(run.records[i]);
    if (jsonl) *jsonl = dup(serialize_records(run.records));
    return 0;
  });
}

// Program-driven simulate (a custom one-op AllReduce
// program is expressible only through the C++ API): layout, sim config and
// faults come from the scenario JSON, the program from `pd` with every op's
// msg_bytes set to `msg_bytes`. run_simulation: proj/include/collsight/
// sim.hpp:90.
int ref_simulate_prog(const char* cfg_json, const csg_program_desc* pd,
                      uint64_t msg_bytes, csg_packed_record** out, size_t* n) {
  return guard([&] {
    const ScenarioConfig cfg = parse_scenario(cfg_json);
    const Topology topo = cfg.build_topology();
    OpProgram program = make_program(pd);
    for (auto& op : program.ops) op.msg_bytes = msg_bytes;
    validate_program(program, topo);
    std::vector<TraceRecord> records;
    run_simulation(topo, program, cfg.faults, cfg.sim,
                   [&](const TraceRecord& r) { records.push_back(r); });
    *n = records.size();
    *out = static_cast<csg_packed_record*>(
        std::malloc(sizeof(csg_packed_record) * (records.size() + 1)));
    for (std::size_t i = 0; i < records.size(); ++i) (*out)[i] = pack(records[i]);
    return 0;
  });
}

// Scenario-driven detection over packed records. Returns reports_to_jsonl
// bytes and the full structured reports.
int ref_run_detection_cfg(const char* cfg_json, const csg_packed_record* recs,
                          size_t n, char** reports, char** full,
                          int32_t* sampled, size_t cap, size_t* n_sampled,
                          double* seconds) {
  return guard([&] {
    const ScenarioConfig cfg = parse_scenario(cfg_json);
    std::vector<TraceRecord> records;
    records.reserve(n);
    for (std::size_t i = 0; i < n; ++i) records.push_back(unpack(recs[i], i));
    const Topology topo = cfg.build_topology();
    const OpProgram program = cfg.build_program(topo);
    std::vector<RankId> s;
    const auto t0 = std::chrono::steady_clock::now();
    const auto outcomes = run_detection(records, topo, program, cfg, &s);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (reports) *reports = dup(reports_to_jsonl(outcomes, cfg));
    if (full) {
      std::string f;
      for (const auto& o : outcomes) f += full_report(o.report);
      *full = dup(f);
    }
    if (n_sampled) *n_sampled = s.size();
    for (std::size_t i = 0; i < s.size() && i < cap; ++i) sampled[i] = s[i];
    return 0;
  });
}

// Table-driven detection (hand-built topologies).
int ref_run_detection(const csg_topology_desc* td, const csg_program_desc* pd,
                      const csg_trigger_config* tc,
                      const csg_analysis_config* ac, uint64_t seed,
                      const csg_packed_record* recs, size_t n, int has_onset,
                      double onset, char** reports, char** full,
                      double* seconds) {
  return guard([&] {
    const Topology topo = make_topo(td);
    const OpProgram program = make_program(pd);
    ScenarioConfig cfg = onset_cfg(has_onset, onset);
    cfg.trigger = make_tcfg(tc);
    cfg.analysis = make_acfg(ac);
    cfg.sim.seed = seed;
    std::vector<TraceRecord> records;
    records.reserve(n);
    for (std::size_t i = 0; i < n; ++i) records.push_back(unpack(recs[i], i));
    const auto t0 = std::chrono::steady_clock::now();
    const auto outcomes = run_detection(records, topo, program, cfg, nullptr);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (reports) *reports = dup(reports_to_jsonl(outcomes, cfg));
    if (full) {
      std::string f;
      for (const auto& o : outcomes) f += full_report(o.report);
      *full = dup(f);
    }
    return 0;
  });
}

int ref_analyze(const csg_topology_desc* td, const csg_program_desc* pd,
                const csg_analysis_config* ac, const csg_packed_record* recs,
                size_t n, const csg_trigger_event* trig, int mode, char** full,
                double* seconds) {
  return guard([&] {
    const Topology topo = make_topo(td);
    const OpProgram program = make_program(pd);
    const TraceStore store = make_store(recs, n);
    AnalysisContext ctx;
    ctx.topo = &topo;
    ctx.program = &program;
    ctx.cfg = make_acfg(ac);
    TriggerEvent t{static_cast<TriggerKind>(trig->kind), trig->suspect_rank,
                   trig->time_ms};
    const auto t0 = std::chrono::steady_clock::now();
    RootCauseReport r = mode == 1   ? analyze_failure(store, ctx, t)
                        : mode == 2 ? analyze_straggler(store, ctx, t)
                                    : analyze(store, ctx, t);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    *full = dup(full_report(r));
    return 0;
  });
}

int ref_affected_groups(const csg_topology_desc* td,
                        const csg_program_desc* pd,
                        const csg_analysis_config* ac,
                        const csg_packed_record* recs, size_t n,
                        const csg_trigger_event* trig, int32_t* out,
                        size_t cap, size_t* n_out, uint64_t* scanned) {
  return guard([&] {
    const Topology topo = make_topo(td);
    const OpProgram program = make_program(pd);
    const TraceStore store = make_store(recs, n);
    AnalysisContext ctx;
    ctx.topo = &topo;
    ctx.program = &program;
    ctx.cfg = make_acfg(ac);
    TriggerEvent t{static_cast<TriggerKind>(trig->kind), trig->suspect_rank,
                   trig->time_ms};
    std::size_t sc = 0;
    const auto g = affected_groups(store, ctx, t, &sc);
    *n_out = g.size();
    for (std::size_t i = 0; i < g.size() && i < cap; ++i) out[i] = g[i];
    if (scanned) *scanned = sc;
    return 0;
  });
}

int ref_query(const csg_packed_record* recs, size_t n, const int32_t* ranks,
              size_t nr, double t0, double t1, uint64_t* out, size_t cap,
              size_t* n_out) {
  return guard([&] {
    const TraceStore store = make_store(recs, n);
    const auto q = store.query(std::span<const RankId>(ranks, nr), t0, t1);
    *n_out = q.size();
    for (std::size_t i = 0; i < q.size() && i < cap; ++i)
      out[i] = static_cast<uint64_t>(q[i].node());
    return 0;
  });
}

int ref_last_log_per_rank(const csg_packed_record* recs, size_t n,
                          const int32_t* members, size_t nm, double t,
                          int32_t* out_rank, uint64_t* out_idx,
                          size_t* n_out) {
  return guard([&] {
    const TraceStore store = make_store(recs, n);
    CommGroup g;
    g.members.assign(members, members + nm);
    const auto l = store.last_log_per_rank(g, t);
    *n_out = l.size();
    for (std::size_t i = 0; i < l.size(); ++i) {
      out_rank[i] = l[i].first;
      out_idx[i] = l[i].second;
    }
    return 0;
  });
}

void* ref_trigger_state_new(void) { return new TriggerState(); }
void ref_trigger_state_free(void* s) { delete static_cast<TriggerState*>(s); }

int ref_evaluate(const csg_packed_record* recs, size_t n,
                 const int32_t* sampled, size_t ns, double t, void* state,
                 const csg_trigger_config* tc, int* tripped,
                 csg_trigger_event* ev) {
  return guard([&] {
    const TraceStore store = make_store(recs, n);
    std::vector<RankId> s(sampled, sampled + ns);
    const auto r =
        evaluate(store, s, t, *static_cast<TriggerState*>(state), make_tcfg(tc));
    *tripped = r.has_value() ? 1 : 0;
    if (r) {
      ev->kind = static_cast<int32_t>(r->kind);
      ev->suspect_rank = r->suspect_rank;
      ev->time_ms = r->time_ms;
    }
    return 0;
  });
}

int ref_sample_ranks(const csg_topology_desc* td, int32_t max_sampled,
                     uint64_t seed, int32_t* out, size_t cap, size_t* n_out) {
  return guard([&] {
    const Topology topo = make_topo(td);
    TriggerConfig c;
    c.max_sampled_ranks = max_sampled;
    const auto s = sample_ranks(topo, c, seed);
    *n_out = s.size();
    for (std::size_t i = 0; i < s.size() && i < cap; ++i) out[i] = s[i];
    return 0;
  });
}

// Layout + default program as JSON, for building test tables from the
// reference's own build_layout/default_program (proj/src/topology.cpp:80,
// proj/src/program.cpp:25).
int ref_layout(int tp, int pp, int dp, int rpn, int cpp, int nics,
               uint64_t msg_bytes, char** json) {
  return guard([&] {
    const Topology topo = build_layout(tp, pp, dp, rpn, cpp, nics);
    const OpProgram prog = default_program(topo, msg_bytes);
    std::string o = "{\"world_size\":" + std::to_string(topo.world_size());
    o += ",\"groups\":[";
    for (std::size_t g = 0; g < topo.groups.size(); ++g) {
      if (g) o += ",";
      o += "{\"kind\":" + std::to_string(static_cast<int>(topo.groups[g].kind)) +
           ",\"members\":[";
      for (std::size_t i = 0; i < topo.groups[g].members.size(); ++i) {
        if (i) o += ",";
        o += std::to_string(topo.groups[g].members[i]);
      }
      o += "]}";
    }
    o += "],\"ops\":[";
    for (std::size_t i = 0; i < prog.ops.size(); ++i) {
      const CollOpSpec& op = prog.ops[i];
      if (i) o += ",";
      o += "{\"name\":" + std::to_string(static_cast<int>(op.op_name)) +
           ",\"group\":" + std::to_string(op.group) +
           ",\"src\":" + std::to_string(op.src) +
           ",\"dst\":" + std::to_string(op.dst) + ",\"deps\":[";
      for (std::size_t k = 0; k < op.depends_on.size(); ++k) {
        if (k) o += ",";
        o += std::to_string(op.depends_on[k]);
      }
      o += "]}";
    }
    o += "]}";
    *json = dup(o);
    return 0;
  });
}

int ref_check_min_op(const int32_t* ranks, const int64_t* ops, size_t n,
                     int32_t* out, size_t* n_out, int* has_min) {
  return guard([&] {
    std::vector<std::pair<RankId, OpSeq>> v;
    for (std::size_t i = 0; i < n; ++i) v.emplace_back(ranks[i], ops[i]);
    const auto r = check_min_op(v);
    *has_min = r.has_value() ? 1 : 0;
    *n_out = r ? r->size() : 0;
    if (r)
      for (std::size_t i = 0; i < r->size(); ++i) out[i] = (*r)[i];
    return 0;
  });
}

int ref_check_min_data(const int32_t* ranks, const csg_progress* p, size_t n,
                       int32_t* out, size_t* n_out) {
  return guard([&] {
    std::vector<std::pair<RankId, ProgressTriple>> v;
    for (std::size_t i = 0; i < n; ++i)
      v.emplace_back(ranks[i], ProgressTriple{p[i].gpu_ready,
                                              p[i].rdma_transmitted,
                                              p[i].rdma_done});
    const auto r = check_min_data(v);
    *n_out = r.size();
    for (std::size_t i = 0; i < r.size(); ++i) out[i] = r[i];
    return 0;
  });
}

int ref_check_rc_table(const csg_progress* c, const csg_progress* peer,
                       int* category, int* side) {
  return guard([&] {
    ProgressTriple a{c->gpu_ready, c->rdma_transmitted, c->rdma_done};
    ProgressTriple b;
    if (peer) b = ProgressTriple{peer->gpu_ready, peer->rdma_transmitted,
                                 peer->rdma_done};
    const auto r = check_rc_table(a, peer ? &b : nullptr);
    *category = static_cast<int>(r.first);
    *side = static_cast<int>(r.second);
    return 0;
  });
}

// ---- benchmark CPU leg: one store, many windows ----------------------------

void* ref_store_new(const csg_packed_record* recs, size_t n) {
  auto* st = new TraceStore();
  for (std::size_t i = 0; i < n; ++i) st->append(unpack(recs[i], i));
  return st;
}

void ref_store_free(void* s) { delete static_cast<TraceStore*>(s); }

// One detection window of the reference: evaluate at tick
// t with the scenario's sampled ranks (fresh trigger state), then analyze
// its trigger if it tripped. Times each phase separately.
int ref_window(void* store, const char* cfg_json, double t, double* eval_s,
               double* analyze_s, int* tripped, char** full) {
  return guard([&] {
    const ScenarioConfig cfg = parse_scenario(cfg_json);
    const Topology topo = cfg.build_topology();
    const OpProgram program = cfg.build_program(topo);
    const TraceStore& st = *static_cast<const TraceStore*>(store);
    const auto sampled = sample_ranks(topo, cfg.trigger, cfg.sim.seed);
    TriggerState state;
    const auto t0 = std::chrono::steady_clock::now();
    const auto trig = evaluate(st, sampled, t, state, cfg.trigger);
    const auto t1 = std::chrono::steady_clock::now();
    *eval_s = std::chrono::duration<double>(t1 - t0).count();
    *tripped = trig.has_value() ? 1 : 0;
    *analyze_s = 0;
    if (trig) {
      AnalysisContext ctx;
      ctx.topo = &topo;
      ctx.program = &program;
      ctx.cfg = cfg.analysis;
      const auto t2 = std::chrono::steady_clock::now();
      const RootCauseReport r = analyze(st, ctx, *trig);
      const auto t3 = std::chrono::steady_clock::now();
      *analyze_s = std::chrono::duration<double>(t3 - t2).count();
      if (full) *full = dup(full_report(r));
    }
    return 0;
  });
}

}  // extern "C"
