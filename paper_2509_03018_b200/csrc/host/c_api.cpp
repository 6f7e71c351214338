// c_api.cpp — collsight.h / collsight_b200.h over the B200 engine.
//
// Conventions of the reference C API (proj/src/c_api.cpp:27-158): opaque
// handles, thread-local last-error text, ConfigError -> 2, TraceParseError
// -> 3, any other failure -> 4, NULL arguments -> 5 before any work.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime_api.h>

#include "collsight.h"
#include "collsight_b200.h"
#include "host.h"

struct collsight_scenario {
  csh::Scenario cfg;
};

struct collsight_result {
  std::string summary_json;
  std::string reports_jsonl;
  uint64_t triggers = 0;
  // reports_to_text (+ the run summary) is rendered on the first
  // collsight_result_text call, from the reports kept here: the same bytes
  // as the reference's eager rendering, not paid by callers that only read
  // the JSONL reports
  csh::Scenario cfg;
  csg_results* res = nullptr;
  std::once_flag text_once;
  std::string text;
  ~collsight_result() { csg_results_free(res); }
  const std::string& text_view() {
    std::call_once(text_once, [&] {
      std::vector<csg_report_view> views(res ? csg_results_count(res) : 0);
      for (size_t i = 0; i < views.size(); ++i) csg_results_get(res, i, &views[i]);
      text = csh::reports_to_text(views, cfg) + csh::analyze_summary_text();
    });
    return text;
  }
};

namespace {

thread_local std::string g_last_error;

collsight_status fail(collsight_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

template <typename Fn>
collsight_status guarded(Fn&& fn) {
  try {
    return fn();
  } catch (const csh::ConfigError& e) {
    return fail(COLLSIGHT_ERR_CONFIG, e.what());
  } catch (const csh::TraceParseError& e) {
    return fail(COLLSIGHT_ERR_TRACE_PARSE, e.what());
  } catch (const std::exception& e) {
    return fail(COLLSIGHT_ERR_RUNTIME, e.what());
  }
}

// Engine status -> the same C++ error class the reference would raise.
void check(csg_status s) {
  if (s == CSG_OK) return;
  const std::string msg = csg_last_error();
  if (s == CSG_ERR_CONFIG) throw csh::ConfigError(msg);
  throw std::runtime_error(msg);
}

// One engine context per process (device from COLLSIGHT_B200_DEVICE, else
// 0); calls through the C API serialize on it.
std::mutex g_mu;
csg_ctx* g_ctx = nullptr;

csg_ctx* engine() {
  if (!g_ctx) {
    const char* d = std::getenv("COLLSIGHT_B200_DEVICE");
    check(csg_ctx_create(d ? std::atoi(d) : 0, &g_ctx));
  }
  return g_ctx;
}

// Device store + layout tables kept across calls, so repeated replays reuse
// their HBM allocations (the model is rebuilt only when the layout changes).
csg_store* g_store = nullptr;
csg_model* g_model = nullptr;
std::string g_model_key;

struct Results {
  csg_results* res = nullptr;
  ~Results() { csg_results_free(res); }
};

// Fills the (cleared) device store: packed records, or a JSONL trace file
// parsed on the device (falling back to the exact host parser, which raises
// the reference's TraceParseError, when the device parser defers).
struct StoreInput {
  const csg_packed_record* recs = nullptr;
  size_t n = 0;
  const char* jsonl_path = nullptr;
};

void fill_store(csg_store* store, const StoreInput& in) {
  if (!in.jsonl_path) {
    check(csg_store_append(store, in.recs, in.n));
    return;
  }
  const bool host_only = std::getenv("CSG_JSONL_HOST") != nullptr;  // A/B switch
  int accepted = 0;
  if (!host_only) check(csg_store_append_jsonl_file(store, in.jsonl_path, &accepted));
  if (accepted) return;
  const std::vector<csg_packed_record> recs = csh::load_trace_file(in.jsonl_path);
  check(csg_store_clear(store));
  check(csg_store_append(store, recs.data(), recs.size()));
}

collsight_result* analyze_records(const csh::Scenario& cfg, const StoreInput& in,
                                  const char* report_out_path) {
  std::lock_guard<std::mutex> lk(g_mu);
  csg_ctx* ctx = nullptr;
  try {
    ctx = engine();
  } catch (...) {
    // no usable device: a bad trace is still reported first, as the
    // reference's load_trace_file would
    if (in.jsonl_path) (void)csh::load_trace_file(in.jsonl_path);
    throw;
  }
  // CSG_E2E_PROF=1: wall time of each phase on stderr
  static const bool prof = std::getenv("CSG_E2E_PROF") != nullptr;
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  // the trace first (load_trace_file precedes the layout in the reference's
  // run_analyze path, so a bad trace is reported before a bad layout)
  if (!g_store) check(csg_store_create(ctx, &g_store));
  check(csg_store_clear(g_store));
  fill_store(g_store, in);
  const std::string key = std::to_string(cfg.tp) + "," + std::to_string(cfg.pp) +
                          "," + std::to_string(cfg.dp) + "," +
                          std::to_string(cfg.ranks_per_node) + "," +
                          std::to_string(cfg.channels_per_pair) + "," +
                          std::to_string(cfg.nics_per_node) + "," +
                          std::to_string(cfg.msg_bytes);
  if (!g_model || key != g_model_key) {
    const csh::Layout layout = cfg.layout();
    const csh::Program program = cfg.program(layout);
    const csh::Tables tables(layout, program);
    if (g_model) csg_model_free(g_model);
    g_model = nullptr;
    check(csg_model_create(ctx, &tables.topo, &tables.prog, &g_model));
    g_model_key = key;
  }
  if (prof) cudaDeviceSynchronize();
  const auto t1 = clk::now();
  Results e;
  check(csg_run_detection(g_store, g_model, &cfg.trigger, &cfg.analysis,
                          cfg.seed, &e.res, nullptr, 0, nullptr));
  const auto t2 = clk::now();
  std::vector<csg_report_view> views(csg_results_count(e.res));
  for (size_t i = 0; i < views.size(); ++i) check(csg_results_get(e.res, i, &views[i]));
  auto out = std::make_unique<collsight_result>();
  out->reports_jsonl = csh::reports_to_jsonl(views, cfg);
  const auto t3 = clk::now();
  out->cfg = cfg;
  out->res = e.res;  // the result handle owns the reports from here on
  e.res = nullptr;
  out->summary_json = csh::analyze_summary_json(views.size());
  out->triggers = views.size();
  if (report_out_path) csh::write_file(report_out_path, out->reports_jsonl);
  const auto t4 = clk::now();
  if (prof) {
    auto ms = [](clk::time_point a, clk::time_point b) {
      return std::chrono::duration<double, std::milli>(b - a).count();
    };
    std::fprintf(stderr,
                 "[e2e] append %.3f ms, run_detection %.3f ms, jsonl %.3f ms, summary+file "
                 "%.3f ms (%zu reports, %zu jsonl bytes)\n",
                 ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), views.size(),
                 out->reports_jsonl.size());
  }
  return out.release();
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

}  // namespace

extern "C" {

const char* collsight_version(void) { return "0.1.0"; }

const char* collsight_last_error(void) { return g_last_error.c_str(); }

collsight_status collsight_scenario_load(const char* path,
                                         collsight_scenario** out) {
  if (!path || !out) return fail(COLLSIGHT_ERR_ARG, "null argument");
  return guarded([&] {
    *out = new collsight_scenario{csh::load_scenario_file(path)};
    return COLLSIGHT_OK;
  });
}

collsight_status collsight_scenario_parse(const char* json_text,
                                          collsight_scenario** out) {
  if (!json_text || !out) return fail(COLLSIGHT_ERR_ARG, "null argument");
  return guarded([&] {
    *out = new collsight_scenario{csh::parse_scenario(json_text)};
    return COLLSIGHT_OK;
  });
}

collsight_status collsight_scenario_set_seed(collsight_scenario* s,
                                             uint64_t seed) {
  if (!s) return fail(COLLSIGHT_ERR_ARG, "null scenario");
  s->cfg.seed = seed;
  return COLLSIGHT_OK;
}

void collsight_scenario_free(collsight_scenario* s) { delete s; }

collsight_status collsight_run_simulate(const collsight_scenario* s,
                                        const char* trace_out_path,
                                        collsight_result** out) {
  (void)trace_out_path;
  if (!s || !out) return fail(COLLSIGHT_ERR_ARG, "null argument");
  return fail(COLLSIGHT_ERR_RUNTIME,
              "collsight-b200: the trace simulator is not part of this build; "
              "use collsight_run_analyze on a recorded trace");
}

collsight_status collsight_run_e2e(const collsight_scenario* s,
                                   const char* report_out_path,
                                   collsight_result** out) {
  (void)report_out_path;
  if (!s || !out) return fail(COLLSIGHT_ERR_ARG, "null argument");
  return fail(COLLSIGHT_ERR_RUNTIME,
              "collsight-b200: the trace simulator is not part of this build; "
              "use collsight_run_analyze on a recorded trace");
}

collsight_status collsight_run_analyze(const collsight_scenario* s,
                                       const char* trace_in_path,
                                       const char* report_out_path,
                                       collsight_result** out) {
  if (!s || !trace_in_path || !out)
    return fail(COLLSIGHT_ERR_ARG, "null argument");
  return guarded([&] {
    StoreInput in;
    in.jsonl_path = trace_in_path;
    *out = analyze_records(s->cfg, in, report_out_path);
    return COLLSIGHT_OK;
  });
}

const char* collsight_result_text(const collsight_result* r) {
  return r ? const_cast<collsight_result*>(r)->text_view().c_str() : "";
}
const char* collsight_result_summary_json(const collsight_result* r) {
  return r ? r->summary_json.c_str() : "";
}
const char* collsight_result_reports_jsonl(const collsight_result* r) {
  return r ? r->reports_jsonl.c_str() : "";
}
uint64_t collsight_result_trigger_count(const collsight_result* r) {
  return r ? r->triggers : 0;
}
void collsight_result_free(collsight_result* r) { delete r; }

collsight_status collsight_b200_run_analyze_packed(
    const collsight_scenario* s, const csg_packed_record* records, size_t n,
    const char* report_out_path, collsight_result** out) {
  if (!s || (!records && n) || !out) return fail(COLLSIGHT_ERR_ARG, "null argument");
  return guarded([&] {
    StoreInput in;
    in.recs = records;
    in.n = n;
    *out = analyze_records(s->cfg, in, report_out_path);
    return COLLSIGHT_OK;
  });
}

collsight_status collsight_b200_scenario_layout_json(const collsight_scenario* s,
                                                     char** json_out) {
  if (!s || !json_out) return fail(COLLSIGHT_ERR_ARG, "null argument");
  return guarded([&] {
    const csh::Layout l = s->cfg.layout();
    *json_out = dup(csh::layout_json(l, s->cfg.program(l)));
    return COLLSIGHT_OK;
  });
}

collsight_status collsight_b200_scenario_configs(const collsight_scenario* s,
                                                 csg_trigger_config* trigger,
                                                 csg_analysis_config* analysis,
                                                 uint64_t* seed) {
  if (!s) return fail(COLLSIGHT_ERR_ARG, "null argument");
  if (trigger) *trigger = s->cfg.trigger;
  if (analysis) *analysis = s->cfg.analysis;
  if (seed) *seed = s->cfg.seed;
  return COLLSIGHT_OK;
}

collsight_status collsight_b200_results_jsonl(const collsight_scenario* s,
                                              const csg_results* res, char** jsonl_out) {
  if (!s || !res || !jsonl_out) return fail(COLLSIGHT_ERR_ARG, "null argument");
  return guarded([&] {
    std::vector<csg_report_view> views(csg_results_count(res));
    for (size_t i = 0; i < views.size(); ++i) check(csg_results_get(res, i, &views[i]));
    *jsonl_out = dup(csh::reports_to_jsonl(views, s->cfg));
    return COLLSIGHT_OK;
  });
}

collsight_status collsight_b200_layout_json(int tp, int pp, int dp, int rpn,
                                            int cpp, int nics,
                                            uint64_t msg_bytes,
                                            char** json_out) {
  if (!json_out) return fail(COLLSIGHT_ERR_ARG, "null argument");
  return guarded([&] {
    const csh::Layout l = csh::build_layout(tp, pp, dp, rpn, cpp, nics);
    *json_out = dup(csh::layout_json(l, csh::default_program(l, msg_bytes)));
    return COLLSIGHT_OK;
  });
}

collsight_status collsight_b200_parse_trace(const char* text, size_t len,
                                            csg_packed_record** out,
                                            size_t* n) {
  if ((!text && len) || !out || !n) return fail(COLLSIGHT_ERR_ARG, "null argument");
  return guarded([&] {
    const auto v = csh::parse_trace_text(std::string_view(text, len));
    *n = v.size();
    *out = static_cast<csg_packed_record*>(
        std::malloc(sizeof(csg_packed_record) * (v.size() + 1)));
    if (!v.empty()) std::memcpy(*out, v.data(), v.size() * sizeof(csg_packed_record));
    return COLLSIGHT_OK;
  });
}

collsight_status collsight_b200_serialize_trace(const csg_packed_record* records,
                                                size_t n, int32_t ranks_per_node,
                                                char** text, size_t* len) {
  if ((!records && n) || !text || !len) return fail(COLLSIGHT_ERR_ARG, "null argument");
  return guarded([&] {
    const std::string s = csh::serialize_packed(records, n, ranks_per_node);
    *text = dup(s);
    *len = s.size();
    return COLLSIGHT_OK;
  });
}

collsight_status collsight_b200_write_trace(const csg_packed_record* records, size_t n,
                                            int32_t ranks_per_node, const char* path) {
  if ((!records && n) || !path) return fail(COLLSIGHT_ERR_ARG, "null argument");
  return guarded([&] {
    csh::write_file(path, csh::serialize_packed(records, n, ranks_per_node));
    return COLLSIGHT_OK;
  });
}

void collsight_b200_free(void* p) { std::free(p); }

collsight_status collsight_b200_engine_context(csg_ctx** out) {
  if (!out) return fail(COLLSIGHT_ERR_ARG, "null argument");
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_mu);
    *out = engine();
    return COLLSIGHT_OK;
  });
}

collsight_status collsight_b200_synthesize(const collsight_scenario* s,
                                           uint64_t target,
                                           csg_packed_record** out, size_t* n) {
  return collsight_b200_synthesize_ranks(s, target, 0, 0x7fffffff, out, n);
}

collsight_status collsight_b200_synthesize_ranks(const collsight_scenario* s,
                                                 uint64_t target, int32_t rank_lo,
                                                 int32_t rank_hi,
                                                 csg_packed_record** out, size_t* n) {
  if (!s || !out || !n) return fail(COLLSIGHT_ERR_ARG, "null argument");
  return guarded([&] {
    const auto v = csh::synthesize(s->cfg, target, rank_lo, rank_hi);
    *n = v.size();
    *out = static_cast<csg_packed_record*>(
        std::malloc(sizeof(csg_packed_record) * (v.size() + 1)));
    if (!v.empty()) std::memcpy(*out, v.data(), v.size() * sizeof(csg_packed_record));
    return COLLSIGHT_OK;
  });
}

collsight_status collsight_b200_synthesize_store(const collsight_scenario* s,
                                                 uint64_t target, int32_t rank_lo,
                                                 int32_t rank_hi, csg_store* store,
                                                 uint64_t* n) {
  if (!s || !store || !n) return fail(COLLSIGHT_ERR_ARG, "null argument");
  return guarded([&] {
    const csh::SynthPlan plan = csh::synth_plan(s->cfg, target, rank_lo, rank_hi);
    *n = csg::synth_append_device(store, plan.flows.data(), plan.flows.size(), plan.params,
                                  target);
    return COLLSIGHT_OK;
  });
}

}  // extern "C"
