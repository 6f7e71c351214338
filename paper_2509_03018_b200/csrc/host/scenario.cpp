// scenario.cpp — JSON scenario configs, accepted and rejected exactly like
// the reference's parse_scenario (proj/src/scenario.cpp:84-147) including
// its derived defaults (trigger.delta_ms = 2 * state_log_window_ms,
// analysis.delta_ms = trigger.delta_ms) and every precondition check it runs
// through ScenarioConfig::validate (scenario.cpp:74-82: layout, SimConfig,
// TriggerConfig, AnalysisConfig, msg_bytes, faults, program).
//
// JSON parsing uses nlohmann/json, the library the reference itself uses at
// this boundary, so type errors surface with identical messages.
#include <fstream>
#include <sstream>

#include <json.hpp>

#include "host.h"

namespace csh {

namespace {

using nlohmann::json;

const json& field(const json& j, const char* key, const std::string& where) {
  auto it = j.find(key);
  if (it == j.end())
    throw ConfigError(where + ": missing field '" + key + "'");
  return *it;
}

template <typename T>
void maybe(const json& j, const char* key, T& out) {
  auto it = j.find(key);
  if (it != j.end()) out = it->get<T>();
}

const char* kFaultKinds[] = {"nic_shutdown",     "nic_bandwidth_limit",
                             "pcie_downgrade",   "gpu_power_limit",
                             "background_compute", "background_traffic",
                             "proxy_delay"};

Fault fault_from(const json& j, size_t idx) {
  const std::string where = "faults[" + std::to_string(idx) + "]";
  Fault f;
  const std::string kind = field(j, "kind", where).get<std::string>();
  f.kind = -1;
  for (int k = 0; k < 7; ++k)
    if (kind == kFaultKinds[k]) f.kind = k;
  if (f.kind < 0)
    throw ConfigError(where + ": unknown fault kind '" + kind + "'");
  f.onset_ms = field(j, "onset_ms", where).get<double>();
  if (j.contains("rank")) {
    f.target = 2;
    f.rank = j.at("rank").get<int32_t>();
  } else if (j.contains("nic")) {
    f.target = 1;
    if (!j.contains("node")) throw ConfigError(where + ": nic target needs 'node'");
    f.node = j.at("node").get<int32_t>();
    f.nic = j.at("nic").get<int>();
  } else if (j.contains("node")) {
    f.target = 0;
    f.node = j.at("node").get<int32_t>();
  } else {
    throw ConfigError(where +
                      ": needs a target ('rank', 'node', or 'node'+'nic')");
  }
  maybe(j, "bandwidth_factor", f.bandwidth_factor);
  maybe(j, "copy_factor", f.copy_factor);
  maybe(j, "delay_ms", f.delay_ms);
  maybe(j, "delay_prob", f.delay_prob);
  maybe(j, "stop_logs_after_ms", f.stop_logs_after_ms);
  return f;
}

void check_sim(const Scenario& s) {  // SimConfig::validate, sim.cpp:14-27
  if (s.chunk_bytes == 0) throw ConfigError("sim: chunk_bytes must be > 0");
  if (s.link_bandwidth <= 0) throw ConfigError("sim: link_bandwidth must be > 0");
  if (s.intra_bandwidth < 0) throw ConfigError("sim: intra_bandwidth must be >= 0");
  if (s.link_latency_ms <= 0) throw ConfigError("sim: link_latency_ms must be > 0");
  if (s.ack_latency_ms <= 0) throw ConfigError("sim: ack_latency_ms must be > 0");
  if (s.copy_rate <= 0) throw ConfigError("sim: copy_rate must be > 0");
  if (s.reduce_factor < 0) throw ConfigError("sim: reduce_factor must be >= 0");
  if (s.state_log_window_ms <= 0)
    throw ConfigError("sim: state_log_window_ms must be > 0");
  if (s.max_sim_ms <= 0) throw ConfigError("sim: max_sim_ms must be > 0");
  if (s.iterations < 0) throw ConfigError("sim: iterations must be >= 0");
  if (s.buffer_capacity == 0) throw ConfigError("sim: buffer_capacity must be > 0");
}

void check_trigger(const csg_trigger_config& t) {  // trigger.cpp:9-23
  if (t.delta_ms <= 0) throw ConfigError("trigger: delta_ms must be > 0");
  if (t.detect_interval_ms <= 0)
    throw ConfigError("trigger: detect_interval_ms must be > 0");
  if (t.throughput_drop_factor <= 0 || t.throughput_drop_factor >= 1)
    throw ConfigError("trigger: throughput_drop_factor must be in (0,1)");
  if (t.interval_inflation_factor <= 1)
    throw ConfigError("trigger: interval_inflation_factor must be > 1");
  if (t.max_sampled_ranks < 1)
    throw ConfigError("trigger: max_sampled_ranks must be >= 1");
  if (t.ema_alpha <= 0 || t.ema_alpha > 1)
    throw ConfigError("trigger: ema_alpha must be in (0,1]");
  if (t.warmup_windows < 1)
    throw ConfigError("trigger: warmup_windows must be >= 1");
}

void check_analysis(const csg_analysis_config& a) {  // rca.cpp:63-71
  if (a.straggler_threshold_ms <= 0)
    throw ConfigError("analysis: straggler_threshold_ms must be > 0");
  if (a.consecutive_iterations_k < 1)
    throw ConfigError("analysis: consecutive_iterations_k must be >= 1");
  if (a.delta_ms <= 0) throw ConfigError("analysis: delta_ms must be > 0");
  if (a.flow_skew_factor <= 1)
    throw ConfigError("analysis: flow_skew_factor must be > 1");
}

void check_faults(const Scenario& s, const Layout& l) {  // sim.cpp:54-90
  for (const Fault& f : s.faults) {
    if (f.onset_ms < 0) throw ConfigError("fault: onset_ms must be >= 0");
    if (f.bandwidth_factor <= 0 || f.bandwidth_factor > 1)
      throw ConfigError("fault: bandwidth_factor must be in (0,1]");
    if (f.copy_factor <= 0 || f.copy_factor > 1)
      throw ConfigError("fault: copy_factor must be in (0,1]");
    if (f.delay_prob < 0 || f.delay_prob > 1)
      throw ConfigError("fault: delay_prob must be in [0,1]");
    if (f.delay_ms < 0) throw ConfigError("fault: delay_ms must be >= 0");
    if (f.stop_logs_after_ms < 0)
      throw ConfigError("fault: stop_logs_after_ms must be >= 0");
    const int nodes = l.nodes();
    if (f.target == 0) {
      if (f.node < 0 || f.node >= nodes)
        throw ConfigError("fault: node target " + std::to_string(f.node) +
                          " does not exist");
    } else if (f.target == 1) {
      if (f.node < 0 || f.node >= nodes)
        throw ConfigError("fault: nic target on unknown node " +
                          std::to_string(f.node));
      if (f.nic < 0 || f.nic >= l.nics_per_node)
        throw ConfigError("fault: nic index " + std::to_string(f.nic) +
                          " does not exist on node " + std::to_string(f.node));
    } else {
      if (f.rank < 0 || f.rank >= l.world())
        throw ConfigError("fault: rank target " + std::to_string(f.rank) +
                          " does not exist");
    }
  }
}

}  // namespace

Layout Scenario::layout() const {
  return build_layout(tp, pp, dp, ranks_per_node, channels_per_pair,
                      nics_per_node);
}

Program Scenario::program(const Layout& l) const {
  return default_program(l, msg_bytes);
}

std::optional<double> Scenario::first_onset() const {
  std::optional<double> o;
  for (const Fault& f : faults)
    if (!o || f.onset_ms < *o) o = f.onset_ms;
  return o;
}

Scenario parse_scenario(const std::string& text) {
  json j = json::parse(text, nullptr, false);
  if (j.is_discarded()) throw ConfigError("config: not valid JSON");
  Scenario s;
  csg_trigger_config_default(&s.trigger);
  csg_analysis_config_default(&s.analysis);
  const json& lay = field(j, "layout", "config");
  s.tp = field(lay, "tp", "layout").get<int>();
  s.pp = field(lay, "pp", "layout").get<int>();
  s.dp = field(lay, "dp", "layout").get<int>();
  s.ranks_per_node = field(lay, "ranks_per_node", "layout").get<int>();
  s.channels_per_pair = field(lay, "channels_per_pair", "layout").get<int>();
  maybe(lay, "nics_per_node", s.nics_per_node);
  if (j.contains("sim")) {
    const json& sim = j.at("sim");
    maybe(sim, "chunk_bytes", s.chunk_bytes);
    maybe(sim, "link_bandwidth", s.link_bandwidth);
    maybe(sim, "intra_bandwidth", s.intra_bandwidth);
    maybe(sim, "link_latency_ms", s.link_latency_ms);
    maybe(sim, "ack_latency_ms", s.ack_latency_ms);
    maybe(sim, "copy_rate", s.copy_rate);
    maybe(sim, "reduce_factor", s.reduce_factor);
    maybe(sim, "state_log_window_ms", s.state_log_window_ms);
    maybe(sim, "max_sim_ms", s.max_sim_ms);
    maybe(sim, "buffer_capacity", s.buffer_capacity);
  }
  maybe(j, "msg_bytes", s.msg_bytes);
  s.iterations = field(j, "iterations", "config").get<int>();
  s.seed = field(j, "seed", "config").get<uint64_t>();
  s.trigger.delta_ms = 2.0 * s.state_log_window_ms;
  if (j.contains("trigger")) {
    const json& t = j.at("trigger");
    maybe(t, "delta_ms", s.trigger.delta_ms);
    maybe(t, "detect_interval_ms", s.trigger.detect_interval_ms);
    maybe(t, "throughput_drop_factor", s.trigger.throughput_drop_factor);
    maybe(t, "interval_inflation_factor", s.trigger.interval_inflation_factor);
    maybe(t, "max_sampled_ranks", s.trigger.max_sampled_ranks);
    maybe(t, "ema_alpha", s.trigger.ema_alpha);
    maybe(t, "warmup_windows", s.trigger.warmup_windows);
  }
  s.analysis.delta_ms = s.trigger.delta_ms;
  if (j.contains("analysis")) {
    const json& a = j.at("analysis");
    maybe(a, "straggler_threshold_ms", s.analysis.straggler_threshold_ms);
    maybe(a, "consecutive_iterations_k", s.analysis.consecutive_iterations_k);
    maybe(a, "delta_ms", s.analysis.delta_ms);
    maybe(a, "flow_skew_factor", s.analysis.flow_skew_factor);
  }
  if (j.contains("faults")) {
    const json& fs = j.at("faults");
    if (!fs.is_array()) throw ConfigError("config: 'faults' must be a list");
    for (size_t i = 0; i < fs.size(); ++i) s.faults.push_back(fault_from(fs[i], i));
  }
  // ScenarioConfig::validate order
  const Layout l = s.layout();
  check_sim(s);
  check_trigger(s.trigger);
  check_analysis(s.analysis);
  if (s.msg_bytes == 0) throw ConfigError("msg_bytes must be > 0");
  check_faults(s, l);
  validate_program(s.program(l), l);
  return s;
}

Scenario load_scenario_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ConfigError("cannot open config file '" + path + "'");
  std::ostringstream ss;
  ss << in.rdbuf();
  return parse_scenario(ss.str());
}

}  // namespace csh
