// host.h — host-side C++ of the drop-in library: scenario configs, layout +
// program tables, the JSONL trace codec and report rendering. None of this
// is on the analysis hot path; it prepares the engine's tables and turns its
// results into the reference's byte-exact text formats.
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "csg_engine.h"
#include "synth_flow.h"

namespace csh {

// Error taxonomy of the reference (proj/include/collsight/types.hpp:46-75),
// mapped to statuses 2 / 3 / 4 at the C API.
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct TraceParseError : std::runtime_error {
  TraceParseError(int line, const std::string& what)
      : std::runtime_error("line " + std::to_string(line) + ": " + what) {}
};
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Layout {
  int tp = 1, pp = 1, dp = 1, ranks_per_node = 1, channels_per_pair = 1,
      nics_per_node = 4;
  std::vector<uint8_t> kind;                 // per comm_id
  std::vector<std::vector<int32_t>> members; // ring order
  int world() const { return tp * pp * dp; }
  int nodes() const { return world() / ranks_per_node; }
};

struct Op {
  uint8_t name = CSG_OP_ALLGATHER;
  int32_t group = -1;
  int32_t src = -1, dst = -1;
  std::vector<int64_t> deps;
};

struct Program {
  std::vector<Op> ops;
};

Layout build_layout(int tp, int pp, int dp, int ranks_per_node,
                    int channels_per_pair, int nics_per_node);
Program default_program(const Layout& l, uint64_t msg_bytes);
void validate_program(const Program& p, const Layout& l);

struct Fault {
  int kind = 0;
  int target = 0;  // 0 node, 1 nic, 2 rank
  int32_t node = -1, nic = -1, rank = -1;
  double onset_ms = 0, bandwidth_factor = 1, copy_factor = 1, delay_ms = 0,
         delay_prob = 0, stop_logs_after_ms = 0;
};

struct Scenario {
  int tp = 1, pp = 1, dp = 1, ranks_per_node = 1, channels_per_pair = 1,
      nics_per_node = 4;
  // SimConfig (proj/include/collsight/sim.hpp:16-29): validated, not run
  uint64_t chunk_bytes = 4ull * 1024 * 1024;
  double link_bandwidth = 4194304.0, intra_bandwidth = 0.0,
         link_latency_ms = 0.05, ack_latency_ms = 0.02, copy_rate = 4194304.0,
         reduce_factor = 1.0, state_log_window_ms = 100.0, max_sim_ms = 60000.0;
  uint64_t seed = 0;
  int iterations = 1;
  size_t buffer_capacity = 16384;
  uint64_t msg_bytes = 64ull * 1024 * 1024;
  csg_trigger_config trigger;
  csg_analysis_config analysis;
  std::vector<Fault> faults;

  Layout layout() const;
  Program program(const Layout& l) const;
  std::optional<double> first_onset() const;
};

Scenario parse_scenario(const std::string& json_text);
Scenario load_scenario_file(const std::string& path);

// Synthetic benchmark traces (synth.cpp). target = 0: no record cap.
// Only records of ranks in [rank_lo, rank_hi) are emitted (a shard's view;
// the schedule is still simulated for every rank).
std::vector<csg_packed_record> synthesize(const Scenario& s, uint64_t target,
                                          int32_t rank_lo = 0,
                                          int32_t rank_hi = 0x7fffffff);
// The schedule half of it: one Flow per (op instance, executing rank) of
// the shard, in emission order, plus the expansion parameters (the device
// generator expands them, synth_gpu.cu).
struct SynthPlan {
  std::vector<csg_synth::Flow> flows;
  csg_synth::Params params;
  uint64_t target = 0;
};
SynthPlan synth_plan(const Scenario& s, uint64_t target, int32_t rank_lo, int32_t rank_hi);

// Trace codec.
// Multithreaded parse of a valid trace; false when the exact parser must
// decide (fast_jsonl.cpp).
bool fast_parse_trace(std::string_view text, std::vector<csg_packed_record>& out);
std::vector<csg_packed_record> parse_trace_text(std::string_view text);
std::vector<csg_packed_record> load_trace_file(const std::string& path);
// packed records -> reference-format JSONL (serialize.cpp)
std::string serialize_packed(const csg_packed_record* recs, size_t n, int32_t ranks_per_node);

// Report rendering over engine results.
struct Outcome {
  csg_report_view r;
};
std::string reports_to_jsonl(const std::vector<csg_report_view>& o,
                             const Scenario& s);
std::string reports_to_text(const std::vector<csg_report_view>& o,
                            const Scenario& s);
std::string analyze_summary_json(size_t triggers);
std::string analyze_summary_text();
void write_file(const std::string& path, const std::string& content);
std::string layout_json(const Layout& l, const Program& p);

// Engine tables of a layout/program (keeps the arrays alive).
struct Tables {
  std::vector<uint8_t> kind;
  std::vector<int64_t> member_off;
  std::vector<int32_t> members;
  std::vector<uint8_t> op_name;
  std::vector<int32_t> group, src, dst;
  std::vector<int64_t> dep_off, deps;
  csg_topology_desc topo;
  csg_program_desc prog;
  Tables(const Layout& l, const Program& p);
};

}  // namespace csh
