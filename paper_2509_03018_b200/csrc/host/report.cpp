// report.cpp — byte-exact renderings of the analyzer output: the JSONL
// report stream (reports_to_jsonl, proj/src/runner.cpp:103-169), the text
// rendering (reports_to_text, :171-209) and the analyze-mode summaries
// (summary_to_json / summary_to_text over a default SimSummary, :211-265).
// Doubles use std::to_chars' shortest round-trip form, integers decimal.
#include <charconv>
#include <fstream>

#include "host.h"

namespace csh {

namespace {

void num(std::string& out, double v) {
  char buf[64];
  auto [end, ec] = std::to_chars(buf, buf + sizeof(buf), v);
  (void)ec;
  out.append(buf, end);
}

const char* kTrigger[] = {"failure", "straggler"};
const char* kVerdict[] = {"suspects", "undetermined", "false_trigger",
                          "insufficient_history", "no_straggler"};
const char* kCategory[] = {"uninitialized_or_blocked",
                           "rdma_issue_or_receiver_not_ready",
                           "rdma_issue_or_receiver_failed",
                           "gpu_issue",
                           "straggler_late_start",
                           "straggler_late_end",
                           "flow_incomplete",
                           "flow_skewed"};
const char* kSide[] = {"local", "remote", "undetermined"};

const char* name_of(const char* const* table, int n, int v) {
  return v >= 0 && v < n ? table[v] : "?";
}

}  // namespace

std::string reports_to_jsonl(const std::vector<csg_report_view>& o,
                             const Scenario& s) {
  const std::optional<double> onset = s.first_onset();
  std::string out;
  for (const csg_report_view& r : o) {
    const char* kind = name_of(kTrigger, 2, r.trigger.kind);
    out += "{\"type\":\"trigger\",\"kind\":\"";
    out += kind;
    out += "\",\"suspect_rank\":" + std::to_string(r.trigger.suspect_rank);
    out += ",\"time_ms\":";
    num(out, r.trigger.time_ms);
    if (onset && r.trigger.time_ms >= *onset) {
      out += ",\"latency_ms\":";
      num(out, r.trigger.time_ms - *onset);
    }
    out += "}\n{\"type\":\"report\",\"time_ms\":";
    num(out, r.trigger.time_ms);
    out += ",\"trigger_kind\":\"";
    out += kind;
    out += "\",\"verdict\":\"";
    out += name_of(kVerdict, 5, r.verdict);
    out += "\",\"suspects\":[";
    for (size_t i = 0; i < r.n_suspects; ++i) {
      const csg_suspect& x = r.suspects[i];
      if (i) out += ",";
      out += "{\"rank\":" + std::to_string(x.rank) + ",\"category\":\"";
      out += name_of(kCategory, 8, x.category);
      out += "\",\"side\":\"";
      out += name_of(kSide, 3, x.side);
      out += "\",\"group\":" + std::to_string(x.group) +
             ",\"op_seq\":" + std::to_string(x.stuck_op) + ",\"onset_ms\":";
      num(out, x.onset_ms);
      out += "}";
    }
    out += "],\"affected_groups\":[";
    for (size_t i = 0; i < r.n_affected; ++i) {
      if (i) out += ",";
      out += std::to_string(r.affected_groups[i]);
    }
    out += "],\"evidence\":[";
    for (size_t i = 0; i < r.n_evidence; ++i) {
      const csg_evidence& e = r.evidence[i];
      if (i) out += ",";
      out += "{\"rank\":" + std::to_string(e.rank) +
             ",\"channel\":" + std::to_string(e.channel) + ",\"time_ms\":";
      num(out, e.time_ms);
      out += ",\"op_seq\":" + std::to_string(e.op_seq) + "}";
    }
    out += "],\"records_scanned\":" + std::to_string(r.records_scanned) + "}\n";
  }
  return out;
}

std::string reports_to_text(const std::vector<csg_report_view>& o,
                            const Scenario& s) {
  const std::optional<double> onset = s.first_onset();
  if (o.empty()) return "no triggers\n";
  std::string out;
  for (const csg_report_view& r : o) {
    out += "[t=";
    num(out, r.trigger.time_ms);
    out += " ms] ";
    out += name_of(kTrigger, 2, r.trigger.kind);
    out += " trigger on rank " + std::to_string(r.trigger.suspect_rank);
    if (onset && r.trigger.time_ms >= *onset) {
      out += " (";
      num(out, r.trigger.time_ms - *onset);
      out += " ms after fault onset)";
    }
    out += "\n  verdict: ";
    out += name_of(kVerdict, 5, r.verdict);
    out += "\n";
    for (size_t i = 0; i < r.n_suspects; ++i) {
      const csg_suspect& x = r.suspects[i];
      out += "  suspect rank " + std::to_string(x.rank) + ": ";
      out += name_of(kCategory, 8, x.category);
      out += " (side ";
      out += name_of(kSide, 3, x.side);
      out += ", group " + std::to_string(x.group) + ", op " +
             std::to_string(x.stuck_op) + ")\n";
    }
  }
  return out;
}

// run_analyze leaves the simulation summary default-constructed
// (proj/src/runner.cpp:92-101).
std::string analyze_summary_json(size_t triggers) {
  return "{\"completed\":false,\"end_ms\":0,\"events\":0,\"records\":0,"
         "\"triggers\":" +
         std::to_string(triggers) + ",\"rank_completion_ms\":[]}";
}

std::string analyze_summary_text() {
  return "simulated 0 ms, 0 events, 0 trace records, run stalled\n";
}

void write_file(const std::string& path, const std::string& content) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw ConfigError("cannot write file '" + path + "'");
  out << content;
  if (!out) throw ConfigError("write failed for '" + path + "'");
}

}  // namespace csh
