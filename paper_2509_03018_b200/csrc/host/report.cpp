// report.cpp — byte-exact renderings of the analyzer output: the JSONL
// report stream (reports_to_jsonl, proj/src/runner.cpp:103-169), the text
// rendering (reports_to_text, :171-209) and the analyze-mode summaries
// (summary_to_json / summary_to_text over a default SimSummary, :211-265).
// Doubles use std::to_chars' shortest round-trip form, integers decimal.
#include <algorithm>
#include <atomic>
#include <charconv>
#include <fstream>
#include <thread>

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

// One report's trigger + report lines. Integers and doubles go straight
// into the output through std::to_chars (no temporaries): the evidence list
// of a hang report runs to thousands of entries.
void report_jsonl(std::string& out, const csg_report_view& r,
                  const std::optional<double>& onset) {
  auto lit = [&](const char* s) { out.append(s); };
  auto i64 = [&](long long v) {
    char buf[24];
    auto [end, ec] = std::to_chars(buf, buf + sizeof(buf), v);
    (void)ec;
    out.append(buf, end);
  };
  const char* kind = name_of(kTrigger, 2, r.trigger.kind);
  lit("{\"type\":\"trigger\",\"kind\":\"");
  lit(kind);
  lit("\",\"suspect_rank\":");
  i64(r.trigger.suspect_rank);
  lit(",\"time_ms\":");
  num(out, r.trigger.time_ms);
  if (onset && r.trigger.time_ms >= *onset) {
    lit(",\"latency_ms\":");
    num(out, r.trigger.time_ms - *onset);
  }
  lit("}\n{\"type\":\"report\",\"time_ms\":");
  num(out, r.trigger.time_ms);
  lit(",\"trigger_kind\":\"");
  lit(kind);
  lit("\",\"verdict\":\"");
  lit(name_of(kVerdict, 5, r.verdict));
  lit("\",\"suspects\":[");
  for (size_t i = 0; i < r.n_suspects; ++i) {
    const csg_suspect& x = r.suspects[i];
    if (i) out.push_back(',');
    lit("{\"rank\":");
    i64(x.rank);
    lit(",\"category\":\"");
    lit(name_of(kCategory, 8, x.category));
    lit("\",\"side\":\"");
    lit(name_of(kSide, 3, x.side));
    lit("\",\"group\":");
    i64(x.group);
    lit(",\"op_seq\":");
    i64(x.stuck_op);
    lit(",\"onset_ms\":");
    num(out, x.onset_ms);
    out.push_back('}');
  }
  lit("],\"affected_groups\":[");
  for (size_t i = 0; i < r.n_affected; ++i) {
    if (i) out.push_back(',');
    i64(r.affected_groups[i]);
  }
  lit("],\"evidence\":[");
  for (size_t i = 0; i < r.n_evidence; ++i) {
    const csg_evidence& e = r.evidence[i];
    if (i) out.push_back(',');
    lit("{\"rank\":");
    i64(e.rank);
    lit(",\"channel\":");
    i64(e.channel);
    lit(",\"time_ms\":");
    num(out, e.time_ms);
    lit(",\"op_seq\":");
    i64(e.op_seq);
    out.push_back('}');
  }
  lit("],\"records_scanned\":");
  out.append(std::to_string(r.records_scanned));
  lit("}\n");
}

}  // namespace

// Reports are rendered independently (one thread each when the batch is
// large) and concatenated in trigger order.
std::string reports_to_jsonl(const std::vector<csg_report_view>& o,
                             const Scenario& s) {
  const std::optional<double> onset = s.first_onset();
  size_t items = 0;
  for (const csg_report_view& r : o) items += r.n_evidence + r.n_affected + r.n_suspects;
  std::string out;
  if (o.size() < 2 || items < 20000) {
    out.reserve(items * 64 + o.size() * 256);
    for (const csg_report_view& r : o) report_jsonl(out, r, onset);
    return out;
  }
  std::vector<std::string> part(o.size());
  const unsigned T = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(),
                                                     static_cast<unsigned>(o.size())));
  std::atomic<size_t> next{0};
  auto work = [&] {
    for (size_t i; (i = next.fetch_add(1)) < o.size();) {
      const csg_report_view& r = o[i];
      part[i].reserve((r.n_evidence + r.n_affected + r.n_suspects) * 64 + 256);
      report_jsonl(part[i], r, onset);
    }
  };
  std::vector<std::thread> th;
  for (unsigned t = 1; t < T; ++t) th.emplace_back(work);
  work();
  for (auto& x : th) x.join();
  size_t total = 0;
  for (const auto& p : part) total += p.size();
  out.reserve(total);
  for (const auto& p : part) out += p;
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
