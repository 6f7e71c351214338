// trace_io.cpp — JSONL trace ingest into packed records.
//
// Accepts and rejects exactly what the reference's parse_trace_text /
// parse_record accept (proj/src/trace.cpp:241-337): one JSON object per
// line, empty lines skipped but counted, unknown fields rejected, missing
// fields named with the 1-based line number, record invariants checked
// (validate_record, trace.cpp:39-57) and reported as a TraceParseError.
// Fields the analyzer never reads (node, stuck_ms, total_chunks) are checked
// and then dropped; state counters must fit the packed u32 lanes.
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>

#include <json.hpp>

#include "host.h"

namespace csh {

namespace {

using nlohmann::json;

const json& need(const json& j, const char* key, int line) {
  auto it = j.find(key);
  if (it == j.end())
    throw TraceParseError(line, std::string("missing field '") + key + "'");
  return *it;
}

const char* kCompletion[] = {"type",    "node",    "comm_id",   "rank",
                             "channel", "op_seq",  "op_name",   "msg_bytes",
                             "start_ms", "end_ms"};
const char* kState[] = {"type",         "node",      "comm_id",
                        "rank",         "channel",   "op_seq",
                        "window_end_ms", "stuck_ms", "total_chunks",
                        "gpu_ready",    "rdma_transmitted", "rdma_done"};
const char* kOpNames[] = {"AllGather", "ReduceScatter", "AllReduce", "Send",
                          "Recv"};

template <size_t N>
void reject_unknown(const json& j, const char* (&allowed)[N], int line) {
  for (auto it = j.begin(); it != j.end(); ++it) {
    bool ok = false;
    for (const char* f : allowed)
      if (it.key() == f) {
        ok = true;
        break;
      }
    if (!ok) throw TraceParseError(line, "unknown field '" + it.key() + "'");
  }
}

csg_packed_record parse_line(std::string_view text, int line) {
  json j = json::parse(text, nullptr, false);
  if (j.is_discarded()) throw TraceParseError(line, "not valid JSON");
  if (!j.is_object()) throw TraceParseError(line, "record is not an object");
  const std::string type = need(j, "type", line).get<std::string>();
  csg_packed_record p;
  std::memset(&p, 0, sizeof(p));
  if (type == "completion") {
    reject_unknown(j, kCompletion, line);
    need(j, "node", line).get<int32_t>();
    p.comm_id = need(j, "comm_id", line).get<int32_t>();
    p.rank = need(j, "rank", line).get<int32_t>();
    p.channel = need(j, "channel", line).get<int>();
    p.op_seq = need(j, "op_seq", line).get<int64_t>();
    const std::string name = need(j, "op_name", line).get<std::string>();
    int op = -1;
    for (int k = 0; k < 5; ++k)
      if (name == kOpNames[k]) op = k;
    if (op < 0) throw TraceParseError(line, "unknown op_name '" + name + "'");
    const uint64_t bytes = need(j, "msg_bytes", line).get<uint64_t>();
    const double start = need(j, "start_ms", line).get<double>();
    const double end = need(j, "end_ms", line).get<double>();
    if (end < start)
      throw TraceParseError(line, "completion record with end_ms < start_ms");
    if (bytes == 0) throw TraceParseError(line, "completion record with msg_bytes 0");
    if (p.rank < 0 || p.channel < 0)
      throw TraceParseError(line, "completion record with negative rank or channel");
    p.kind = CSG_KIND_COMPLETION;
    p.op_name = static_cast<uint8_t>(op);
    p.ts = end;
    p.u.c.start_ms = start;
    p.u.c.msg_bytes = bytes;
  } else if (type == "state") {
    reject_unknown(j, kState, line);
    need(j, "node", line).get<int32_t>();
    p.comm_id = need(j, "comm_id", line).get<int32_t>();
    p.rank = need(j, "rank", line).get<int32_t>();
    p.channel = need(j, "channel", line).get<int>();
    p.op_seq = need(j, "op_seq", line).get<int64_t>();
    const double wend = need(j, "window_end_ms", line).get<double>();
    const double stuck = need(j, "stuck_ms", line).get<double>();
    const uint64_t total = need(j, "total_chunks", line).get<uint64_t>();
    const uint64_t ready = need(j, "gpu_ready", line).get<uint64_t>();
    const uint64_t tx = need(j, "rdma_transmitted", line).get<uint64_t>();
    const uint64_t done = need(j, "rdma_done", line).get<uint64_t>();
    if (!(total >= ready && ready >= tx && tx >= done))
      throw TraceParseError(line,
                            "state record violates total >= gpu_ready >= "
                            "rdma_transmitted >= rdma_done");
    if (stuck < 0) throw TraceParseError(line, "state record with negative stuck_ms");
    if (p.rank < 0 || p.channel < 0)
      throw TraceParseError(line, "state record with negative rank or channel");
    if (ready > 0xffffffffull)
      throw TraceParseError(line,
                            "state counter exceeds the packed format's 2^32-1");
    p.kind = CSG_KIND_STATE;
    p.ts = wend;
    p.u.s.gpu_ready = static_cast<uint32_t>(ready);
    p.u.s.rdma_transmitted = static_cast<uint32_t>(tx);
    p.u.s.rdma_done = static_cast<uint32_t>(done);
  } else {
    throw TraceParseError(line, "unknown record type '" + type + "'");
  }
  return p;
}

}  // namespace

std::vector<csg_packed_record> parse_trace_text(std::string_view text) {
  std::vector<csg_packed_record> out;
  // multithreaded fast path for valid traces (fast_jsonl.cpp); anything it
  // does not fully vouch for is parsed again below with the exact grammar
  // and error reporting
  static const bool exact_only = std::getenv("CSG_JSONL_EXACT") != nullptr;
  if (!exact_only && fast_parse_trace(text, out)) return out;
  out.clear();
  int line = 0;
  size_t pos = 0;
  while (pos < text.size()) {
    size_t eol = text.find('\n', pos);
    if (eol == std::string_view::npos) eol = text.size();
    ++line;
    if (eol > pos) out.push_back(parse_line(text.substr(pos, eol - pos), line));
    pos = eol + 1;
  }
  return out;
}

std::vector<csg_packed_record> load_trace_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw TraceParseError(0, "cannot open trace file '" + path + "'");
  std::ostringstream ss;
  ss << in.rdbuf();
  return parse_trace_text(ss.str());
}

}  // namespace csh
