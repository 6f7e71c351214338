// serialize.cpp — packed records -> JSONL trace text in the reference's
// format (serialize_record / serialize_records, proj/src/trace.cpp:189-
// 322: fixed key order, integers and doubles through std::to_chars, the
// double in its shortest round-trip form), multithreaded (SURVEY.md §8(f)
// row 4: the reference serializes at ~0.73 us/record on one core).
//
// The packed record drops three fields the analyzer never reads (node,
// stuck_ms, total_chunks; csg_engine.h). They are written as node = rank /
// ranks_per_node (the simulator's placement), stuck_ms = 0 and total_chunks
// = gpu_ready, which satisfy validate_record, so parse(serialize(r)) == r
// for every packed record (doubles: shortest form + correctly rounded parse).
#include <charconv>
#include <cstring>
#include <thread>

#include "host.h"

namespace csh {

namespace {

const char* op_text(uint8_t op) {
  static const char* names[] = {"AllGather", "ReduceScatter", "AllReduce", "Send", "Recv"};
  return op < 5 ? names[op] : "AllGather";
}

struct Out {
  char* p;
  template <typename T>
  void num(T v) {
    p = std::to_chars(p, p + 32, v).ptr;
  }
  void lit(const char* s) {
    const size_t n = std::strlen(s);
    std::memcpy(p, s, n);
    p += n;
  }
};

// one record, '\n'-terminated, into dst (>= 384 bytes); returns the end
char* write_record(const csg_packed_record& r, int32_t rpn, char* dst) {
  Out o{dst};
  const int64_t node = rpn > 0 ? r.rank / rpn : 0;
  if (r.kind == CSG_KIND_COMPLETION) {
    o.lit("{\"type\":\"completion\",\"node\":");
    o.num(node);
    o.lit(",\"comm_id\":");
    o.num(static_cast<int64_t>(r.comm_id));
    o.lit(",\"rank\":");
    o.num(static_cast<int64_t>(r.rank));
    o.lit(",\"channel\":");
    o.num(static_cast<int64_t>(r.channel));
    o.lit(",\"op_seq\":");
    o.num(r.op_seq);
    o.lit(",\"op_name\":\"");
    o.lit(op_text(r.op_name));
    o.lit("\",\"msg_bytes\":");
    o.num(r.u.c.msg_bytes);
    o.lit(",\"start_ms\":");
    o.num(r.u.c.start_ms);
    o.lit(",\"end_ms\":");
    o.num(r.ts);
    o.lit("}\n");
  } else {
    o.lit("{\"type\":\"state\",\"node\":");
    o.num(node);
    o.lit(",\"comm_id\":");
    o.num(static_cast<int64_t>(r.comm_id));
    o.lit(",\"rank\":");
    o.num(static_cast<int64_t>(r.rank));
    o.lit(",\"channel\":");
    o.num(static_cast<int64_t>(r.channel));
    o.lit(",\"op_seq\":");
    o.num(r.op_seq);
    o.lit(",\"window_end_ms\":");
    o.num(r.ts);
    o.lit(",\"stuck_ms\":0,\"total_chunks\":");
    o.num(static_cast<uint64_t>(r.u.s.gpu_ready));
    o.lit(",\"gpu_ready\":");
    o.num(static_cast<uint64_t>(r.u.s.gpu_ready));
    o.lit(",\"rdma_transmitted\":");
    o.num(static_cast<uint64_t>(r.u.s.rdma_transmitted));
    o.lit(",\"rdma_done\":");
    o.num(static_cast<uint64_t>(r.u.s.rdma_done));
    o.lit("}\n");
  }
  return o.p;
}

}  // namespace

std::string serialize_packed(const csg_packed_record* recs, size_t n, int32_t rpn) {
  unsigned T = std::max(1u, std::thread::hardware_concurrency());
  if (n < (1u << 14)) T = 1;
  T = static_cast<unsigned>(std::min<size_t>(T, std::max<size_t>(1, n / 4096)));
  std::vector<std::string> parts(T);
  auto work = [&](unsigned t) {
    const size_t b = n * t / T, e = n * (t + 1) / T;
    std::string& s = parts[t];
    s.resize((e - b) * 384 + 16);
    char* p = s.data();
    for (size_t i = b; i < e; ++i) p = write_record(recs[i], rpn, p);
    s.resize(static_cast<size_t>(p - s.data()));
  };
  if (T == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t) th.emplace_back(work, t);
    for (auto& x : th) x.join();
  }
  size_t total = 0;
  for (auto& s : parts) total += s.size();
  std::string out;
  out.reserve(total);
  for (auto& s : parts) out += s;
  return out;
}

}  // namespace csh
