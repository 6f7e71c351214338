// fast_jsonl.cpp — multithreaded JSONL -> packed-record parser for valid
// traces (the reference's nlohmann-based
// parse_trace_text, proj/src/trace.cpp:241-337, runs at ~33 MB/s).
//
// The text is split at line boundaries into one chunk per hardware thread;
// each thread parses its lines with a schema-specialised scanner:
//   * one flat JSON object per line, keys without escapes, values that are
//     plain JSON numbers or short strings;
//   * integers through std::from_chars (range-checked to the field's type),
//     doubles through std::from_chars (correctly rounded, the same value
//     nlohmann's strtod-based parser produces);
//   * the record invariants of validate_record (trace.cpp:39-57).
// Anything else — a duplicate or unknown key, a missing field, an escape, a
// float in an integer field, a value out of range, an invariant violation,
// malformed JSON — makes the fast path give up, and the caller re-parses the
// whole text with the exact parser (trace_io.cpp), which then reports the
// reference's error message and line number, or accepts what only the exact
// JSON grammar accepts. Valid input therefore yields exactly the records of
// the exact parser.
#include <algorithm>
#include <charconv>
#include <cstring>
#include <thread>

#include "host.h"

namespace csh {

namespace {

struct Cursor {
  const char* p;
  const char* e;
  void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n')) ++p;
  }
  bool lit(char c) {
    ws();
    if (p < e && *p == c) {
      ++p;
      return true;
    }
    return false;
  }
  // "key" without escapes
  bool str(std::string_view& out) {
    ws();
    if (p >= e || *p != '"') return false;
    const char* s = ++p;
    while (p < e && *p != '"') {
      if (*p == '\\' || static_cast<unsigned char>(*p) < 0x20) return false;
      ++p;
    }
    if (p >= e) return false;
    out = std::string_view(s, p - s);
    ++p;
    return true;
  }
  // raw JSON number token [-]digits[.digits][e[+-]digits]
  bool num(std::string_view& tok, bool& is_int) {
    ws();
    const char* s = p;
    if (p < e && *p == '-') ++p;
    if (p >= e || *p < '0' || *p > '9') return false;
    if (*p == '0' && p + 1 < e && p[1] >= '0' && p[1] <= '9') return false;  // leading zero
    while (p < e && *p >= '0' && *p <= '9') ++p;
    is_int = true;
    if (p < e && *p == '.') {
      is_int = false;
      ++p;
      if (p >= e || *p < '0' || *p > '9') return false;
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    if (p < e && (*p == 'e' || *p == 'E')) {
      is_int = false;
      ++p;
      if (p < e && (*p == '+' || *p == '-')) ++p;
      if (p >= e || *p < '0' || *p > '9') return false;
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    tok = std::string_view(s, p - s);
    return true;
  }
};

enum Field : int {
  F_TYPE, F_NODE, F_COMM, F_RANK, F_CHAN, F_OP, F_OPNAME, F_BYTES, F_START, F_END,
  F_WEND, F_STUCK, F_TOTAL, F_READY, F_TX, F_DONE, F_N
};

int field_of(std::string_view k) {
  static const char* names[F_N] = {"type",     "node",          "comm_id",  "rank",
                                   "channel",  "op_seq",        "op_name",  "msg_bytes",
                                   "start_ms", "end_ms",        "window_end_ms",
                                   "stuck_ms", "total_chunks",  "gpu_ready",
                                   "rdma_transmitted",          "rdma_done"};
  for (int f = 0; f < F_N; ++f)
    if (k == names[f]) return f;
  return -1;
}

template <typename T>
bool to_int(std::string_view tok, bool is_int, T& out) {
  if (!is_int) return false;
  const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), out);
  return r.ec == std::errc() && r.ptr == tok.data() + tok.size();
}

bool to_double(std::string_view tok, double& out) {
  // an integer token "-0" is integer 0 to nlohmann (+0.0 as a double);
  // leave that one to the exact parser
  if (tok.size() >= 2 && tok[0] == '-' &&
      tok.find_first_not_of('0', 1) == std::string_view::npos)
    return false;
  const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), out);
  return r.ec == std::errc() && r.ptr == tok.data() + tok.size();
}

// One line -> record; false on anything the exact parser must decide.
bool parse_one(const char* b, const char* e, csg_packed_record& rec) {
  Cursor c{b, e};
  if (!c.lit('{')) return false;
  std::string_view tok[F_N];
  bool isint[F_N] = {};
  std::string_view sval[F_N];
  uint32_t seen = 0;
  if (!c.lit('}')) {
    do {
      std::string_view key;
      if (!c.str(key)) return false;
      const int f = field_of(key);
      if (f < 0 || (seen >> f) & 1u) return false;  // unknown / duplicate
      if (!c.lit(':')) return false;
      c.ws();
      if (c.p < c.e && *c.p == '"') {
        if (f != F_TYPE && f != F_OPNAME) return false;
        if (!c.str(sval[f])) return false;
      } else {
        if (f == F_TYPE || f == F_OPNAME) return false;
        if (!c.num(tok[f], isint[f])) return false;
      }
      seen |= 1u << f;
    } while (c.lit(','));
    if (!c.lit('}')) return false;
  }
  c.ws();
  if (c.p != c.e) return false;
  if (!((seen >> F_TYPE) & 1u)) return false;
  std::memset(&rec, 0, sizeof(rec));
  int32_t node = 0;
  auto common = [&]() {
    return to_int(tok[F_NODE], isint[F_NODE], node) &&
           to_int(tok[F_COMM], isint[F_COMM], rec.comm_id) &&
           to_int(tok[F_RANK], isint[F_RANK], rec.rank) &&
           to_int(tok[F_CHAN], isint[F_CHAN], rec.channel) &&
           to_int(tok[F_OP], isint[F_OP], rec.op_seq);
  };
  if (sval[F_TYPE] == "completion") {
    constexpr uint32_t need = (1u << F_TYPE) | (1u << F_NODE) | (1u << F_COMM) |
                              (1u << F_RANK) | (1u << F_CHAN) | (1u << F_OP) |
                              (1u << F_OPNAME) | (1u << F_BYTES) | (1u << F_START) |
                              (1u << F_END);
    if (seen != need) return false;
    if (!common()) return false;
    static const char* ops[] = {"AllGather", "ReduceScatter", "AllReduce", "Send", "Recv"};
    int op = -1;
    for (int k = 0; k < 5; ++k)
      if (sval[F_OPNAME] == ops[k]) op = k;
    if (op < 0) return false;
    uint64_t bytes = 0;
    double start = 0, end = 0;
    if (!to_int(tok[F_BYTES], isint[F_BYTES], bytes) || !to_double(tok[F_START], start) ||
        !to_double(tok[F_END], end))
      return false;
    if (end < start || bytes == 0 || rec.rank < 0 || rec.channel < 0) return false;
    rec.kind = CSG_KIND_COMPLETION;
    rec.op_name = static_cast<uint8_t>(op);
    rec.ts = end;
    rec.u.c.start_ms = start;
    rec.u.c.msg_bytes = bytes;
    return true;
  }
  if (sval[F_TYPE] == "state") {
    constexpr uint32_t need = (1u << F_TYPE) | (1u << F_NODE) | (1u << F_COMM) |
                              (1u << F_RANK) | (1u << F_CHAN) | (1u << F_OP) |
                              (1u << F_WEND) | (1u << F_STUCK) | (1u << F_TOTAL) |
                              (1u << F_READY) | (1u << F_TX) | (1u << F_DONE);
    if (seen != need) return false;
    if (!common()) return false;
    double wend = 0, stuck = 0;
    uint64_t total = 0, ready = 0, tx = 0, done = 0;
    if (!to_double(tok[F_WEND], wend) || !to_double(tok[F_STUCK], stuck) ||
        !to_int(tok[F_TOTAL], isint[F_TOTAL], total) ||
        !to_int(tok[F_READY], isint[F_READY], ready) ||
        !to_int(tok[F_TX], isint[F_TX], tx) || !to_int(tok[F_DONE], isint[F_DONE], done))
      return false;
    if (!(total >= ready && ready >= tx && tx >= done) || stuck < 0 || rec.rank < 0 ||
        rec.channel < 0 || ready > 0xffffffffull)
      return false;
    rec.kind = CSG_KIND_STATE;
    rec.ts = wend;
    rec.u.s.gpu_ready = static_cast<uint32_t>(ready);
    rec.u.s.rdma_transmitted = static_cast<uint32_t>(tx);
    rec.u.s.rdma_done = static_cast<uint32_t>(done);
    return true;
  }
  return false;
}

}  // namespace

bool fast_parse_trace(std::string_view text, std::vector<csg_packed_record>& out) {
  const size_t n = text.size();
  unsigned T = std::max(1u, std::thread::hardware_concurrency());
  if (n < (1u << 20)) T = 1;  // small inputs: no threads
  T = static_cast<unsigned>(std::min<size_t>(T, std::max<size_t>(1, n / (1u << 16))));
  // chunk boundaries at line starts
  std::vector<size_t> cut(T + 1, n);
  cut[0] = 0;
  for (unsigned t = 1; t < T; ++t) {
    size_t s = n * t / T;
    const void* nl = s < n ? std::memchr(text.data() + s, '\n', n - s) : nullptr;
    cut[t] = nl ? static_cast<const char*>(nl) - text.data() + 1 : n;
    if (cut[t] < cut[t - 1]) cut[t] = cut[t - 1];
  }
  std::vector<std::vector<csg_packed_record>> parts(T);
  std::vector<char> ok(T, 1);
  auto work = [&](unsigned t) {
    const char* p = text.data() + cut[t];
    const char* e = text.data() + cut[t + 1];
    auto& v = parts[t];
    v.reserve(static_cast<size_t>(e - p) / 150 + 16);
    while (p < e) {
      const char* nl = static_cast<const char*>(std::memchr(p, '\n', e - p));
      const char* le = nl ? nl : e;
      if (le > p) {
        csg_packed_record r;
        if (!parse_one(p, le, r)) {
          ok[t] = 0;
          return;
        }
        v.push_back(r);
      }
      p = le + 1;
    }
  };
  if (T == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    th.reserve(T);
    for (unsigned t = 0; t < T; ++t) th.emplace_back(work, t);
    for (auto& x : th) x.join();
  }
  for (unsigned t = 0; t < T; ++t)
    if (!ok[t]) return false;
  size_t total = 0;
  for (auto& v : parts) total += v.size();
  out.clear();
  out.reserve(total);
  for (auto& v : parts) out.insert(out.end(), v.begin(), v.end());
  return true;
}

}  // namespace csh
