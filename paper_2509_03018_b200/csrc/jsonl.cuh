// jsonl.cuh — one JSONL trace line -> csg_packed_record, as a host+device
// function (the device ingest runs it per line; the host instantiation is
// exported as a known-answer hook so CPU tests can pin it).
//
// Accepts exactly what the host fast path accepts (host/fast_jsonl.cpp): one
// flat JSON object per line of the reference schema (proj/src/trace.cpp:241-
// 337: "completion" or "state" records, every field present once, no
// unknown fields), keys without escapes, numbers as plain JSON tokens,
// validate_record's invariants (trace.cpp:39-57). Anything else — escapes,
// duplicate or unknown keys, a float in an integer field, out-of-range
// values, more than 19 significant digits, subnormal/overflowing doubles —
// returns false, and the caller hands the whole text to the exact host
// parser, which reports the reference's error and line number (or accepts
// what only the full JSON grammar accepts). Accepted lines therefore yield
// bit-identical records to the exact parser.
//
// Doubles: std::from_chars is correctly rounded, so is this: Clinger's fast
// path (w <= 2^53, |q| <= 22: one IEEE multiply or divide of exact values),
// else the Eisel-Lemire algorithm over 128-bit truncated powers of five
// (pow5_table.h; no fallback is needed for <= 19 digits: Mushtak & Lemire,
// "Fast Number Parsing Without Fallback", 2023).
#pragma once

#include <cstdint>

#include "csg_engine.h"
#include "pow5_table.h"

#ifdef __CUDACC__
#define CSG_HD __host__ __device__ __forceinline__
#else
#define CSG_HD inline
#endif

namespace csg {
namespace jsonl {

// shortest valid line: a completion with every value one character
// ({"type":"completion",...,"op_name":"Send",...}): 129 bytes
constexpr int kMinLine = 129;

#ifdef __CUDACC__
__device__ const uint64_t kPow5D[] = {CSG_POW5_TABLE};
#endif
static const uint64_t kPow5H[] = {CSG_POW5_TABLE};

CSG_HD uint64_t pow5_word(int i) {
#ifdef __CUDA_ARCH__
  return kPow5D[i];
#else
  return kPow5H[i];
#endif
}

CSG_HD void mul128(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
#ifdef __CUDA_ARCH__
  lo = a * b;
  hi = __umul64hi(a, b);
#else
  const unsigned __int128 r = static_cast<unsigned __int128>(a) * b;
  lo = static_cast<uint64_t>(r);
  hi = static_cast<uint64_t>(r >> 64);
#endif
}

CSG_HD int clz64(uint64_t x) {
#ifdef __CUDA_ARCH__
  return __clzll(static_cast<long long>(x));
#else
  return __builtin_clzll(x);
#endif
}

CSG_HD double bits_to_double(uint64_t b) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(b));
#else
  double d;
  __builtin_memcpy(&d, &b, 8);
  return d;
#endif
}

// 10^0 .. 10^22, all exact doubles (Clinger's fast path)
#define CSG_P10_TABLE                                                                  \
  1e0, 1e1, 1e2, 1e3, 1e4, 1e5, 1e6, 1e7, 1e8, 1e9, 1e10, 1e11, 1e12, 1e13, 1e14, 1e15, \
      1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22
#ifdef __CUDACC__
__device__ const double kP10D[23] = {CSG_P10_TABLE};
#endif
static const double kP10H[23] = {CSG_P10_TABLE};

CSG_HD double pow10_exact(int i) {
#ifdef __CUDA_ARCH__
  return kP10D[i];
#else
  return kP10H[i];
#endif
}

CSG_HD bool is_digit(char c) { return c >= '0' && c <= '9'; }

// w * 10^q as the nearest double (ties to even), w in [1, 2^64); false when
// the result is not a normal finite double.
CSG_HD bool eisel_lemire(uint64_t w, int64_t q, uint64_t& bits) {
  if (q < CSG_POW5_MIN || q > CSG_POW5_MAX) return false;
  const int lz = clz64(w);
  w <<= lz;
  const int idx = 2 * static_cast<int>(q - CSG_POW5_MIN);
  uint64_t hi, lo;
  mul128(w, pow5_word(idx), hi, lo);
  if ((hi & 0x1FF) == 0x1FF) {  // the truncated product may be short: refine
    uint64_t h2, l2;
    mul128(w, pow5_word(idx + 1), h2, l2);
    lo += h2;
    if (h2 > lo) ++hi;
  }
  const int upper = static_cast<int>(hi >> 63);
  const int shift = upper + 9;  // 64 - 52 - 3
  uint64_t m = hi >> shift;
  // floor(log2(10^q)) + 63 (exact for |q| <= 342), then the IEEE bias
  const int64_t p2 = (((152170 + 65536) * q) >> 16) + 63 + upper - lz + 1023;
  if (p2 <= 0) return false;  // subnormal or zero: left to from_chars
  if (lo <= 1 && q >= -4 && q <= 23 && (m & 3) == 1 && (m << shift) == hi)
    m &= ~uint64_t(1);  // exactly halfway: round to even (down)
  m += m & 1;
  m >>= 1;
  int64_t e = p2;
  if (m >= (uint64_t(2) << 52)) {
    m = uint64_t(1) << 52;
    ++e;
  }
  m &= ~(uint64_t(1) << 52);
  if (e >= 0x7FF) return false;  // overflow: from_chars reports a range error
  bits = m | (static_cast<uint64_t>(e) << 52);
  return true;
}

// JSON number token -> double as std::from_chars (round to nearest).
CSG_HD bool tok_to_double(const char* s, int n, double& out) {
  int i = 0;
  const bool neg = n > 0 && s[0] == '-';
  if (neg) {
    // "-0" is integer 0 to nlohmann (+0.0 as a double): exact parser's call
    bool allz = true;
    for (int k = 1; k < n; ++k)
      if (s[k] != '0') {
        allz = false;
        break;
      }
    if (allz) return false;
    ++i;
  }
  uint64_t w = 0;
  int nd = 0;
  int64_t q = 0;
  for (; i < n && is_digit(s[i]); ++i) {
    const int d = s[i] - '0';
    if (nd == 0 && d == 0) continue;
    if (nd == 19) return false;
    w = w * 10 + static_cast<uint64_t>(d);
    ++nd;
  }
  if (i < n && s[i] == '.') {
    for (++i; i < n && is_digit(s[i]); ++i) {
      const int d = s[i] - '0';
      --q;
      if (nd == 0 && d == 0) continue;
      if (nd == 19) return false;
      w = w * 10 + static_cast<uint64_t>(d);
      ++nd;
    }
  }
  if (i < n && (s[i] == 'e' || s[i] == 'E')) {
    ++i;
    bool en = false;
    if (i < n && (s[i] == '+' || s[i] == '-')) en = s[i++] == '-';
    int64_t e = 0;
    for (; i < n && is_digit(s[i]); ++i)
      if (e < 1000000) e = e * 10 + (s[i] - '0');
    q += en ? -e : e;
  }
  if (i != n) return false;
  if (w == 0) {
    out = neg ? -0.0 : 0.0;
    return true;
  }
  if (q >= -22 && q <= 22 && w <= (uint64_t(1) << 53)) {
    double d = static_cast<double>(w);
    d = q < 0 ? d / pow10_exact(static_cast<int>(-q)) : d * pow10_exact(static_cast<int>(q));
    out = neg ? -d : d;
    return true;
  }
  uint64_t b;
  if (!eisel_lemire(w, q, b)) return false;
  out = bits_to_double(b | (neg ? (uint64_t(1) << 63) : 0));
  return true;
}

// Integer token (no fraction/exponent) -> value in [lo, hi] (signed) as
// std::from_chars<T> with a range check.
CSG_HD bool tok_to_i64(const char* s, int n, int64_t lo, int64_t hi, int64_t& out) {
  int i = 0;
  const bool neg = n > 0 && s[0] == '-';
  if (neg) ++i;
  if (i >= n) return false;
  uint64_t v = 0;
  for (; i < n; ++i) {
    if (!is_digit(s[i])) return false;
    const uint64_t d = static_cast<uint64_t>(s[i] - '0');
    if (v > (~uint64_t(0) - d) / 10) return false;
    v = v * 10 + d;
  }
  if (neg) {
    if (v > static_cast<uint64_t>(-(lo + 1)) + 1) return false;
    out = v == 0 ? 0 : -static_cast<int64_t>(v - 1) - 1;
  } else {
    if (v > static_cast<uint64_t>(hi)) return false;
    out = static_cast<int64_t>(v);
  }
  return true;
}

CSG_HD bool tok_to_u64(const char* s, int n, uint64_t& out) {
  if (n <= 0 || s[0] == '-') return false;
  uint64_t v = 0;
  for (int i = 0; i < n; ++i) {
    if (!is_digit(s[i])) return false;
    const uint64_t d = static_cast<uint64_t>(s[i] - '0');
    if (v > (~uint64_t(0) - d) / 10) return false;
    v = v * 10 + d;
  }
  out = v;
  return true;
}

enum Field : int {
  F_TYPE, F_NODE, F_COMM, F_RANK, F_CHAN, F_OP, F_OPNAME, F_BYTES, F_START, F_END,
  F_WEND, F_STUCK, F_TOTAL, F_READY, F_TX, F_DONE, F_N
};

CSG_HD bool eq(const char* a, int n, const char* lit) {
  int i = 0;
  for (; i < n; ++i)
    if (lit[i] != a[i]) return false;
  return lit[i] == 0;
}

CSG_HD int field_of(const char* k, int n) {
  switch (n) {
    case 4:
      if (eq(k, n, "type")) return F_TYPE;
      if (eq(k, n, "node")) return F_NODE;
      if (eq(k, n, "rank")) return F_RANK;
      return -1;
    case 6:
      if (eq(k, n, "op_seq")) return F_OP;
      if (eq(k, n, "end_ms")) return F_END;
      return -1;
    case 7:
      if (eq(k, n, "comm_id")) return F_COMM;
      if (eq(k, n, "channel")) return F_CHAN;
      if (eq(k, n, "op_name")) return F_OPNAME;
      return -1;
    case 8:
      if (eq(k, n, "start_ms")) return F_START;
      if (eq(k, n, "stuck_ms")) return F_STUCK;
      return -1;
    case 9:
      if (eq(k, n, "msg_bytes")) return F_BYTES;
      if (eq(k, n, "gpu_ready")) return F_READY;
      if (eq(k, n, "rdma_done")) return F_DONE;
      return -1;
    case 12:
      return eq(k, n, "total_chunks") ? F_TOTAL : -1;
    case 13:
      return eq(k, n, "window_end_ms") ? F_WEND : -1;
    case 16:
      return eq(k, n, "rdma_transmitted") ? F_TX : -1;
    default:
      return -1;
  }
}

struct Cursor {
  const char* p;
  const char* e;
  CSG_HD void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n')) ++p;
  }
  CSG_HD bool lit(char c) {
    ws();
    if (p < e && *p == c) {
      ++p;
      return true;
    }
    return false;
  }
  // "..." without escapes or control characters
  CSG_HD bool str(const char*& s, int& n) {
    ws();
    if (p >= e || *p != '"') return false;
    s = ++p;
    while (p < e && *p != '"') {
      if (*p == '\\' || static_cast<unsigned char>(*p) < 0x20) return false;
      ++p;
    }
    if (p >= e) return false;
    n = static_cast<int>(p - s);
    ++p;
    return true;
  }
  // JSON number token [-](0|[1-9]digits)[.digits][(e|E)[+-]digits]
  CSG_HD bool num(const char*& s, int& n, bool& is_int) {
    ws();
    s = p;
    if (p < e && *p == '-') ++p;
    if (p >= e || !is_digit(*p)) return false;
    if (*p == '0' && p + 1 < e && is_digit(p[1])) return false;
    while (p < e && is_digit(*p)) ++p;
    is_int = true;
    if (p < e && *p == '.') {
      is_int = false;
      ++p;
      if (p >= e || !is_digit(*p)) return false;
      while (p < e && is_digit(*p)) ++p;
    }
    if (p < e && (*p == 'e' || *p == 'E')) {
      is_int = false;
      ++p;
      if (p < e && (*p == '+' || *p == '-')) ++p;
      if (p >= e || !is_digit(*p)) return false;
      while (p < e && is_digit(*p)) ++p;
    }
    n = static_cast<int>(p - s);
    return true;
  }
};

// One line (without its '\n') -> record; false: the exact parser decides.
CSG_HD bool parse_line(const char* b, const char* e, csg_packed_record& rec) {
  Cursor c{b, e};
  if (!c.lit('{')) return false;
  const char* ts[F_N];
  int tn[F_N];
  bool isint[F_N];
  uint32_t seen = 0;
  if (!c.lit('}')) {
    do {
      const char* k;
      int kn;
      if (!c.str(k, kn)) return false;
      const int f = field_of(k, kn);
      if (f < 0 || ((seen >> f) & 1u)) return false;  // unknown / duplicate
      if (!c.lit(':')) return false;
      c.ws();
      if (c.p < c.e && *c.p == '"') {
        if (f != F_TYPE && f != F_OPNAME) return false;
        if (!c.str(ts[f], tn[f])) return false;
        isint[f] = false;
      } else {
        if (f == F_TYPE || f == F_OPNAME) return false;
        if (!c.num(ts[f], tn[f], isint[f])) return false;
      }
      seen |= 1u << f;
    } while (c.lit(','));
    if (!c.lit('}')) return false;
  }
  c.ws();
  if (c.p != c.e) return false;
  if (!((seen >> F_TYPE) & 1u)) return false;
  // all fields of the packed record, padding included, start zeroed
  rec.ts = 0;
  rec.op_seq = 0;
  rec.rank = rec.comm_id = rec.channel = 0;
  rec.kind = rec.op_name = 0;
  rec.reserved = 0;
  rec.u.s.gpu_ready = rec.u.s.rdma_transmitted = rec.u.s.rdma_done = rec.u.s.reserved = 0;
  int64_t v;
  auto i32 = [&](int f, int32_t& out) {
    if (!isint[f] || !tok_to_i64(ts[f], tn[f], INT32_MIN, INT32_MAX, v)) return false;
    out = static_cast<int32_t>(v);
    return true;
  };
  auto common = [&]() {
    int32_t node;
    if (!i32(F_NODE, node) || !i32(F_COMM, rec.comm_id) || !i32(F_RANK, rec.rank) ||
        !i32(F_CHAN, rec.channel))
      return false;
    if (!isint[F_OP] || !tok_to_i64(ts[F_OP], tn[F_OP], INT64_MIN, INT64_MAX, v))
      return false;
    rec.op_seq = v;
    return true;
  };
  if (eq(ts[F_TYPE], tn[F_TYPE], "completion")) {
    constexpr uint32_t need = (1u << F_TYPE) | (1u << F_NODE) | (1u << F_COMM) |
                              (1u << F_RANK) | (1u << F_CHAN) | (1u << F_OP) |
                              (1u << F_OPNAME) | (1u << F_BYTES) | (1u << F_START) |
                              (1u << F_END);
    if (seen != need || !common()) return false;
    const char* on = ts[F_OPNAME];
    const int nn = tn[F_OPNAME];
    int op = -1;
    if (eq(on, nn, "AllGather")) op = CSG_OP_ALLGATHER;
    else if (eq(on, nn, "ReduceScatter")) op = CSG_OP_REDUCESCATTER;
    else if (eq(on, nn, "AllReduce")) op = CSG_OP_ALLREDUCE;
    else if (eq(on, nn, "Send")) op = CSG_OP_SEND;
    else if (eq(on, nn, "Recv")) op = CSG_OP_RECV;
    if (op < 0) return false;
    uint64_t bytes;
    double start, end;
    if (!isint[F_BYTES] || !tok_to_u64(ts[F_BYTES], tn[F_BYTES], bytes) ||
        !tok_to_double(ts[F_START], tn[F_START], start) ||
        !tok_to_double(ts[F_END], tn[F_END], end))
      return false;
    if (end < start || bytes == 0 || rec.rank < 0 || rec.channel < 0) return false;
    rec.kind = CSG_KIND_COMPLETION;
    rec.op_name = static_cast<uint8_t>(op);
    rec.ts = end;
    rec.u.c.start_ms = start;
    rec.u.c.msg_bytes = bytes;
    return true;
  }
  if (eq(ts[F_TYPE], tn[F_TYPE], "state")) {
    constexpr uint32_t need = (1u << F_TYPE) | (1u << F_NODE) | (1u << F_COMM) |
                              (1u << F_RANK) | (1u << F_CHAN) | (1u << F_OP) |
                              (1u << F_WEND) | (1u << F_STUCK) | (1u << F_TOTAL) |
                              (1u << F_READY) | (1u << F_TX) | (1u << F_DONE);
    if (seen != need || !common()) return false;
    double wend, stuck;
    uint64_t total, ready, tx, done;
    if (!tok_to_double(ts[F_WEND], tn[F_WEND], wend) ||
        !tok_to_double(ts[F_STUCK], tn[F_STUCK], stuck) || !isint[F_TOTAL] ||
        !tok_to_u64(ts[F_TOTAL], tn[F_TOTAL], total) || !isint[F_READY] ||
        !tok_to_u64(ts[F_READY], tn[F_READY], ready) || !isint[F_TX] ||
        !tok_to_u64(ts[F_TX], tn[F_TX], tx) || !isint[F_DONE] ||
        !tok_to_u64(ts[F_DONE], tn[F_DONE], done))
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

// ---- canonical-order fast path -------------------------------------------
// The reference's serializer writes every line in one fixed field order with
// no whitespace (serialize_record, proj/src/trace.cpp:187-236). parse_fast
// reads exactly that form straight into registers (no per-field token
// tables, so no local memory on the device) and applies the same
// conversions and checks as parse_line; anything else — another field
// order, whitespace, a failed check — returns false and the caller runs
// parse_line, which decides. So both paths accept the same lines with the
// same records.

// the 48-byte record as six words (little-endian csg_packed_record layout)
struct Words {
  uint64_t w[6];
};

// lit is a NUL-terminated literal; advances p past it
CSG_HD bool expect(const char*& p, const char* e, const char* lit) {
  for (; *lit; ++lit, ++p)
    if (p >= e || *p != *lit) return false;
  return true;
}

// JSON number token (grammar of Cursor::num, no surrounding whitespace)
CSG_HD bool num_tok(const char*& p, const char* e, const char*& s, int& n, bool& is_int) {
  s = p;
  if (p < e && *p == '-') ++p;
  if (p >= e || !is_digit(*p)) return false;
  if (*p == '0' && p + 1 < e && is_digit(p[1])) return false;
  while (p < e && is_digit(*p)) ++p;
  is_int = true;
  if (p < e && *p == '.') {
    is_int = false;
    ++p;
    if (p >= e || !is_digit(*p)) return false;
    while (p < e && is_digit(*p)) ++p;
  }
  if (p < e && (*p == 'e' || *p == 'E')) {
    is_int = false;
    ++p;
    if (p < e && (*p == '+' || *p == '-')) ++p;
    if (p >= e || !is_digit(*p)) return false;
    while (p < e && is_digit(*p)) ++p;
  }
  n = static_cast<int>(p - s);
  return true;
}

CSG_HD bool fast_i64(const char*& p, const char* e, int64_t lo, int64_t hi, int64_t& v) {
  const char* s;
  int n;
  bool is_int;
  return num_tok(p, e, s, n, is_int) && is_int && tok_to_i64(s, n, lo, hi, v);
}

CSG_HD bool fast_u64(const char*& p, const char* e, uint64_t& v) {
  const char* s;
  int n;
  bool is_int;
  return num_tok(p, e, s, n, is_int) && is_int && tok_to_u64(s, n, v);
}

CSG_HD bool fast_f64(const char*& p, const char* e, double& v) {
  const char* s;
  int n;
  bool is_int;
  return num_tok(p, e, s, n, is_int) && tok_to_double(s, n, v);
}

CSG_HD uint64_t dbits(double d) {
#ifdef __CUDA_ARCH__
  return static_cast<uint64_t>(__double_as_longlong(d));
#else
  uint64_t b;
  __builtin_memcpy(&b, &d, 8);
  return b;
#endif
}

CSG_HD bool parse_fast(const char* p, const char* e, Words& out) {
  if (!expect(p, e, "{\"type\":\"")) return false;
  const bool comp = p < e && *p == 'c';
  if (!expect(p, e, comp ? "completion\",\"node\":" : "state\",\"node\":")) return false;
  int64_t node, comm, rank, chan, op;
  if (!fast_i64(p, e, INT32_MIN, INT32_MAX, node) || !expect(p, e, ",\"comm_id\":") ||
      !fast_i64(p, e, INT32_MIN, INT32_MAX, comm) || !expect(p, e, ",\"rank\":") ||
      !fast_i64(p, e, INT32_MIN, INT32_MAX, rank) || !expect(p, e, ",\"channel\":") ||
      !fast_i64(p, e, INT32_MIN, INT32_MAX, chan) || !expect(p, e, ",\"op_seq\":") ||
      !fast_i64(p, e, INT64_MIN, INT64_MAX, op))
    return false;
  if (rank < 0 || chan < 0) return false;
  out.w[1] = static_cast<uint64_t>(op);
  out.w[2] = static_cast<uint32_t>(rank) | (static_cast<uint64_t>(static_cast<uint32_t>(comm)) << 32);
  if (comp) {
    if (!expect(p, e, ",\"op_name\":\"")) return false;
    const char* nm = p;
    while (p < e && *p != '"' && *p != '\\') ++p;
    const int nn = static_cast<int>(p - nm);
    int opn = -1;
    if (eq(nm, nn, "AllGather")) opn = CSG_OP_ALLGATHER;
    else if (eq(nm, nn, "ReduceScatter")) opn = CSG_OP_REDUCESCATTER;
    else if (eq(nm, nn, "AllReduce")) opn = CSG_OP_ALLREDUCE;
    else if (eq(nm, nn, "Send")) opn = CSG_OP_SEND;
    else if (eq(nm, nn, "Recv")) opn = CSG_OP_RECV;
    uint64_t bytes;
    double start, end;
    if (opn < 0 || !expect(p, e, "\",\"msg_bytes\":") || !fast_u64(p, e, bytes) ||
        !expect(p, e, ",\"start_ms\":") || !fast_f64(p, e, start) ||
        !expect(p, e, ",\"end_ms\":") || !fast_f64(p, e, end) || !expect(p, e, "}") || p != e)
      return false;
    if (end < start || bytes == 0) return false;
    out.w[0] = dbits(end);
    out.w[3] = static_cast<uint32_t>(chan) | (static_cast<uint64_t>(CSG_KIND_COMPLETION) << 32) |
               (static_cast<uint64_t>(opn) << 40);
    out.w[4] = dbits(start);
    out.w[5] = bytes;
    return true;
  }
  double wend, stuck;
  uint64_t total, ready, tx, done;
  if (!expect(p, e, ",\"window_end_ms\":") || !fast_f64(p, e, wend) ||
      !expect(p, e, ",\"stuck_ms\":") || !fast_f64(p, e, stuck) ||
      !expect(p, e, ",\"total_chunks\":") || !fast_u64(p, e, total) ||
      !expect(p, e, ",\"gpu_ready\":") || !fast_u64(p, e, ready) ||
      !expect(p, e, ",\"rdma_transmitted\":") || !fast_u64(p, e, tx) ||
      !expect(p, e, ",\"rdma_done\":") || !fast_u64(p, e, done) || !expect(p, e, "}") ||
      p != e)
    return false;
  if (!(total >= ready && ready >= tx && tx >= done) || stuck < 0 || ready > 0xffffffffull)
    return false;
  out.w[0] = dbits(wend);
  out.w[3] = static_cast<uint32_t>(chan) | (static_cast<uint64_t>(CSG_KIND_STATE) << 32);
  out.w[4] = ready | (tx << 32);
  out.w[5] = done;
  return true;
}

}  // namespace jsonl
}  // namespace csg
