// jsonl.cu — JSONL trace ingest on the device.
//
// Reference: collsight_run_analyze (proj/src/c_api.cpp:111-123) loads the
// trace with load_trace_file -> parse_trace_text (proj/src/trace.cpp:241-
// 337, nlohmann/json, ~33 MB/s): one record per non-empty line, in line
// order (the store's emission order). Here the text streams to HBM and is
// parsed there:
//
//   host     the file (or caller's text) is read in 16 MB chunks into pinned
//            staging slots, one reader thread per slot (hardware threads
//            - 2, at most 16), each chunk copied to the device text buffer
//            behind the previous one (copy engine);
//   k_jsonl_count  per 32 KB tile: number of line starts (non-empty lines);
//   k_jsonl_scan   one block: exclusive scan of the tile counts -> record
//                  index of each tile's first line (running total kept on
//                  the device across super-chunks);
//   k_jsonl_parse  per tile: the tile (+ up to 8 KB of the last line's
//                  overhang) staged in shared memory, line starts ranked by
//                  a block scan, one thread per line running
//                  jsonl::parse_fast (the serializer's canonical field
//                  order, registers only), else jsonl::parse_line (any
//                  field order / whitespace), into the packed record at its
//                  line index.
//
// Text larger than the device budget is processed in super-chunks cut at
// the last newline. Any line the device parser cannot vouch for sets an
// error word; the call then reports "not accepted" and leaves the store
// unchanged, and the caller parses the whole text with the exact host parser
// (the reference's error message and line number, trace.cpp:256-311).
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <future>
#include <string>
#include <thread>
#include <vector>

#include "jsonl.cuh"
#include "objects.h"

namespace csg {
namespace {

constexpr uint32_t kJTile = 32768;       // text bytes per tile
constexpr uint32_t kJOver = 8192;        // longest line overhang staged
constexpr int kJThreads = 256;
constexpr int kJMaxLines = 512;          // > 32768 / 129 + 1 (valid lines per tile)
constexpr size_t kJChunk = 16ull << 20;  // host staging chunk
constexpr int kJMaxSlots = 16;           // pinned staging slots = reader threads

enum : uint32_t { JERR_LINE = 1, JERR_TILE = 2, JERR_CAP = 4, JERR_LONG = 8 };

// Line starts among 16 text bytes (bit j: byte j starts a line, i.e. it is
// not '\n' and the byte before it is '\n'); prev = the byte before byte 0.
__device__ __forceinline__ uint32_t starts16(const uint4& q, unsigned char prev) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
  uint32_t m = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const unsigned char x = static_cast<unsigned char>(w[j >> 2] >> (8 * (j & 3)));
    m |= static_cast<uint32_t>((x != '\n') & (prev == '\n')) << j;
    prev = x;
  }
  return m;
}

// 16 bytes at text offset p, '\n'-padded past len (callers also mask the
// start bits at and past len)
__device__ __forceinline__ uint4 load16(const unsigned char* t, uint64_t p, uint64_t len) {
  if (p + 16 <= len) return *reinterpret_cast<const uint4*>(t + p);
  unsigned char b[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) b[j] = p + j < len ? t[p + j] : '\n';
  uint4 q;
  memcpy(&q, b, 16);
  return q;
}

// Block-cooperative pass over one tile in rounds of 4 KB (thread t owns
// bytes [16t, 16t + 16) of each round: coalesced, bank-conflict free); the
// byte before a thread's 16 comes from its lane neighbour (lane 0 loads it).
// Per round: starts mask of the thread's 16 bytes.
template <typename Load, typename Prev>
__device__ __forceinline__ uint32_t round_mask(Load load, Prev prev_byte, uint64_t p,
                                               uint64_t lim) {
  const uint4 q = load(p);
  const unsigned char last = static_cast<unsigned char>(q.w >> 24);
  unsigned char prev = static_cast<unsigned char>(__shfl_up_sync(0xffffffffu, last, 1));
  if ((threadIdx.x & 31) == 0) prev = prev_byte(p);
  uint32_t m = p < lim ? starts16(q, prev) : 0u;
  if (p < lim && lim - p < 16) m &= (1u << (lim - p)) - 1u;
  return m;
}

constexpr uint32_t kJRound = kJThreads * 16;  // 4 KB
constexpr int kJRounds = kJTile / kJRound;    // 8

__global__ void __launch_bounds__(kJThreads)
    k_jsonl_count(const unsigned char* __restrict__ text, uint64_t len,
                  uint32_t* __restrict__ counts) {
  __shared__ uint32_t wsum[kJThreads / 32];
  const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kJTile;
  const uint64_t t1 = min(t0 + kJTile, len);
  uint32_t c = 0;
  auto load = [&](uint64_t p) { return load16(text, p, len); };
  auto prev = [&](uint64_t p) -> unsigned char {
    return p == 0 || p > len ? '\n' : text[p - 1];
  };
#pragma unroll 2
  for (int r = 0; r < kJRounds; ++r) {
    const uint64_t p = t0 + r * kJRound + 16 * threadIdx.x;
    c += __popc(round_mask(load, prev, p, t1));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < kJThreads / 32; ++w) s += wsum[w];
    counts[blockIdx.x] = s;
  }
}

// One block: bases[t] = total_in + sum(counts[0..t)), total advanced.
__global__ void __launch_bounds__(1024)
    k_jsonl_scan(const uint32_t* __restrict__ counts, uint32_t ntiles,
                 unsigned long long* __restrict__ bases, unsigned long long* total,
                 unsigned long long cap, uint32_t* err) {
  __shared__ unsigned long long wsum[32];
  __shared__ unsigned long long carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = *total;
  __syncthreads();
  for (uint32_t t0 = 0; t0 < ntiles; t0 += blockDim.x) {
    const uint32_t t = t0 + threadIdx.x;
    const unsigned long long v = t < ntiles ? counts[t] : 0ull;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      unsigned long long s = lane < static_cast<int>(blockDim.x >> 5) ? wsum[lane] : 0ull;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      wsum[lane] = s;
    }
    __syncthreads();
    const unsigned long long excl = carry + (warp ? wsum[warp - 1] : 0ull) + x - v;
    if (t < ntiles) bases[t] = excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += wsum[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (carry > cap) atomicOr(err, JERR_CAP);
    *total = carry;
  }
}

// Lines outside the canonical form: the general parser, kept out of line so
// its per-field token tables (local memory) cost nothing on the fast path.
// Writes the record to *out (when idx < cap) and returns 1, 0 when rejected.
__device__ __noinline__ int parse_general(const char* b, const char* e,
                                          csg_packed_record* out, bool in_cap) {
  csg_packed_record rec;
  if (!jsonl::parse_line(b, e, rec)) return 0;
  if (in_cap) *out = rec;
  return 1;
}

__global__ void __launch_bounds__(kJThreads)
    k_jsonl_parse(const unsigned char* __restrict__ text, uint64_t len,
                  const unsigned long long* __restrict__ bases,
                  csg_packed_record* __restrict__ out, unsigned long long cap,
                  uint32_t* __restrict__ err) {
  __shared__ __align__(16) unsigned char buf[16 + kJTile + kJOver];  // buf[15] = byte t0-1
  __shared__ uint16_t starts[kJMaxLines];
  __shared__ uint32_t wsum[kJThreads / 32];
  __shared__ uint32_t nlines;
  const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kJTile;
  const uint64_t t1 = min(t0 + kJTile, len);
  const uint64_t ld_end = min(t1 + kJOver, len);
  const uint32_t nb = static_cast<uint32_t>(ld_end - t0);
  unsigned char* tb = buf + 16;
  {  // stage [t0, ld_end): 16-byte loads (t0 is tile-aligned), byte tail
    const uint32_t n16 = nb / 16;
    const uint4* src = reinterpret_cast<const uint4*>(text + t0);
    uint4* dst = reinterpret_cast<uint4*>(tb);
    for (uint32_t i = threadIdx.x; i < n16; i += kJThreads) dst[i] = __ldg(src + i);
    for (uint32_t i = n16 * 16 + threadIdx.x; i < nb; i += kJThreads) tb[i] = text[t0 + i];
    if (threadIdx.x == 0) buf[15] = t0 == 0 ? '\n' : text[t0 - 1];
  }
  __syncthreads();
  // line starts of this tile, ranked in text order: per 4 KB round a
  // block exclusive scan of the threads' start counts
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t tl = static_cast<uint32_t>(t1 - t0);
  auto load = [&](uint64_t p) {
    return p + 16 <= nb ? *reinterpret_cast<const uint4*>(tb + p) : load16(tb, p, nb);
  };
  auto prev = [&](uint64_t p) -> unsigned char { return tb[static_cast<int64_t>(p) - 1]; };
  if (threadIdx.x == 0) nlines = 0;
  __syncthreads();
  for (int r = 0; r < kJRounds; ++r) {
    const uint32_t p = r * kJRound + 16 * threadIdx.x;
    uint32_t m = round_mask(load, prev, p, tl);
    const uint32_t c = __popc(m);
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    uint32_t before = nlines;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    uint32_t k = before + x - c;
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      if (k < kJMaxLines) starts[k] = static_cast<uint16_t>(p + j);
      ++k;
    }
    __syncthreads();
    if (threadIdx.x == kJThreads - 1) nlines = k;
    __syncthreads();
  }
  const uint32_t total = nlines;
  if (total > kJMaxLines) {  // cannot be a valid trace (lines >= 129 bytes)
    if (threadIdx.x == 0) atomicOr(err, JERR_TILE);
    return;
  }
  const unsigned long long base = bases[blockIdx.x];
  for (uint32_t j = threadIdx.x; j < total; j += kJThreads) {
    const uint32_t s = starts[j];
    uint32_t e = s;
    while (e < nb && tb[e] != '\n') ++e;
    if (e == nb && ld_end < len) {  // the line runs past the staged overhang
      atomicOr(err, JERR_LONG);
      continue;
    }
    const unsigned long long idx = base + j;
    const char* lb = reinterpret_cast<const char*>(tb + s);
    const char* le = reinterpret_cast<const char*>(tb + e);
    jsonl::Words w;
    const bool in_cap = idx < cap;
    if (e - s >= static_cast<uint32_t>(jsonl::kMinLine) && jsonl::parse_fast(lb, le, w)) {
      if (in_cap) {
        ulonglong2* o2 = reinterpret_cast<ulonglong2*>(out + idx);
        o2[0] = make_ulonglong2(w.w[0], w.w[1]);
        o2[1] = make_ulonglong2(w.w[2], w.w[3]);
        o2[2] = make_ulonglong2(w.w[4], w.w[5]);
      }
    } else if (e - s < static_cast<uint32_t>(jsonl::kMinLine) ||
               !parse_general(lb, le, out + idx, in_cap)) {
      atomicOr(err, JERR_LINE);
      continue;
    }
    if (!in_cap) atomicOr(err, JERR_CAP);
  }
}

}  // namespace

// Source of the text: the caller's memory or a file descriptor.
struct JsonlSource {
  const char* mem = nullptr;
  int fd = -1;
  bool read(char* dst, uint64_t off, size_t n) const {
    if (mem) {
      std::memcpy(dst, mem + off, n);
      return true;
    }
    size_t got = 0;
    while (got < n) {
      const ssize_t r = pread(fd, dst + got, n - got, static_cast<off_t>(off + got));
      if (r <= 0) return false;
      got += static_cast<size_t>(r);
    }
    return true;
  }
};

// Appends the records of the text; *accepted = 0 (store unchanged) when some
// line must go to the exact host parser.
void store_append_jsonl(csg_store* s, const JsonlSource& src, uint64_t len, int* accepted) {
  csg_ctx* c = s->ctx;
  cudaStream_t st = c->stream;
  *accepted = 0;
  if (len == 0) {
    *accepted = 1;
    return;
  }
  static const uint64_t super_max = [] {
    const char* e = std::getenv("CSG_JSONL_SUPER_MB");
    const uint64_t mb = e ? std::strtoull(e, nullptr, 10) : 16384;
    return std::max<uint64_t>(mb, 1) << 20;
  }();
  // records: valid lines are >= 129 bytes + '\n' (the last may lack it)
  const uint64_t cap = len / (jsonl::kMinLine + 1) + 2;
  {
    const size_t need = (s->n + cap) * sizeof(csg_packed_record);
    if (need > s->recs.bytes) {
      DevBuf nb;
      nb.ensure(std::max(need, s->recs.bytes + s->recs.bytes / 2));
      if (s->n)
        CSG_CUDA(cudaMemcpyAsync(nb.p, s->recs.p, s->n * sizeof(csg_packed_record),
                                 cudaMemcpyDeviceToDevice, st));
      CSG_CUDA(cudaStreamSynchronize(st));
      std::swap(nb.p, s->recs.p);
      std::swap(nb.bytes, s->recs.bytes);
    }
  }
  const uint64_t dev_bytes = std::min(len, super_max);
  DevBuf& text = c->buf("jsonl.text");
  text.ensure(dev_bytes + 64);
  const uint32_t max_tiles = static_cast<uint32_t>((dev_bytes + kJTile - 1) / kJTile);
  DevBuf& counts = c->buf("jsonl.counts");
  DevBuf& bases = c->buf("jsonl.bases");
  DevBuf& ctl = c->buf("jsonl.ctl");  // [0] records so far, [1] error bits
  counts.ensure(static_cast<size_t>(max_tiles) * 4 + 4);
  bases.ensure(static_cast<size_t>(max_tiles) * 8 + 8);
  ctl.ensure(16);
  CSG_CUDA(cudaMemsetAsync(ctl.p, 0, 16, st));
  unsigned long long* total = ctl.as<unsigned long long>();
  uint32_t* err = reinterpret_cast<uint32_t*>(total + 1);
  csg_packed_record* out = s->recs.as<csg_packed_record>() + s->n;
  // pinned staging slots (grow-only, per context) and their release events;
  // one reader thread per slot (pread from the page cache is a CPU copy: the
  // readers, not the copy engine, bound the text rate)
  static const int nslots = [] {
    const char* e = std::getenv("CSG_JSONL_READERS");
    const int hw = static_cast<int>(std::thread::hardware_concurrency());
    const int v = e ? std::atoi(e) : hw - 2;
    return std::clamp(v, 2, kJMaxSlots);
  }();
  HostBuf* slot[kJMaxSlots];
  static const size_t chunk_cfg = [] {  // CSG_JSONL_CHUNK_KB: tests only
    const char* e = std::getenv("CSG_JSONL_CHUNK_KB");
    const size_t kb = e ? std::strtoull(e, nullptr, 10) : 0;
    return kb ? std::max<size_t>(kb, 64) << 10 : kJChunk;
  }();
  const size_t chunk = std::min<uint64_t>(chunk_cfg, len);
  std::vector<cudaEvent_t> ev(nslots);
  for (int i = 0; i < nslots; ++i) {
    const std::string name = "jsonl.slot" + std::to_string(i);
    slot[i] = &c->hbuf(name.c_str());
    slot[i]->ensure(chunk);
    CSG_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
  }
  const int kJSlots = nslots;
  struct EvGuard {
    std::vector<cudaEvent_t>& v;
    ~EvGuard() {
      for (cudaEvent_t e : v) cudaEventDestroy(e);
    }
  } evg{ev};
  bool ok = true;
  uint64_t pos = 0;
  uint64_t chunk_no = 0;  // global chunk counter: slot = chunk_no % kJSlots
  std::vector<char> slot_used(kJSlots, 0);
  // CSG_E2E_PROF=1: wall time of the ingest and the time spent waiting on
  // the readers, on stderr
  static const bool prof = std::getenv("CSG_E2E_PROF") != nullptr;
  using clk = std::chrono::steady_clock;
  const auto w0 = clk::now();
  double wait_ms = 0;
  while (ok && pos < len) {
    uint64_t end = std::min(len, pos + dev_bytes);
    const uint64_t nch = (end - pos + chunk - 1) / chunk;
    // readers run up to kJSlots chunks ahead of the copies
    std::vector<std::future<bool>> fut(nch);
    auto launch_read = [&](uint64_t i) {
      const int sl = static_cast<int>((chunk_no + i) % kJSlots);
      const uint64_t off = pos + i * chunk;
      const size_t n = static_cast<size_t>(std::min<uint64_t>(chunk, end - off));
      const bool wait = slot_used[sl] != 0;
      slot_used[sl] = 1;
      cudaEvent_t e = ev[sl];
      char* dst = slot[sl]->as<char>();
      const int dev = c->device;
      fut[i] = std::async(std::launch::async, [=, &src]() {
        if (wait && (cudaSetDevice(dev) != cudaSuccess || cudaEventSynchronize(e) != cudaSuccess))
          return false;
        return src.read(dst, off, n);
      });
    };
    for (uint64_t i = 0; i < std::min<uint64_t>(nch, kJSlots); ++i) launch_read(i);
    for (uint64_t i = 0; i < nch; ++i) {
      const int sl = static_cast<int>((chunk_no + i) % kJSlots);
      const uint64_t off = pos + i * chunk;
      size_t n = static_cast<size_t>(std::min<uint64_t>(chunk, end - off));
      const auto g0 = clk::now();
      if (!fut[i].get()) ok = false;
      wait_ms += std::chrono::duration<double, std::milli>(clk::now() - g0).count();
      if (ok && i + 1 == nch && end < len) {
        // super-chunk boundary: cut after the last newline of this chunk
        const char* b = slot[sl]->as<char>();
        size_t k = n;
        while (k > 0 && b[k - 1] != '\n') --k;
        if (k == 0) ok = false;  // a line longer than a chunk: exact parser
        n = k;
        end = off + n;
      }
      if (ok)
        CSG_CUDA(cudaMemcpyAsync(text.as<char>() + (off - pos), slot[sl]->p, n,
                                 cudaMemcpyHostToDevice, st));
      CSG_CUDA(cudaEventRecord(ev[sl], st));
      c->h2d_bytes += n;
      if (i + kJSlots < nch) launch_read(i + kJSlots);
    }
    for (auto& f : fut)
      if (f.valid()) f.get();
    if (!ok) break;
    chunk_no += nch;
    const uint64_t sl_len = end - pos;
    const uint32_t nt = static_cast<uint32_t>((sl_len + kJTile - 1) / kJTile);
    {
      ProfScope ps_(c->lc, "k_jsonl_count", st);
      k_jsonl_count<<<nt, kJThreads, 0, st>>>(text.as<unsigned char>(), sl_len,
                                             counts.as<uint32_t>());
    }
    {
      ProfScope ps_(c->lc, "k_jsonl_scan", st);
      k_jsonl_scan<<<1, 1024, 0, st>>>(counts.as<uint32_t>(), nt,
                                       bases.as<unsigned long long>(), total, cap, err);
    }
    {
      ProfScope ps_(c->lc, "k_jsonl_parse", st);
      k_jsonl_parse<<<nt, kJThreads, 0, st>>>(text.as<unsigned char>(), sl_len,
                                             bases.as<unsigned long long>(), out, cap, err);
    }
    CSG_CUDA(cudaGetLastError());
    pos = end;
  }
  HostBuf& hb = c->hbuf("jsonl.ctl");
  hb.ensure(16);
  FetchArgs fa{};
  fa.add(ctl.p, hb.p, 16);
  ctx_sync(c, &fa);
  if (prof)
    std::fprintf(stderr, "[jsonl] %llu bytes, %d readers x %zu KB: %.3f ms (%.3f ms waiting on reads)\n",
                 static_cast<unsigned long long>(len), kJSlots, chunk >> 10,
                 std::chrono::duration<double, std::milli>(clk::now() - w0).count(), wait_ms);
  if (!ok) return;
  uint64_t nrec = 0;
  uint32_t e = 0;
  std::memcpy(&nrec, hb.p, 8);
  std::memcpy(&e, hb.as<unsigned char>() + 8, 4);
  if (e) return;
  s->n += nrec;
  s->indexed = false;
  s->op_indexed = false;
  s->flow_indexed = false;
  s->flow_early = false;
  *accepted = 1;
}

void store_append_jsonl_mem(csg_store* s, const char* text, uint64_t len, int* accepted) {
  JsonlSource src;
  src.mem = text;
  store_append_jsonl(s, src, len, accepted);
}

// false: the file cannot be opened/read here (the exact loader reports it)
void store_append_jsonl_file(csg_store* s, const char* path, int* accepted) {
  *accepted = 0;
  const int fd = open(path, O_RDONLY | O_CLOEXEC);
  if (fd < 0) return;
  struct FdGuard {
    int fd;
    ~FdGuard() { close(fd); }
  } g{fd};
  struct stat sb;
  if (fstat(fd, &sb) != 0 || !S_ISREG(sb.st_mode)) return;
  posix_fadvise(fd, 0, 0, POSIX_FADV_SEQUENTIAL);
  JsonlSource src;
  src.fd = fd;
  store_append_jsonl(s, src, static_cast<uint64_t>(sb.st_size), accepted);
}

}  // namespace csg

// Known-answer hooks: the host instantiation of the device line parser.
extern "C" int csg_jsonl_parse_line(const char* line, size_t len, csg_packed_record* out) {
  if (!line || !out) return 0;
  // the kernel's decision: the canonical fast path, else the general parser
  csg::jsonl::Words w;
  if (len >= static_cast<size_t>(csg::jsonl::kMinLine) &&
      csg::jsonl::parse_fast(line, line + len, w)) {
    std::memcpy(out, &w, sizeof(w));
    return 1;
  }
  return len >= static_cast<size_t>(csg::jsonl::kMinLine) &&
                 csg::jsonl::parse_line(line, line + len, *out)
             ? 1
             : 0;
}

extern "C" int csg_jsonl_parse_double(const char* tok, size_t len, double* out) {
  if (!tok || !out || len == 0 || len > 4096) return 0;
  return csg::jsonl::tok_to_double(tok, static_cast<int>(len), *out) ? 1 : 0;
}
