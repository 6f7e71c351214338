// sort.cuh — stable LSD radix sort of (key, u32 value) pairs and a
// device-wide exclusive scan, hand-written for sm_100a.
//
// Used by the store index (rank-major order, the reference's RankIndex of
// proj/src/rca.cpp:77-90 and TraceStore::query's stable (ts, rank) sort of
// proj/src/trace.cpp:112-117) and by the op-ordered completion index that
// serves the straggler self-evidence pass (proj/src/rca.cpp:803-815).
#pragma once

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "engine_internal.h"

namespace csg {

// Per-kernel CUDA-event timing on the launching stream (enabled on demand;
// the benchmark reads it to compute each kernel's achieved bandwidth).
struct Profiler {
  bool enabled = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  struct Rec {
    const char* name;
    cudaEvent_t a, b;
    double host_us;  // host clock at launch (CSG_TIMELINE)
  };
  std::vector<Rec> pending;
  std::map<std::string, std::pair<double, uint64_t>> totals;
  cudaEvent_t take() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  // Call after the stream has been synchronized. CSG_TIMELINE=1 prints
  // every launch (start offset, duration, idle gap before it) to stderr.
  void collect() {
    static const bool tl = std::getenv("CSG_TIMELINE") != nullptr;
    if (tl && !pending.empty()) {
      float prev_end = 0;
      for (const Rec& r : pending) {
        float s0 = 0, e0 = 0;
        if (!r.b || cudaEventElapsedTime(&s0, pending[0].a, r.a) != cudaSuccess ||
            cudaEventElapsedTime(&e0, pending[0].a, r.b) != cudaSuccess)
          continue;
        fprintf(stderr,
                "timeline %-22s start %9.1f us  dur %8.1f us  gap %8.1f us  host %9.1f us"
                "  abs %14.1f\n",
                r.name, s0 * 1e3, (e0 - s0) * 1e3, (s0 - prev_end) * 1e3,
                r.host_us - pending[0].host_us, r.host_us);
        prev_end = e0;
      }
    }
    for (const Rec& r : pending) {
      float ms = 0;
      if (r.b && cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
        auto& t = totals[r.name];
        t.first += ms;
        t.second += 1;
      }
    }
    pending.clear();
    used = 0;
  }
  ~Profiler() {
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
  }
};

// CSG_TIMELINE=1: host-side marks on the same clock as the launch records.
inline void tl_mark(const char* what) {
  static const bool tl = std::getenv("CSG_TIMELINE") != nullptr;
  if (!tl) return;
  const double hus = std::chrono::duration<double, std::micro>(
                         std::chrono::steady_clock::now().time_since_epoch())
                         .count();
  fprintf(stderr, "hostmark %-28s %14.1f us\n", what, hus);
}

struct LaunchCounter {
  uint64_t launches = 0;
  Profiler prof;
};

struct ProfScope {
  LaunchCounter& lc;
  cudaStream_t st;
  bool on;
  const char* name_;
  ProfScope(LaunchCounter& l, const char* name, cudaStream_t s, bool ours = true)
      : lc(l), st(s), on(l.prof.enabled), name_(name) {
    if (ours) ++lc.launches;  // NCCL collectives are timed, not counted
    if (on) {
      cudaEvent_t a = lc.prof.take();
      cudaEventRecord(a, st);
      const double hus = std::chrono::duration<double, std::micro>(
                             std::chrono::steady_clock::now().time_since_epoch())
                             .count();
      lc.prof.pending.push_back({name, a, nullptr, hus});
    }
  }
  ~ProfScope() {
    static const bool sync_each = std::getenv("CSG_SYNC_EACH") != nullptr;
    if (sync_each) {  // debugging aid: name the kernel that faulted
      const cudaError_t e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) fprintf(stderr, "CSG_SYNC_EACH: %s after %s\n",
                                    cudaGetErrorString(e), name_);
    }
    if (on) {
      cudaEvent_t b = lc.prof.take();
      cudaEventRecord(b, st);
      lc.prof.pending.back().b = b;
    }
  }
};

struct SortScratch {
  DevBuf keys2, vals2, counts, scan_tmp;
};

// Stable sort of keys[0,n) (and vals alongside) by bits [0, nbits) of the
// key. nbits may be 0 (no-op). Results land back in keys/vals.
void radix_sort_u32(uint32_t* keys, uint32_t* vals, uint64_t n, int nbits,
                    SortScratch& s, cudaStream_t st, LaunchCounter& lc);
void radix_sort_u64(uint64_t* keys, uint32_t* vals, uint64_t n, int nbits,
                    SortScratch& s, cudaStream_t st, LaunchCounter& lc);

// In-place exclusive prefix sum of u32 (sum must fit u32).
void exclusive_scan_u32(uint32_t* data, uint64_t n, DevBuf& tmp,
                        cudaStream_t st, LaunchCounter& lc);

inline int bits_for(uint64_t max_value) {
  int b = 0;
  while (b < 64 && (max_value >> b) != 0) ++b;
  return b;
}

}  // namespace csg

namespace csg {

// ---- single-pass exclusive scan (decoupled look-back) -----------------------
// out[i] = sum of ld(0 .. i-1) for i < n. Tiles of 4096 values claim an
// order through an atomic ticket, publish their aggregate, look back over
// their predecessors' published aggregates / inclusive prefixes with one warp
// and publish their inclusive prefix: one launch instead of reduce + scan +
// apply. flags: (ntiles + 1) zeroed u64 words (the last one is the ticket).
constexpr int kLbThreads = 256;
constexpr int kLbItems = 16;
constexpr int kLbTile = kLbThreads * kLbItems;

__device__ inline uint32_t lb_block_excl(uint32_t v, uint32_t* wsum, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t s = lane < kLbThreads / 32 ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < kLbThreads / 32) wsum[lane] = s;
  }
  __syncthreads();
  *total = wsum[kLbThreads / 32 - 1];
  return (warp ? wsum[warp - 1] : 0) + x - v;
}

template <typename Load>
__global__ void __launch_bounds__(kLbThreads)
    k_scan_lookback(Load ld, uint64_t n, uint32_t* __restrict__ out,
                    unsigned long long* __restrict__ flags, uint32_t ntiles) {
  __shared__ uint32_t s_tile, s_prefix;
  __shared__ uint32_t wsum[32];
  constexpr unsigned long long AGG = 1ull << 62, INC = 2ull << 62;
  if (threadIdx.x == 0) s_tile = atomicAdd(reinterpret_cast<unsigned*>(flags + ntiles), 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t base = static_cast<uint64_t>(tile) * kLbTile + threadIdx.x * kLbItems;
  uint32_t x[kLbItems];
  uint32_t t = 0;
#pragma unroll
  for (int k = 0; k < kLbItems; ++k) {
    x[k] = base + k < n ? ld(base + k) : 0u;
    t += x[k];
  }
  uint32_t agg;
  const uint32_t off = lb_block_excl(t, wsum, &agg);
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    uint32_t prefix = 0;
    if (tile == 0) {
      if (lane == 0) {
        __threadfence();
        atomicExch(flags + tile, INC | agg);
      }
    } else {
      if (lane == 0) atomicExch(flags + tile, AGG | agg);
      int64_t w = static_cast<int64_t>(tile) - 1;  // window end (closest predecessor)
      while (true) {
        const int64_t q = w - lane;
        unsigned long long f = INC;  // before tile 0: nothing left to add
        if (q >= 0) {
          do {
            f = atomicAdd(flags + q, 0ull);
          } while ((f >> 62) == 0);
        }
        const unsigned inc = __ballot_sync(0xffffffffu, (f >> 62) == 2);
        // lanes up to and including the first inclusive one contribute
        const int stop = inc ? __ffs(inc) - 1 : 31;
        uint32_t v = lane <= stop ? static_cast<uint32_t>(f & 0xffffffffull) : 0u;
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        prefix += v;
        if (inc) break;
        w -= 32;
      }
      if (lane == 0) atomicExch(flags + tile, INC | static_cast<unsigned long long>(prefix + agg));
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  uint32_t run = s_prefix + off;
#pragma unroll
  for (int k = 0; k < kLbItems; ++k) {
    if (base + k < n) out[base + k] = run;
    run += x[k];
  }
}

struct LoadU32 {
  const uint32_t* p;
  __device__ uint32_t operator()(uint64_t i) const { return p[i]; }
};

}  // namespace csg
