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
  ProfScope(LaunchCounter& l, const char* name, cudaStream_t s)
      : lc(l), st(s), on(l.prof.enabled) {
    ++lc.launches;
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
