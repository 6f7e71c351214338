// sort.cuh — stable LSD radix sort of (key, u32 value) pairs and a
// device-wide exclusive scan, hand-written for sm_100a.
//
// Used by the store index (rank-major order, the reference's RankIndex of
// proj/src/rca.cpp:77-90 and TraceStore::query's stable (ts, rank) sort of
// proj/src/trace.cpp:112-117) and by the op-ordered completion index that
// serves the straggler self-evidence pass (proj/src/rca.cpp:803-815).
#pragma once

#include "engine_internal.h"

namespace csg {

struct LaunchCounter {
  uint64_t launches = 0;
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
