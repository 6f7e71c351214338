// fetch.cuh — device side of the mapped-memory fetch (ctx_fetch_issue /
// ctx_sync): copy the segments into pinned host memory, then raise the
// completion word the host polls.
#pragma once

#include "objects.h"

namespace csg {

// The segments' copies, shared by threads gt of nt.
__device__ inline void fetch_copy(const FetchArgs& a, uint32_t gt, uint32_t nt) {
  for (int sgi = 0; sgi < a.n; ++sgi) {
    const FetchSeg& g = a.seg[sgi];
    if (g.row_len) {  // rows with device-side lengths, one warp per row
      const int lane = threadIdx.x & 31;
      for (uint32_t rw = gt >> 5; rw < g.nrows; rw += nt >> 5) {
        const uint32_t* s4 = reinterpret_cast<const uint32_t*>(g.src + rw * g.bytes);
        uint32_t* d4 = reinterpret_cast<uint32_t*>(g.dst + rw * g.bytes);
        const int32_t len = g.row_len[rw];
        for (int32_t i = lane; i < len; i += 32) d4[i] = s4[i];
      }
      continue;
    }
    const bool vec = ((reinterpret_cast<uintptr_t>(g.src) | reinterpret_cast<uintptr_t>(g.dst) |
                       g.bytes) & 15) == 0;
    if (vec) {
      const uint4* s4 = reinterpret_cast<const uint4*>(g.src);
      uint4* d4 = reinterpret_cast<uint4*>(g.dst);
      for (uint32_t i = gt; i < g.bytes / 16; i += nt) d4[i] = s4[i];
    } else {
      for (uint32_t i = gt; i < g.bytes; i += nt) g.dst[i] = g.src[i];
    }
  }
}

// Every block of the calling grid, at its end: the last block to arrive
// (device-side counter `done`, zero between fetches) does the copies and
// raises the completion word — a kernel's own tail instead of a k_fetch
// launch behind it.
__device__ inline void fetch_tail(const FetchArgs& a, unsigned long long* flag,
                                  unsigned long long v, unsigned* done,
                                  bool wrote_host = true) {
  __shared__ unsigned s_last;
  // this block's own writes first (system scope if it wrote mapped memory:
  // the host reads them once the completion word is up)
  if (wrote_host) __threadfence_system();
  else __threadfence();
  __syncthreads();
  if (threadIdx.x == 0)
    s_last = atomicAdd(done, 1u) == gridDim.x * gridDim.y * gridDim.z - 1 ? 1u : 0u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  fetch_copy(a, threadIdx.x, blockDim.x);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    *done = 0;  // ready for the next fetch
    __threadfence_system();
    *reinterpret_cast<volatile unsigned long long*>(flag) = v;
    __threadfence_system();
  }
}

}  // namespace csg
