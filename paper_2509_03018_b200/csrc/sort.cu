// sort.cu — stable LSD radix sort + exclusive scan for sm_100a.
//
// One pass = upsweep (per-tile 8-bit digit histogram) -> device scan of the
// digit-major histogram -> downsweep. The downsweep ranks every key inside
// its 2048-key tile with warp __match_any_sync (stable: tile order is warp,
// then item, then lane, which is element order), stages the tile in shared
// memory in digit order, and writes each digit run contiguously, so global
// writes come out as ~8-key runs per digit instead of scattered words.
#include "sort.cuh"

namespace csg {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;  // 2048
constexpr int kRadix = 256;
constexpr int kWarps = kThreads / 32;

template <typename K>
__global__ void __launch_bounds__(kThreads)
    k_upsweep(const K* __restrict__ keys, uint64_t n, int shift,
              uint32_t* __restrict__ counts, uint32_t ntiles) {
  __shared__ uint32_t hist[kRadix];
  const int tid = threadIdx.x;
  hist[tid] = 0;
  __syncthreads();
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kTile;
  // every key of the tile loaded before the first match (kItems loads in
  // flight per thread; the guarded load-match-atomic chain serialised them)
  uint32_t d[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t idx = base + static_cast<uint64_t>(i) * kThreads + tid;
    d[i] = idx < n ? static_cast<uint32_t>((keys[idx] >> shift) & 255u) : kRadix;
  }
  // Warp-aggregated increment: one shared atomic per distinct digit (the
  // out-of-range sentinel kRadix is skipped).
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const unsigned peers = __match_any_sync(0xffffffffu, d[i]);
    if (d[i] < kRadix && (threadIdx.x & 31) == __ffs(peers) - 1)
      atomicAdd(&hist[d[i]], __popc(peers));
  }
  __syncthreads();
  counts[static_cast<uint64_t>(tid) * ntiles + blockIdx.x] = hist[tid];
}

__device__ inline uint32_t block_exclusive_scan_256(uint32_t v,
                                                    uint32_t* wsum) {
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
    uint32_t s = lane < kWarps ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < kWarps) wsum[lane] = s;
  }
  __syncthreads();
  const uint32_t before = warp ? wsum[warp - 1] : 0;
  return before + x - v;
}

template <typename K>
__global__ void __launch_bounds__(kThreads)
    k_downsweep(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                K* __restrict__ kout, uint32_t* __restrict__ vout, uint64_t n,
                int shift, const uint32_t* __restrict__ offs,
                uint32_t ntiles) {
  __shared__ uint32_t wcnt[kWarps][kRadix + 1];
  __shared__ uint32_t tile_base[kRadix];
  __shared__ uint32_t gbase[kRadix];
  __shared__ uint32_t wsum[kWarps];
  __shared__ K skeys[kTile];
  __shared__ uint32_t svals[kTile];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kWarps * (kRadix + 1); i += kThreads)
    (&wcnt[0][0])[i] = 0;
  __syncthreads();

  const uint64_t wbase = static_cast<uint64_t>(blockIdx.x) * kTile +
                         static_cast<uint64_t>(warp) * 32 * kItems;
  K k[kItems];
  uint32_t v[kItems];
  uint32_t d[kItems];
  uint32_t r[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t idx = wbase + static_cast<uint64_t>(i) * 32 + lane;
    const bool valid = idx < n;
    k[i] = valid ? kin[idx] : K(0);
    v[i] = valid ? vin[idx] : 0u;
    d[i] = valid ? static_cast<uint32_t>((k[i] >> shift) & 255u) : kRadix;
  }
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const unsigned peers = __match_any_sync(0xffffffffu, d[i]);
    const uint32_t before = wcnt[warp][d[i]];
    r[i] = before + __popc(peers & ((1u << lane) - 1u));
    __syncwarp();
    if (lane == __ffs(peers) - 1) wcnt[warp][d[i]] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {
    const int dd = tid;  // kThreads == kRadix
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = wcnt[w][dd];
      wcnt[w][dd] = run;
      run += c;
    }
    gbase[dd] = offs[static_cast<uint64_t>(dd) * ntiles + blockIdx.x];
    tile_base[dd] = block_exclusive_scan_256(run, wsum);
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    if (d[i] < kRadix) {
      const uint32_t p = tile_base[d[i]] + wcnt[warp][d[i]] + r[i];
      skeys[p] = k[i];
      svals[p] = v[i];
    }
  }
  __syncthreads();
  const uint64_t tbase = static_cast<uint64_t>(blockIdx.x) * kTile;
  const uint32_t tile_n =
      static_cast<uint32_t>(n - tbase < kTile ? n - tbase : kTile);
  for (uint32_t p = tid; p < tile_n; p += kThreads) {
    const K kk = skeys[p];
    const uint32_t dd = static_cast<uint32_t>((kk >> shift) & 255u);
    const uint32_t o = gbase[dd] + (p - tile_base[dd]);
    kout[o] = kk;
    vout[o] = svals[p];
  }
}

constexpr int kScanPer = 4;
constexpr int kScanTile = kThreads * kScanPer;  // 1024

__global__ void __launch_bounds__(kThreads)
    k_scan_block(uint32_t* __restrict__ data, uint64_t n,
                 uint32_t* __restrict__ sums) {
  __shared__ uint32_t wsum[kWarps];
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile +
                        static_cast<uint64_t>(threadIdx.x) * kScanPer;
  uint32_t x[kScanPer];
  uint32_t t = 0;
#pragma unroll
  for (int i = 0; i < kScanPer; ++i) {
    x[i] = base + i < n ? data[base + i] : 0u;
    t += x[i];
  }
  uint32_t run = block_exclusive_scan_256(t, wsum);
#pragma unroll
  for (int i = 0; i < kScanPer; ++i) {
    if (base + i < n) data[base + i] = run;
    run += x[i];
  }
  if (threadIdx.x == kThreads - 1 && sums) sums[blockIdx.x] = run;
}

__global__ void k_scan_add(uint32_t* __restrict__ data, uint64_t n,
                           const uint32_t* __restrict__ sums) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * kScanTile + threadIdx.x;
  const uint32_t add = sums[blockIdx.x];
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) {
    const uint64_t idx = i + static_cast<uint64_t>(j) * kThreads;
    if (idx < n) data[idx] += add;
  }
}

void scan_rec(uint32_t* data, uint64_t n, uint32_t* tmp, cudaStream_t st,
              LaunchCounter& lc) {
  if (n == 0) return;
  const uint64_t nb = (n + kScanTile - 1) / kScanTile;
  {
    ProfScope ps_(lc, "k_scan_block", st);
    k_scan_block<<<static_cast<unsigned>(nb), kThreads, 0, st>>>(
        data, n, nb > 1 ? tmp : nullptr);
  }
  if (nb > 1) {
    scan_rec(tmp, nb, tmp + nb, st, lc);
    {
      ProfScope ps_(lc, "k_scan_add", st);
      k_scan_add<<<static_cast<unsigned>(nb), kThreads, 0, st>>>(data, n, tmp);
    }
  }
}

template <typename K>
void radix_sort_impl(K* keys, uint32_t* vals, uint64_t n, int nbits,
                     SortScratch& s, cudaStream_t st, LaunchCounter& lc) {
  if (n <= 1 || nbits <= 0) return;
  const uint32_t ntiles = static_cast<uint32_t>((n + kTile - 1) / kTile);
  s.keys2.ensure(n * sizeof(K));
  s.vals2.ensure(n * sizeof(uint32_t));
  const uint64_t nc = static_cast<uint64_t>(kRadix) * ntiles;
  s.counts.ensure(nc * sizeof(uint32_t));
  s.scan_tmp.ensure((nc / (kScanTile - 1) + 64) * sizeof(uint32_t));
  K* ka = keys;
  uint32_t* va = vals;
  K* kb = s.keys2.as<K>();
  uint32_t* vb = s.vals2.as<uint32_t>();
  int passes = 0;
  for (int shift = 0; shift < nbits; shift += 8, ++passes) {
    {
      ProfScope ps_(lc, "k_upsweep", st);
      k_upsweep<K><<<ntiles, kThreads, 0, st>>>(ka, n, shift,
                                                s.counts.as<uint32_t>(), ntiles);
    }
    scan_rec(s.counts.as<uint32_t>(), nc, s.scan_tmp.as<uint32_t>(), st, lc);
    {
      ProfScope ps_(lc, "k_downsweep", st);
      k_downsweep<K><<<ntiles, kThreads, 0, st>>>(
          ka, va, kb, vb, n, shift, s.counts.as<uint32_t>(), ntiles);
    }
    K* tk = ka; ka = kb; kb = tk;
    uint32_t* tv = va; va = vb; vb = tv;
  }
  if (passes & 1) {
    CSG_CUDA(cudaMemcpyAsync(keys, ka, n * sizeof(K), cudaMemcpyDeviceToDevice, st));
    CSG_CUDA(cudaMemcpyAsync(vals, va, n * sizeof(uint32_t),
                             cudaMemcpyDeviceToDevice, st));
  }
  CSG_CUDA(cudaGetLastError());
}

}  // namespace

void radix_sort_u32(uint32_t* keys, uint32_t* vals, uint64_t n, int nbits,
                    SortScratch& s, cudaStream_t st, LaunchCounter& lc) {
  radix_sort_impl<uint32_t>(keys, vals, n, nbits, s, st, lc);
}

void radix_sort_u64(uint64_t* keys, uint32_t* vals, uint64_t n, int nbits,
                    SortScratch& s, cudaStream_t st, LaunchCounter& lc) {
  radix_sort_impl<uint64_t>(keys, vals, n, nbits, s, st, lc);
}

void exclusive_scan_u32(uint32_t* data, uint64_t n, DevBuf& tmp,
                        cudaStream_t st, LaunchCounter& lc) {
  if (n == 0) return;
  const uint32_t nt = static_cast<uint32_t>((n + kLbTile - 1) / kLbTile);
  tmp.ensure((static_cast<size_t>(nt) + 1) * 8);
  CSG_CUDA(cudaMemsetAsync(tmp.p, 0, (static_cast<size_t>(nt) + 1) * 8, st));
  {
    ProfScope ps_(lc, "k_scan_lookback", st);
    k_scan_lookback<<<nt, kLbThreads, 0, st>>>(LoadU32{data}, n, data,
                                               tmp.as<unsigned long long>(), nt);
  }
  CSG_CUDA(cudaGetLastError());
}

}  // namespace csg
