// store.cu — device TraceStore: ingest statistics, the rank-major index and
// the store queries.
//
// Reference semantics (proj/src/trace.cpp:99-144, proj/src/rca.cpp:77-90):
// the store index is emission order; RankIndex lists each rank's records in
// store order. Here the index is one stable radix sort by rank (store order
// preserved inside a rank), a gather of the packed records into rank-major
// structure-of-arrays columns, and a per-rank running maximum of the
// timestamp. The running max is monotone even though per-rank timestamps are
// not, so every reference "prefix scan that breaks at the
// first ts > t" becomes one upper_bound over it.
#include <cuda.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "comm.cuh"
#include "objects.h"
#include "fetch.cuh"

namespace csg {
namespace {

__device__ inline void atomic_max_u64(unsigned long long* a, unsigned long long v) {
  atomicMax(a, v);
}

// Store statistics accumulated per thread, reduced per block, committed with
// one set of global atomics per block: max timestamp (ordered key), rank /
// channel / op ranges, NaN count.
struct StatAcc {
  unsigned long long tsk = 0, nan = 0;
  int mnr = INT_MAX, mxr = INT_MIN, mnc = INT_MAX, mxc = INT_MIN;
  long long mno = LLONG_MAX, mxo = LLONG_MIN;
  __device__ void add(double t, long long op, int rank, int chan) {
    if (t != t) ++nan; else tsk = max(tsk, (unsigned long long)dkey(t));
    mnr = min(mnr, rank);
    mxr = max(mxr, rank);
    mnc = min(mnc, chan);
    mxc = max(mxc, chan);
    mno = min(mno, op);
    mxo = max(mxo, op);
  }
  __device__ void commit(StoreStats* st) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      tsk = max(tsk, __shfl_xor_sync(0xffffffffu, tsk, o));
      mnr = min(mnr, __shfl_xor_sync(0xffffffffu, mnr, o));
      mxr = max(mxr, __shfl_xor_sync(0xffffffffu, mxr, o));
      mnc = min(mnc, __shfl_xor_sync(0xffffffffu, mnc, o));
      mxc = max(mxc, __shfl_xor_sync(0xffffffffu, mxc, o));
      mno = min(mno, __shfl_xor_sync(0xffffffffu, mno, o));
      mxo = max(mxo, __shfl_xor_sync(0xffffffffu, mxo, o));
      nan += __shfl_xor_sync(0xffffffffu, nan, o);
    }
    __shared__ StatAcc sw[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) sw[warp] = *this;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
        tsk = max(tsk, sw[w].tsk);
        nan += sw[w].nan;
        mnr = min(mnr, sw[w].mnr);
        mxr = max(mxr, sw[w].mxr);
        mnc = min(mnc, sw[w].mnc);
        mxc = max(mxc, sw[w].mxc);
        mno = min(mno, sw[w].mno);
        mxo = max(mxo, sw[w].mxo);
      }
      atomic_max_u64(&st->ts_max_key, tsk);
      atomicMin(&st->min_rank, mnr);
      atomicMax(&st->max_rank, mxr);
      atomicMin(&st->lmin_rank, mnr);
      atomicMax(&st->lmax_rank, mxr);
      atomicMin(&st->min_chan, mnc);
      atomicMax(&st->max_chan, mxc);
      atomicMin(&st->min_op, mno);
      atomicMax(&st->max_op, mxo);
      if (nan) atomicAdd(&st->n_nan, nan);
    }
  }
};

// Fields the index reads from one packed record's first 32 bytes.
__device__ inline void rec_head(const csg_packed_record* r, uint64_t i, ulonglong2& h0,
                                ulonglong2& hm) {
  const ulonglong2* rec = reinterpret_cast<const ulonglong2*>(r + i);
  h0 = __ldg(rec);
  hm = __ldg(rec + 1);
}

// One pass over the packed records: store statistics and the (rank, store
// index) sort pairs (general index path, rank spans > kHistDigits).
__global__ void k_stats_keys(const csg_packed_record* __restrict__ r, uint64_t n,
                             StoreStats* __restrict__ st,
                             uint32_t* __restrict__ keys,
                             uint32_t* __restrict__ vals) {
  StatAcc acc;
  // 4 records in flight per thread (independent 16-byte loads) to keep
  // enough bytes outstanding for HBM.
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i0 < n;
       i0 += 4 * stride) {
    ulonglong2 h0[4], hm[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t i = i0 + k * stride;
      if (i < n) rec_head(r, i, h0[k], hm[k]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t i = i0 + k * stride;
      if (i >= n) break;
      double t;
      memcpy(&t, &h0[k].x, 8);
      const int rank = static_cast<int>(hm[k].x & 0xffffffffu);
      acc.add(t, static_cast<long long>(h0[k].y), rank,
              static_cast<int>(hm[k].y & 0xffffffffu));
      keys[i] = static_cast<uint32_t>(rank);
      vals[i] = static_cast<uint32_t>(i);
    }
  }
  acc.commit(st);
}

// ---- fused rank-major index (rank span <= kHistDigits) ----------------------
//
// The reference's RankIndex (proj/src/rca.cpp:77-90: every rank's records in
// store order) as ONE stable counting-sort pass over 11-bit rank digits:
//   k_stats_hist  statistics + per-tile digit histogram (digit = rank & 2047),
//                 written digit-major (L2-resident, 2048 x tiles words)
//   k_hist_scan*  exclusive scan in (rank - min_rank, tile) order (the
//                 rotation by min_rank & 2047 makes the digit order the rank
//                 order for any span <= 2048, e.g. a shard's rank range)
//   k_scatter     per tile: stable local ranking (warp match_any), digit-
//                 ordered staging of tile indices in shared memory, then each
//                 record is read once and written once into the rank-major
//                 SoA columns in contiguous digit runs.
constexpr int kHistDigits = 2048;
constexpr int kTileThreads = 256;
constexpr int kTileItems = 16;
constexpr int kTile = kTileThreads * kTileItems;  // 4096 records
constexpr uint32_t kScatterCtas = 148;  // persistent scatter: one CTA per SM
constexpr uint32_t kHistChunks = 148;   // tile chunks of the histogram scan (<= 256)

__global__ void __launch_bounds__(kTileThreads, 2)
    k_stats_hist(const csg_packed_record* __restrict__ r, uint64_t n,
                 StoreStats* __restrict__ st, uint32_t* __restrict__ counts,
                 FetchArgs fa, unsigned long long* flag, unsigned long long v,
                 unsigned* __restrict__ fdone) {
  __shared__ __align__(16) uint32_t hist[kHistDigits];
  for (int d = threadIdx.x; d < kHistDigits; d += kTileThreads) hist[d] = 0;
  StatAcc acc;
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kTile;
  // every load of the tile issued before the first use (32 x 16 B per thread
  // in flight: the kernel is a pure HBM stream)
  ulonglong2 h0[kTileItems], hm[kTileItems];
#pragma unroll
  for (int k = 0; k < kTileItems; ++k) {
    const uint64_t i = base + k * kTileThreads + threadIdx.x;
    if (i < n) rec_head(r, i, h0[k], hm[k]);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kTileItems; ++k) {
    const uint64_t i = base + k * kTileThreads + threadIdx.x;
    const bool valid = i < n;
    double t = 0;
    int rank = 0;
    if (valid) {
      memcpy(&t, &h0[k].x, 8);
      rank = static_cast<int>(hm[k].x & 0xffffffffu);
      acc.add(t, static_cast<long long>(h0[k].y), rank,
              static_cast<int>(hm[k].y & 0xffffffffu));
    }
    const uint32_t d = valid ? static_cast<uint32_t>(rank) & (kHistDigits - 1)
                             : 0xFFFFFFFFu;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (valid && (threadIdx.x & 31) == __ffs(peers) - 1)
      atomicAdd(&hist[d], __popc(peers));
  }
  __syncthreads();
  // tile-major row of 2048 digit counts: one coalesced 8 KB store per tile
  uint4* row = reinterpret_cast<uint4*>(counts + static_cast<uint64_t>(blockIdx.x) * kHistDigits);
  const uint4* h4 = reinterpret_cast<const uint4*>(hist);
  for (int d = threadIdx.x; d < kHistDigits / 4; d += kTileThreads) row[d] = h4[d];
  acc.commit(st);
  // flag set: the statistics travel to the host from the last block (no
  // k_fetch launch between this pass and the speculative scatter)
  if (flag) fetch_tail(fa, flag, v, fdone, false);
}

__device__ inline uint32_t block_excl_scan_u32(uint32_t v, uint32_t* wsum, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t s = lane < nw ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) wsum[lane] = s;
  }
  __syncthreads();
  if (total) *total = wsum[nw - 1];
  const uint32_t before = warp ? wsum[warp - 1] : 0;
  const uint32_t r = before + x - v;
  __syncthreads();
  return r;
}

// Per-tile digit counts (tile-major, counts[t][d]) -> scatter bases
// goff[t][j] = sum of all records with rotated digit < j + records of digit
// j in tiles < t (j = (d - d0) & 2047, i.e. rank - min_rank for spans <=
// 2048). Three coalesced passes over chunks of tpc consecutive tiles:
//   k_hist_colsum     per chunk and digit: csum[c][j]
//   k_hist_chunkscan  per digit, exclusive over chunks (in place) + tot[j]
//   k_hist_apply      per chunk: digit bases (block scan of tot) + chunk
//                     prefix, then a running sum over the chunk's tiles
__global__ void __launch_bounds__(1024)
    k_hist_colsum(const uint32_t* __restrict__ counts, uint32_t ntiles, uint32_t tpc,
                  uint32_t d0, int D, uint32_t* __restrict__ csum, const int* go) {
  pdl_wait();
  pdl_trigger();
  if (go && !*go) return;  // speculative launch on a layout that did not hold
  const uint32_t c = blockIdx.x;
  const uint32_t t0 = c * tpc, t1 = min(t0 + tpc, ntiles);
  for (int j = threadIdx.x; j < D; j += blockDim.x) {
    const uint32_t d = (j + d0) & (kHistDigits - 1);
    uint32_t sum = 0;
#pragma unroll 8
    for (uint32_t t = t0; t < t1; ++t) sum += __ldg(counts + static_cast<uint64_t>(t) * kHistDigits + d);
    csum[static_cast<uint64_t>(c) * D + j] = sum;
  }
}

// 32 digits per block (lane = digit), the chunks split into 8 contiguous
// ranges (one per warp): range sums, an exclusive scan over the 8 ranges in
// shared memory, then each warp rewrites its range as prefixes.
__global__ void __launch_bounds__(256)
    k_hist_chunkscan(uint32_t* __restrict__ csum, uint32_t nchunks, int D,
                     uint32_t* __restrict__ tot, const int* go) {
  pdl_wait();
  pdl_trigger();
  if (go && !*go) return;
  __shared__ uint32_t part[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + lane;
  const uint32_t per = (nchunks + 7) / 8;
  const uint32_t c0 = min(warp * per, nchunks), c1 = min(c0 + per, nchunks);
  // nchunks <= 256: a warp's range (<= 32 chunks) stays in registers
  uint32_t v[32];
  uint32_t sum = 0;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const uint32_t c = c0 + k;
    v[k] = j < D && c < c1 ? csum[static_cast<uint64_t>(c) * D + j] : 0u;
    sum += v[k];
  }
  part[warp][lane] = sum;
  __syncthreads();
  uint32_t run = 0;
  for (int w = 0; w < warp; ++w) run += part[w][lane];
  if (warp == 7 && j < D) tot[j] = run + sum;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const uint32_t c = c0 + k;
    if (j < D && c < c1) csum[static_cast<uint64_t>(c) * D + j] = run;
    run += v[k];
  }
}

__global__ void __launch_bounds__(1024)
    k_hist_apply(const uint32_t* __restrict__ counts, const uint32_t* __restrict__ cpre,
                 const uint32_t* __restrict__ tot, uint32_t ntiles, uint32_t tpc, uint32_t d0,
                 int D, uint32_t* __restrict__ goff, const int* go) {
  pdl_wait();
  pdl_trigger();
  if (go && !*go) return;
  __shared__ uint32_t base[kHistDigits];
  __shared__ uint32_t wsum[32];
  const int t2 = 2 * threadIdx.x;
  const uint32_t a = t2 < D ? tot[t2] : 0u, b = t2 + 1 < D ? tot[t2 + 1] : 0u;
  const uint32_t e = block_excl_scan_u32(a + b, wsum, nullptr);
  base[t2] = e;
  base[t2 + 1] = e + a;
  __syncthreads();
  const uint32_t c = blockIdx.x;
  const uint32_t t0 = c * tpc, t1 = min(t0 + tpc, ntiles);
  for (int j = threadIdx.x; j < D; j += blockDim.x) {
    const uint32_t d = (j + d0) & (kHistDigits - 1);
    uint32_t run = base[j] + cpre[static_cast<uint64_t>(c) * D + j];
#pragma unroll 4
    for (uint32_t t = t0; t < t1; ++t) {
      goff[static_cast<uint64_t>(t) * D + j] = run;
      run += __ldg(counts + static_cast<uint64_t>(t) * kHistDigits + d);
    }
  }
}

// Packs the store statistics into order-preserving u64 images (dir 0) so
// one MAX all-reduce combines every extremum across shards (minima travel
// as complements), counts into a SUM pair; dir 1 unpacks the reduced
// values (the shard's own lmin/lmax_rank stay local).
__device__ inline unsigned long long i64_key(long long v) {
  return static_cast<unsigned long long>(v) ^ 0x8000000000000000ull;
}
__device__ inline long long key_i64(unsigned long long k) {
  return static_cast<long long>(k ^ 0x8000000000000000ull);
}
// Sharded statistics as u64 images: pk[0, 7 + 2P) combine by MAX (minima as
// complements; slots 7 + 2i, 8 + 2i carry shard i's own rank range, zero
// elsewhere, so the MAX is an all-gather of the ranges), pk[7 + 2P, 9 + 2P)
// by SUM.
__global__ void k_stats_pack(StoreStats* st, unsigned long long* pk, int dir, int P,
                             int me) {
  if (threadIdx.x || blockIdx.x) return;
  unsigned long long* sum = pk + 7 + 2 * P;
  if (dir == 0) {
    pk[0] = st->ts_max_key;
    pk[1] = ~i64_key(st->min_rank);
    pk[2] = i64_key(st->max_rank);
    pk[3] = ~i64_key(st->min_chan);
    pk[4] = i64_key(st->max_chan);
    pk[5] = ~i64_key(st->min_op);
    pk[6] = i64_key(st->max_op);
    for (int i = 0; i < P; ++i) {
      const bool own = i == me && st->lmin_rank <= st->lmax_rank;  // empty shard: none
      pk[7 + 2 * i] = own ? i64_key(st->lmin_rank) : 0ull;
      pk[8 + 2 * i] = own ? i64_key(st->lmax_rank) : 0ull;
    }
    sum[0] = st->n_nan;
    sum[1] = st->n_total;
  } else {
    st->ts_max_key = pk[0];
    st->min_rank = static_cast<int>(key_i64(~pk[1]));
    st->max_rank = static_cast<int>(key_i64(pk[2]));
    st->min_chan = static_cast<int>(key_i64(~pk[3]));
    st->max_chan = static_cast<int>(key_i64(pk[4]));
    st->min_op = key_i64(~pk[5]);
    st->max_op = key_i64(pk[6]);
    st->n_nan = sum[0];
    st->n_total = sum[1];
    // a rank split across shards would make the RCA's sum all-reduces of
    // per-rank tables add two shards' timestamps: shards must own disjoint
    // rank ranges
    unsigned ov = 0;
    for (int i = 0; i < P; ++i)
      for (int j = i + 1; j < P; ++j) {
        if (!pk[7 + 2 * i] || !pk[7 + 2 * j]) continue;
        const long long lo_i = key_i64(pk[7 + 2 * i]), hi_i = key_i64(pk[8 + 2 * i]);
        const long long lo_j = key_i64(pk[7 + 2 * j]), hi_j = key_i64(pk[8 + 2 * j]);
        if (lo_i <= hi_j && lo_j <= hi_i) ov = 1;
      }
    st->overlap = ov;
  }
}

__device__ int g_scatter_prof_on;
__device__ unsigned long long g_scatter_cyc[6];

struct ScatterOut {
  ulonglong2* tso;  // {ts, op_seq}
  uint4* meta;      // {comm, channel, store index (payload via it), kind | op_name << 1}
};

// The rank-major meta word of a packed record's second 16 bytes (rank |
// comm << 32, channel | kind << 32 | op_name << 40) and its store index.
__device__ __forceinline__ uint4 meta_of(const ulonglong2& hm, uint32_t idx) {
  const uint32_t kind = static_cast<uint32_t>((hm.y >> 32) & 0xff);
  const uint32_t name = static_cast<uint32_t>((hm.y >> 40) & 0xff);
  return make_uint4(static_cast<uint32_t>(hm.x >> 32), static_cast<uint32_t>(hm.y & 0xffffffffu),
                    idx, (kind & 1) | (name << 1));
}

// --- 1D bulk async copies (TMA engine) into shared memory, mbarrier-tracked
__device__ inline uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ inline void mbar_init(unsigned long long* m, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ inline void bulk_load(void* dst, const void* src, uint32_t bytes,
                                 unsigned long long* m) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile(
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)),
      "r"(bytes)
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
      "[%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(m))
      : "memory");
}
__device__ inline void mbar_wait(unsigned long long* m, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(m)), "r"(parity)
        : "memory");
  }
}

// Persistent scatter: every block walks its histogram tiles (kTile records)
// as sub-tiles of 256 x ITEMS records, double-buffered in shared memory by
// bulk async copies, so each packed record is read from HBM exactly once and
// coalesced. Per sub-tile: digits from shared memory, stable warp ranking
// (match_any), digit-ordered staging of sub-tile indices, then every record
// is written once into the rank-major SoA columns in contiguous digit runs.
// bx[d] carries the running global base of digit d through the sub-tiles of
// one histogram tile.
template <int ITEMS, int NBUF, int DPT>
__global__ void __launch_bounds__(kTileThreads, NBUF == 1 ? 3 : 1)
    k_scatter(const csg_packed_record* __restrict__ r, uint64_t n,
              const uint32_t* __restrict__ goff, uint32_t T, int32_t min_rank,
              int32_t D, ScatterOut o, int32_t max_rank, int32_t R,
              uint32_t* __restrict__ rank_off, const int* go) {
  pdl_wait();
  pdl_trigger();
  if (go && !*go) return;
  // CSG_DEBUG_SCATTER: per-phase cycle totals (thread 0 of every block)
  const bool prof = g_scatter_prof_on && threadIdx.x == 0;
  long long pc[6] = {0, 0, 0, 0, 0, 0};
  constexpr int kW = kTileThreads / 32;
  constexpr int TR = kTileThreads * ITEMS;
  constexpr int SUB = kTile / TR;
  constexpr int Dp = DPT * kTileThreads;  // padded digit stride (DPT per thread)
  extern __shared__ __align__(128) unsigned char dyn[];
  unsigned char* buf0 = dyn;
  uint16_t* wc = reinterpret_cast<uint16_t*>(dyn + NBUF * TR * 48);  // [kW][Dp]
  uint32_t* bx = reinterpret_cast<uint32_t*>(wc + kW * Dp);           // [Dp]
  __shared__ uint16_t sidx[TR];
  __shared__ uint32_t wsum[32];
  __shared__ __align__(8) unsigned long long mbar[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // segment offsets over absolute ranks [0, R] from the scanned tile
  // offsets (folded in here: one launch less)
  for (int32_t r = blockIdx.x * kTileThreads + tid; r <= R; r += gridDim.x * kTileThreads)
    rank_off[r] = r < min_rank ? 0u
                  : r > max_rank ? static_cast<uint32_t>(n)
                                 : goff[r - min_rank];
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
  }
  __syncthreads();
  // tiles round-robin over the persistent blocks: the blocks advance through
  // the store together, so each rank's write front stays compact in L2
  auto sub_of = [&](uint32_t j, uint32_t& t, uint64_t& first, uint32_t& cnt) {
    t = blockIdx.x + (j / SUB) * gridDim.x;
    first = static_cast<uint64_t>(t) * kTile + static_cast<uint64_t>(j % SUB) * TR;
    cnt = first < n ? static_cast<uint32_t>(n - first < static_cast<uint64_t>(TR) ? n - first : static_cast<uint64_t>(TR)) : 0u;
    return t < T;
  };
  auto issue = [&](uint32_t j) {
    uint32_t t, cnt;
    uint64_t first;
    const int b = NBUF == 2 ? (j & 1) : 0;
    if (tid == 0 && sub_of(j, t, first, cnt) && cnt)
      bulk_load(buf0 + b * TR * 48, r + first, cnt * 48, &mbar[b]);
  };
  uint32_t par0 = 0, par1 = 0;
  if (NBUF == 2) issue(0);
  for (uint32_t j = 0;; ++j) {
    uint32_t t, cnt;
    uint64_t first;
    if (!sub_of(j, t, first, cnt)) break;
    // double buffer: prefetch the next sub-tile into the buffer released by
    // the barrier ending j - 1; single buffer (several CTAs per SM cover
    // each other's load latency): load this one now
    issue(NBUF == 2 ? j + 1 : j);
    // a new histogram tile starts from its scanned global bases (one
    // contiguous row): loaded now, consumed after phase A (latency hidden)
    const bool fresh = j % SUB == 0;
    uint32_t g0[DPT];
    if (fresh) {
#pragma unroll
      for (int k = 0; k < DPT; ++k) {
        const int dd = tid * DPT + k;
        g0[k] = dd < D ? __ldg(goff + static_cast<uint64_t>(t) * D + dd) : 0u;
      }
    }
    if (cnt == 0) {
      if (fresh)
#pragma unroll
        for (int k = 0; k < DPT; ++k) bx[tid * DPT + k] = g0[k];
      __syncthreads();
      continue;
    }
    const unsigned char* sb = buf0 + (NBUF == 2 ? (j & 1) : 0) * TR * 48;
    {  // clear the warp counters, 16 bytes per store
      uint4* w4 = reinterpret_cast<uint4*>(wc);
      constexpr int n4 = kW * Dp * 2 / 16;
      for (int i = tid; i < n4; i += kTileThreads) w4[i] = make_uint4(0, 0, 0, 0);
    }
    long long pc0 = prof ? clock64() : 0;
    if (NBUF == 2 && (j & 1)) {
      mbar_wait(&mbar[1], par1);
      par1 ^= 1;
    } else {
      mbar_wait(&mbar[0], par0);
      par0 ^= 1;
    }
    __syncthreads();
    if (prof) {
      const long long c = clock64();
      pc[0] += c - pc0;
      pc0 = c;
    }
    // Phase A: warp w owns sub-tile records [32*ITEMS*w, 32*ITEMS*(w+1)),
    // item k of lane l is record 32*ITEMS*w + 32k + l (record order).
    uint32_t d[ITEMS];
    uint16_t rk[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const uint32_t li = warp * (32 * ITEMS) + k * 32 + lane;
      d[k] = li < cnt ? static_cast<uint32_t>(
                            *reinterpret_cast<const int32_t*>(sb + li * 48 + 16) - min_rank)
                      : 0xFFFFFFFFu;
    }
    uint16_t* mine = wc + warp * Dp;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const bool valid = d[k] != 0xFFFFFFFFu;
      const unsigned peers = __match_any_sync(0xffffffffu, d[k]);
      const uint32_t before = valid ? mine[d[k]] : 0u;
      rk[k] = static_cast<uint16_t>(before + __popc(peers & ((1u << lane) - 1u)));
      __syncwarp();
      if (valid && lane == __ffs(peers) - 1)
        mine[d[k]] = static_cast<uint16_t>(before + __popc(peers));
      __syncwarp();
    }
    __syncthreads();
    if (prof) {
      const long long c = clock64();
      pc[1] += c - pc0;
      pc0 = c;
    }
    // per digit (thread t owns digits [DPT*t, DPT*t + DPT), one vector load
    // per warp row): cross-warp prefix + sub-tile start folded into the
    // warp counters; bx becomes (running base - sub-tile start) for phase B
    using VecT = typename std::conditional<DPT == 8, uint4, uint2>::type;
    union DV {
      VecT v;
      uint16_t h[DPT];
    };
    uint32_t tot[DPT];
#pragma unroll
    for (int k = 0; k < DPT; ++k) tot[k] = 0;
#pragma unroll
    for (int w = 0; w < kW; ++w) {
      DV x;
      x.v = *reinterpret_cast<const VecT*>(wc + w * Dp + tid * DPT);
#pragma unroll
      for (int k = 0; k < DPT; ++k) tot[k] += x.h[k];
    }
    uint32_t mysum = 0;
#pragma unroll
    for (int k = 0; k < DPT; ++k) mysum += tot[k];
    uint32_t ts0[DPT];
    ts0[0] = block_excl_scan_u32(mysum, wsum, nullptr);
#pragma unroll
    for (int k = 1; k < DPT; ++k) ts0[k] = ts0[k - 1] + tot[k - 1];
    {
      uint32_t run[DPT];
#pragma unroll
      for (int k = 0; k < DPT; ++k) run[k] = ts0[k];
#pragma unroll
      for (int w = 0; w < kW; ++w) {
        DV x, y;
        x.v = *reinterpret_cast<const VecT*>(wc + w * Dp + tid * DPT);
#pragma unroll
        for (int k = 0; k < DPT; ++k) {
          y.h[k] = static_cast<uint16_t>(run[k]);
          run[k] += x.h[k];
        }
        *reinterpret_cast<VecT*>(wc + w * Dp + tid * DPT) = y.v;
      }
    }
    uint32_t nxt[DPT];
#pragma unroll
    for (int k = 0; k < DPT; ++k) {
      const int dd = tid * DPT + k;
      const uint32_t rb = fresh ? g0[k] : bx[dd];
      nxt[k] = rb + tot[k];
      bx[dd] = rb - ts0[k];
    }
    __syncthreads();
    if (prof) {
      const long long c = clock64();
      pc[2] += c - pc0;
      pc0 = c;
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k)
      if (d[k] != 0xFFFFFFFFu)
        sidx[mine[d[k]] + rk[k]] = static_cast<uint16_t>(warp * (32 * ITEMS) + k * 32 + lane);
    __syncthreads();
    if (prof) {
      const long long c = clock64();
      pc[3] += c - pc0;
      pc0 = c;
    }
    // Phase B: digit order; consecutive threads write consecutive positions
    // of one digit run. Four records per thread in flight (independent
    // shared-memory chains; 8 warps per SM leave little else to hide them).
    constexpr int kB = 4;
    for (uint32_t p0 = tid; p0 < cnt; p0 += kB * kTileThreads) {
      uint32_t li[kB], q[kB];
      ulonglong2 h0[kB], hm[kB];
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        const uint32_t p = p0 + k * kTileThreads;
        li[k] = p < cnt ? sidx[p] : 0u;
      }
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        const ulonglong2* rec = reinterpret_cast<const ulonglong2*>(sb + li[k] * 48);
        h0[k] = rec[0];
        hm[k] = rec[1];
      }
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        const uint32_t p = p0 + k * kTileThreads;
        const int32_t rank = static_cast<int32_t>(hm[k].x & 0xffffffffu);
        q[k] = bx[static_cast<uint32_t>(rank - min_rank)] + p;
      }
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        const uint32_t p = p0 + k * kTileThreads;
        if (p >= cnt) break;
        const uint32_t qq = q[k];
        o.tso[qq] = h0[k];
        o.meta[qq] = meta_of(hm[k], static_cast<uint32_t>(first + li[k]));
      }
    }
    __syncthreads();
    if (prof) {
      pc[4] += clock64() - pc0;
      pc[5] += 1;
    }
#pragma unroll
    for (int k = 0; k < DPT; ++k) bx[tid * DPT + k] = nxt[k];
    __syncthreads();
  }
  if (prof)
    for (int q = 0; q < 6; ++q) atomicAdd(&g_scatter_cyc[q], static_cast<unsigned long long>(pc[q]));
}

// k_scatter with 2-D tensor copies: the TMA engine gathers only the first 32
// bytes of each 48-byte record (the fields the index writes; the payload is
// read later through perm) into dense 32-byte shared-memory rows, which
// leaves room for 16 warps per SM next to two 2048-record buffers (the 1-D
// bulk variant holds whole records and runs 8). Same ranking and write
// phases as k_scatter; tile-major bases, round-robin tiles.
constexpr int kTxThreads = 512;
constexpr int kTxItems = 4;
constexpr int kTxRows = kTxThreads * kTxItems;  // 2048-record sub-tile
constexpr int kTxBox = 256;                     // rows per tensor copy

__device__ inline void tensor_load_2d(void* dst, const CUtensorMap* tm, int x, int y,
                                      unsigned long long* m) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(m))
      : "memory");
}

template <int DPT>
__global__ void __launch_bounds__(kTxThreads, 1)
    k_scatter_tx(const __grid_constant__ CUtensorMap tm, uint64_t n,
                 const uint32_t* __restrict__ goff, uint32_t T, int32_t min_rank,
                 int32_t D, ScatterOut o, int32_t max_rank, int32_t R,
                 uint32_t* __restrict__ rank_off, const int* go) {
  if (go && !*go) return;
  constexpr int kW = kTxThreads / 32;
  constexpr int SUB = kTile / kTxRows;
  constexpr int Dp = DPT * kTxThreads;
  extern __shared__ __align__(128) unsigned char dyn[];
  unsigned char* buf0 = dyn;                                             // [2][2048][32]
  uint16_t* wc = reinterpret_cast<uint16_t*>(dyn + 2 * kTxRows * 32);  // [kW][Dp]
  uint32_t* bx = reinterpret_cast<uint32_t*>(wc + kW * Dp);            // [Dp]
  __shared__ uint16_t sidx[kTxRows];
  __shared__ uint32_t wsum[32];
  __shared__ __align__(8) unsigned long long mbar[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int32_t r = blockIdx.x * kTxThreads + tid; r <= R; r += gridDim.x * kTxThreads)
    rank_off[r] = r < min_rank ? 0u
                  : r > max_rank ? static_cast<uint32_t>(n)
                                 : goff[r - min_rank];
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
  }
  __syncthreads();
  auto sub_of = [&](uint32_t j, uint32_t& t, uint64_t& first, uint32_t& cnt) {
    t = blockIdx.x + (j / SUB) * gridDim.x;
    first = static_cast<uint64_t>(t) * kTile + static_cast<uint64_t>(j % SUB) * kTxRows;
    cnt = first < n ? static_cast<uint32_t>(n - first < static_cast<uint64_t>(kTxRows) ? n - first : static_cast<uint64_t>(kTxRows)) : 0u;
    return t < T;
  };
  auto issue = [&](uint32_t j) {
    uint32_t t, cnt;
    uint64_t first;
    if (tid == 0 && sub_of(j, t, first, cnt) && cnt) {
      unsigned char* dst = buf0 + (j & 1) * kTxRows * 32;
      const uint32_t boxes = (cnt + kTxBox - 1) / kTxBox;  // OOB rows zero-filled
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       smem_u32(&mbar[j & 1])),
                   "r"(boxes * kTxBox * 32)
                   : "memory");
      for (uint32_t b = 0; b < boxes; ++b)
        tensor_load_2d(dst + b * kTxBox * 32, &tm, 0, static_cast<int>(first + b * kTxBox),
                       &mbar[j & 1]);
    }
  };
  uint32_t par[2] = {0, 0};
  issue(0);
  for (uint32_t j = 0;; ++j) {
    uint32_t t, cnt;
    uint64_t first;
    if (!sub_of(j, t, first, cnt)) break;
    issue(j + 1);
    const bool fresh = j % SUB == 0;
    uint32_t g0[DPT];
    if (fresh) {
#pragma unroll
      for (int k = 0; k < DPT; ++k) {
        const int dd = tid * DPT + k;
        g0[k] = dd < D ? __ldg(goff + static_cast<uint64_t>(t) * D + dd) : 0u;
      }
    }
    if (cnt == 0) {
      if (fresh)
#pragma unroll
        for (int k = 0; k < DPT; ++k) bx[tid * DPT + k] = g0[k];
      __syncthreads();
      continue;
    }
    const unsigned char* sb = buf0 + (j & 1) * kTxRows * 32;
    {
      uint4* w4 = reinterpret_cast<uint4*>(wc);
      constexpr int n4 = kW * Dp * 2 / 16;
      for (int i = tid; i < n4; i += kTxThreads) w4[i] = make_uint4(0, 0, 0, 0);
    }
    mbar_wait(&mbar[j & 1], par[j & 1]);
    par[j & 1] ^= 1;
    __syncthreads();
    uint32_t d[kTxItems];
    uint16_t rk[kTxItems];
#pragma unroll
    for (int k = 0; k < kTxItems; ++k) {
      const uint32_t li = warp * (32 * kTxItems) + k * 32 + lane;
      d[k] = li < cnt ? static_cast<uint32_t>(
                            *reinterpret_cast<const int32_t*>(sb + li * 32 + 16) - min_rank)
                      : 0xFFFFFFFFu;
    }
    uint16_t* mine = wc + warp * Dp;
#pragma unroll
    for (int k = 0; k < kTxItems; ++k) {
      const bool valid = d[k] != 0xFFFFFFFFu;
      const unsigned peers = __match_any_sync(0xffffffffu, d[k]);
      const uint32_t before = valid ? mine[d[k]] : 0u;
      rk[k] = static_cast<uint16_t>(before + __popc(peers & ((1u << lane) - 1u)));
      __syncwarp();
      if (valid && lane == __ffs(peers) - 1)
        mine[d[k]] = static_cast<uint16_t>(before + __popc(peers));
      __syncwarp();
    }
    __syncthreads();
    using VecT = typename std::conditional<DPT == 4, uint2, uint32_t>::type;
    union DV {
      VecT v;
      uint16_t h[DPT];
    };
    uint32_t tot[DPT];
#pragma unroll
    for (int k = 0; k < DPT; ++k) tot[k] = 0;
#pragma unroll
    for (int w = 0; w < kW; ++w) {
      DV x;
      x.v = *reinterpret_cast<const VecT*>(wc + w * Dp + tid * DPT);
#pragma unroll
      for (int k = 0; k < DPT; ++k) tot[k] += x.h[k];
    }
    uint32_t mysum = 0;
#pragma unroll
    for (int k = 0; k < DPT; ++k) mysum += tot[k];
    uint32_t ts0[DPT];
    ts0[0] = block_excl_scan_u32(mysum, wsum, nullptr);
#pragma unroll
    for (int k = 1; k < DPT; ++k) ts0[k] = ts0[k - 1] + tot[k - 1];
    {
      uint32_t run[DPT];
#pragma unroll
      for (int k = 0; k < DPT; ++k) run[k] = ts0[k];
#pragma unroll
      for (int w = 0; w < kW; ++w) {
        DV x, y;
        x.v = *reinterpret_cast<const VecT*>(wc + w * Dp + tid * DPT);
#pragma unroll
        for (int k = 0; k < DPT; ++k) {
          y.h[k] = static_cast<uint16_t>(run[k]);
          run[k] += x.h[k];
        }
        *reinterpret_cast<VecT*>(wc + w * Dp + tid * DPT) = y.v;
      }
    }
    uint32_t nxt[DPT];
#pragma unroll
    for (int k = 0; k < DPT; ++k) {
      const int dd = tid * DPT + k;
      const uint32_t rb = fresh ? g0[k] : bx[dd];
      nxt[k] = rb + tot[k];
      bx[dd] = rb - ts0[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kTxItems; ++k)
      if (d[k] != 0xFFFFFFFFu)
        sidx[mine[d[k]] + rk[k]] =
            static_cast<uint16_t>(warp * (32 * kTxItems) + k * 32 + lane);
    __syncthreads();
    // digit order: 4 records per thread in flight
    {
      uint32_t li[kTxItems], q[kTxItems];
      ulonglong2 h0[kTxItems], hm[kTxItems];
#pragma unroll
      for (int k = 0; k < kTxItems; ++k) {
        const uint32_t p = tid + k * kTxThreads;
        li[k] = p < cnt ? sidx[p] : 0u;
      }
#pragma unroll
      for (int k = 0; k < kTxItems; ++k) {
        const ulonglong2* rec = reinterpret_cast<const ulonglong2*>(sb + li[k] * 32);
        h0[k] = rec[0];
        hm[k] = rec[1];
      }
#pragma unroll
      for (int k = 0; k < kTxItems; ++k) {
        const uint32_t p = tid + k * kTxThreads;
        const int32_t rank = static_cast<int32_t>(hm[k].x & 0xffffffffu);
        q[k] = bx[static_cast<uint32_t>(rank - min_rank) & (Dp - 1)] + p;
      }
#pragma unroll
      for (int k = 0; k < kTxItems; ++k) {
        const uint32_t p = tid + k * kTxThreads;
        if (p >= cnt) break;
        const uint32_t qq = q[k];
        o.tso[qq] = h0[k];
        o.meta[qq] = meta_of(hm[k], static_cast<uint32_t>(first + li[k]));
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < DPT; ++k) bx[tid * DPT + k] = nxt[k];
    __syncthreads();
  }
}

// Driver entry point for the tensor-map encoder (no libcuda link needed).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// Tensor map over the packed records as a [n][12] u32 array (48-B rows),
// boxes of 256 rows x the first 8 words.
bool record_head_map(const csg_packed_record* recs, uint64_t n, CUtensorMap* tm) {
  EncodeTiledFn f = encode_tiled();
  if (!f || n == 0 || n >= (1ull << 31)) return false;
  const cuuint64_t dims[2] = {12, static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[1] = {48};
  const cuuint32_t box[2] = {8, static_cast<cuuint32_t>(kTxBox)};
  const cuuint32_t es[2] = {1, 1};
  return f(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<csg_packed_record*>(recs), dims,
           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// Per-rank chunked prefix maximum of ts (StoreView::cmax): one block per rank
// segment, the segment split into one contiguous run of 128-record chunks
// per warp. Each warp reduces its chunks (4 coalesced loads per lane, one
// warp reduction per chunk), warps exchange their part maxima through shared
// memory, and each warp turns its chunk maxima into running maxima with one
// warp scan per 32 chunks. Every reference "prefix scan that stops at the
// first ts > t" (rca.cpp:146-237) becomes a binary search over the chunk
// maxima plus one chunk scan (seg_first), without materialising a running
// maximum per record. The same pass flags segments whose op_seq descends in
// store order (the flow index permutes only those, see k_flow_fix).
__global__ void __launch_bounds__(1024)
    k_chunkmax_blk(const ulonglong2* __restrict__ tso,
                   const uint32_t* __restrict__ off, double* __restrict__ cm,
                   uint32_t* __restrict__ unsorted, uint32_t* __restrict__ list,
                   unsigned* __restrict__ cnt, unsigned long long* __restrict__ max_seg,
                   int32_t r0, const int* go) {
  pdl_wait();
  pdl_trigger();
  if (go && !*go) return;
  __shared__ double pmax[32];
  __shared__ int desc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int32_t r = r0 + blockIdx.x;  // the store's own rank range only
  const uint32_t b = off[r], e = off[r + 1];
  const uint32_t L = e - b;
  if (threadIdx.x == 0) {
    desc = 0;
    if (L) atomicMax(max_seg, static_cast<unsigned long long>(L));
  }
  const uint32_t nc = (L + kCmChunk - 1) / kCmChunk;
  const uint32_t cper = (nc + nw - 1) / nw;  // chunks per warp
  const uint32_t c0 = min(nc, warp * cper), c1 = min(nc, c0 + cper);
  double* cmr = cm + (b / kCmChunk + r);
  double m = -INFINITY;
  bool dsc = false;
  constexpr int G = kCmChunk / 32;  // 32-record groups per chunk
  // op_seq of the record before the current group (descent check)
  long long prev = LLONG_MIN;
  if (c0 < c1 && c0 > 0) prev = static_cast<long long>(__ldg(&tso[b + c0 * kCmChunk - 1].y));
  for (uint32_t c = c0; c < c1; c += 2) {
    // two chunks' loads in flight before any use
    ulonglong2 v[2 * G];
#pragma unroll
    for (int k = 0; k < 2 * G; ++k) {
      const uint32_t p = b + c * kCmChunk + k * 32 + lane;
      v[k] = (c + k / G < c1 && p < e) ? __ldg(tso + p)
                                         : make_ulonglong2(0xFFF0000000000000ull, 0);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (c + h >= c1) break;
      double x = -INFINITY;
#pragma unroll
      for (int k = h * G; k < h * G + G; ++k) {
        const uint32_t p = b + c * kCmChunk + k * 32 + lane;
        double t;
        memcpy(&t, &v[k].x, 8);
        if (p < e && t == t) x = fmax(x, t);  // NaN never breaks a prefix
        const long long op = static_cast<long long>(v[k].y);
        long long pv = __shfl_up_sync(0xffffffffu, op, 1);
        if (lane == 0) pv = prev;
        if (p < e && p > b) dsc |= op < pv;
        prev = __shfl_sync(0xffffffffu, op, 31);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
      if (lane == 0) cmr[c + h] = x;
      m = fmax(m, x);
    }
  }
  if (lane == 0) pmax[warp] = m;
  __syncthreads();
  if (dsc) desc = 1;
  double carry = -INFINITY;
  for (int w = 0; w < warp; ++w) carry = fmax(carry, pmax[w]);
  __syncwarp();
  for (uint32_t cb = c0; cb < c1; cb += 32) {
    const uint32_t c = cb + lane;
    double x = c < c1 ? cmr[c] : -INFINITY;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x = fmax(x, y);
    }
    x = fmax(x, carry);
    carry = __shfl_sync(0xffffffffu, x, 31);
    if (c < c1) cmr[c] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsorted[r] = desc ? 1u : 0u;
    if (desc) list[atomicAdd(cnt, 1u)] = r;
  }
}

// rank_off[r] = first sorted position with key >= r, r in [0, R].
__global__ void k_rank_off(const uint32_t* __restrict__ keys, uint64_t n,
                           int32_t R, uint32_t* __restrict__ off) {
  const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > R) return;
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (keys[mid] < static_cast<uint32_t>(r)) lo = mid + 1; else hi = mid;
  }
  off[r] = static_cast<uint32_t>(lo);
}

// Gather packed AoS records into rank-major columns (general index path).
__global__ void k_gather(const csg_packed_record* __restrict__ r,
                         const uint32_t* __restrict__ perm, uint64_t n, ScatterOut o) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
       p += (uint64_t)gridDim.x * blockDim.x) {
    // 48-byte records are 16-byte aligned: three 16-byte vector loads.
    const ulonglong2* rec =
        reinterpret_cast<const ulonglong2*>(r + perm[p]);
    const ulonglong2 h0 = __ldg(rec), hm = __ldg(rec + 1);
    o.tso[p] = h0;
    o.meta[p] = meta_of(hm, perm[p]);
  }
}

// Fill the op index's entry columns from the rank-major store.
__global__ void k_opidx_fill(StoreView s, const uint32_t* __restrict__ pos,
                             uint64_t n, int32_t* __restrict__ rank,
                             double* __restrict__ ts, double* __restrict__ dur,
                             uint8_t* __restrict__ nm) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t p = pos[i];
    rank[i] = rank_at(s, p);
    const double t = s.ts[p];
    double st;
    const uint64_t pa = s.pa[p];
    memcpy(&st, &pa, 8);
    ts[i] = t;
    dur[i] = t - st;
    nm[i] = static_cast<uint8_t>(ko_opname(s.ko[p]));
  }
}

// Flow index, step 2: persistent blocks over the flagged segments (at most
// P <= kFlowSmemMax records each), ops staged in shared memory. A segment
// made of k <= kFlowRuns ascending runs is merged directly: an element's
// output position is its offset in its run plus, for every other run, the
// number of elements ordered before it there (binary search; earlier runs
// win ties, so the order is stable). Otherwise a bitonic sort of the unique
// keys (op - segment min) << 14 | local index. Longer segments (or op spans
// >= 2^49) count into *overflow and the host falls back to the device-wide
// radix sort.
constexpr int kFlowSmemMax = 16384;
constexpr int kFlowRuns = 8;
__global__ void __launch_bounds__(1024)
    k_flow_fix(StoreView s, const uint32_t* __restrict__ list,
               const unsigned* __restrict__ cnt, int32_t P,
               uint32_t* __restrict__ pos, unsigned* __restrict__ overflow) {
  extern __shared__ long long so[];
  __shared__ uint32_t rs[kFlowRuns + 1];
  __shared__ int nrun;
  __shared__ long long wmin[32], wmax[32];
  const unsigned total = *cnt;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (unsigned w = blockIdx.x; w < total; w += gridDim.x) {
    const uint32_t r = list[w];
    const uint32_t b = s.rank_off[r], e = s.rank_off[r + 1];
    const uint32_t L = e - b;
    if (L > static_cast<uint32_t>(P)) {
      if (threadIdx.x == 0) atomicAdd(overflow, 1u);
      continue;  // uniform over the block
    }
    if (threadIdx.x == 0) nrun = 0;
    for (uint32_t i = threadIdx.x; i < L; i += blockDim.x) so[i] = s.op[b + i];
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < L; i += blockDim.x)
      if (i == 0 || so[i] < so[i - 1]) {
        const int q = atomicAdd(&nrun, 1);
        if (q < kFlowRuns) rs[q] = i;
      }
    __syncthreads();
    const int k = nrun;
    if (k <= kFlowRuns) {
      if (threadIdx.x == 0) {  // order the <= 8 run starts, close the last run
        for (int x = 1; x < k; ++x)
          for (int y = x; y > 0 && rs[y] < rs[y - 1]; --y) {
            const uint32_t t = rs[y];
            rs[y] = rs[y - 1];
            rs[y - 1] = t;
          }
        rs[k] = L;
      }
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < L; i += blockDim.x) {
        const long long x = so[i];
        int ra = 0;
        while (i >= rs[ra + 1]) ++ra;
        uint32_t out = i - rs[ra];
        for (int j = 0; j < k; ++j) {
          if (j == ra) continue;
          uint32_t lo = rs[j], hi = rs[j + 1];
          if (j < ra) {  // elements <= x come first (earlier in store order)
            while (lo < hi) {
              const uint32_t m = (lo + hi) >> 1;
              if (so[m] <= x) lo = m + 1; else hi = m;
            }
          } else {
            while (lo < hi) {
              const uint32_t m = (lo + hi) >> 1;
              if (so[m] < x) lo = m + 1; else hi = m;
            }
          }
          out += lo - rs[j];
        }
        pos[b + out] = b + i;
      }
      __syncthreads();
      continue;
    }
    // general case: bitonic sort of unique keys
    long long mn = LLONG_MAX, mx = LLONG_MIN;
    for (uint32_t i = threadIdx.x; i < L; i += blockDim.x) {
      mn = min(mn, so[i]);
      mx = max(mx, so[i]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
      wmin[warp] = mn;
      wmax[warp] = mx;
    }
    __syncthreads();
    mn = LLONG_MAX;
    mx = LLONG_MIN;
    for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) {
      mn = min(mn, wmin[q]);
      mx = max(mx, wmax[q]);
    }
    if (static_cast<unsigned long long>(mx - mn) >= (1ull << 49)) {
      if (threadIdx.x == 0) atomicAdd(overflow, 1u);
      __syncthreads();
      continue;
    }
    unsigned long long* fk = reinterpret_cast<unsigned long long*>(so);
    for (int32_t i = threadIdx.x; i < P; i += blockDim.x)
      fk[i] = i < static_cast<int32_t>(L)
                  ? (static_cast<unsigned long long>(so[i] - mn) << 14) |
                        static_cast<unsigned long long>(i)
                  : ~0ull;
    __syncthreads();
    for (int32_t kk = 2; kk <= P; kk <<= 1) {
      for (int32_t j = kk >> 1; j > 0; j >>= 1) {
        for (int32_t i = threadIdx.x; i < P; i += blockDim.x) {
          const int32_t x = i ^ j;
          if (x > i) {
            const unsigned long long av = fk[i], cv = fk[x];
            const bool up = (i & kk) == 0;
            if ((av > cv) == up) {
              fk[i] = cv;
              fk[x] = av;
            }
          }
        }
        __syncthreads();
      }
    }
    for (uint32_t i = threadIdx.x; i < L; i += blockDim.x)
      pos[b + i] = b + static_cast<uint32_t>(fk[i] & 0x3fffu);
    __syncthreads();
  }
}

// Global fallback: (rank, op - min_op) keys over the whole store.
template <typename K>
__global__ void k_flow_keys(StoreView s, int64_t min_op, int rank_shift,
                            K* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < s.n;
       p += (uint64_t)gridDim.x * blockDim.x) {
    keys[p] = static_cast<K>(
        (static_cast<unsigned long long>(rank_at(s, static_cast<uint32_t>(p))) << rank_shift) |
        static_cast<unsigned long long>(s.op[p] - min_op));
    vals[p] = static_cast<uint32_t>(p);
  }
}

// Gathered-entry permutation into sorted order.
__global__ void k_opidx_permute(const uint32_t* __restrict__ idx, uint64_t n,
                                const int32_t* __restrict__ r0,
                                const double* __restrict__ t0,
                                const double* __restrict__ d0,
                                const uint8_t* __restrict__ m0,
                                int32_t* __restrict__ r1, double* __restrict__ t1,
                                double* __restrict__ d1, uint8_t* __restrict__ m1) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = idx[i];
    r1[i] = r0[k];
    t1[i] = t0[k];
    d1[i] = d0[k];
    m1[i] = m0[k];
  }
}

__global__ void k_fill_u32(uint32_t* __restrict__ v, uint64_t n, uint32_t x) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    v[i] = x;
}

__global__ void k_iota(uint32_t* __restrict__ v, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    v[i] = static_cast<uint32_t>(i);
}

// ---- query ---------------------------------------------------------------

// Pass 1: per listed rank, count records with t0 <= ts <= t1.
__global__ void k_query_count(StoreView s, const int32_t* __restrict__ ranks,
                              int32_t nr, double t0, double t1,
                              uint32_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= nr) return;
  const int32_t r = ranks[w];
  uint32_t c = 0;
  if (r >= 0 && r < s.R) {
    for (uint32_t p = s.rank_off[r] + lane; p < s.rank_off[r + 1]; p += 32) {
      const double t = s.ts[p];
      c += !(t < t0 || t > t1);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) counts[w] = c;
}

// Pass 2: order-preserving compaction (rank order, then store order).
__global__ void k_query_write(StoreView s, const int32_t* __restrict__ ranks,
                              int32_t nr, double t0, double t1,
                              const uint32_t* __restrict__ offs,
                              uint64_t* __restrict__ okey,
                              uint32_t* __restrict__ oval) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= nr) return;
  const int32_t r = ranks[w];
  if (r < 0 || r >= s.R) return;
  uint32_t o = offs[w];
  const uint32_t b = s.rank_off[r], e = s.rank_off[r + 1];
  for (uint32_t base = b; base < e; base += 32) {
    const uint32_t p = base + lane;
    bool hit = false;
    double t = 0;
    if (p < e) {
      t = s.ts[p];
      hit = !(t < t0 || t > t1);
    }
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (hit) {
      const uint32_t at = o + __popc(m & ((1u << lane) - 1u));
      okey[at] = dkey(t == 0.0 ? 0.0 : t);  // -0 sorts with +0 (== in ref)
      oval[at] = s.perm[p];
    }
    o += __popc(m);
  }
}

// ---- last_log_per_rank -----------------------------------------------------

__global__ void k_last_log(StoreView s, const int32_t* __restrict__ members,
                           int32_t nm, double t, uint64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= nm) return;
  const int32_t r = members[w];
  // best = (ts, store idx) maximal among ts <= t; store idx breaks ties
  // toward the later append (proj/src/trace.cpp:135).
  bool found = false;
  double bt = 0;
  uint32_t bi = 0;
  if (r >= 0 && r < s.R) {
    for (uint32_t p = s.rank_off[r] + lane; p < s.rank_off[r + 1]; p += 32) {
      const double x = s.ts[p];
      if (x > t) continue;
      const uint32_t i = s.perm[p];
      if (!found || x > bt || (x == bt && i > bi)) {
        found = true;
        bt = x;
        bi = i;
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const int f2 = __shfl_xor_sync(0xffffffffu, (int)found, o);
    const double t2 = __shfl_xor_sync(0xffffffffu, bt, o);
    const uint32_t i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    if (f2 && (!found || t2 > bt || (t2 == bt && i2 > bi))) {
      found = true;
      bt = t2;
      bi = i2;
    }
  }
  if (lane == 0) out[w] = found ? bi : ~0ull;
}

// ---- op-ordered completion index -----------------------------------------

__global__ void k_opidx_flags(StoreView s, uint32_t* __restrict__ flags) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < s.n;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint8_t ko = s.ko[p];
    flags[p] = (ko_kind(ko) == CSG_KIND_COMPLETION &&
                ko_opname(ko) != CSG_OP_RECV)
                   ? 1u
                   : 0u;
  }
}

__global__ void k_opidx_scatter(StoreView s, const uint32_t* __restrict__ offs,
                                int64_t min_op, uint64_t* __restrict__ keys,
                                uint32_t* __restrict__ vals) {
  // entry value = rank-major position; the rank is recovered afterwards
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < s.n;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const uint8_t ko = s.ko[p];
    if (ko_kind(ko) == CSG_KIND_COMPLETION && ko_opname(ko) != CSG_OP_RECV) {
      const uint32_t at = offs[p];
      keys[at] = static_cast<uint64_t>(s.op[p] - min_op);
      vals[at] = static_cast<uint32_t>(p);
    }
  }
}

// Dense op-segment offsets of the op index: off[k] = first entry with key
// >= k, k in [0, range + 1] (keys = op - min_op, sorted ascending).
__global__ void k_opidx_off(const uint64_t* __restrict__ keys, uint64_t n, uint64_t range,
                            uint32_t* __restrict__ off) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k <= range + 1;
       k += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (keys[mid] < k) lo = mid + 1; else hi = mid;
    }
    off[k] = static_cast<uint32_t>(lo);
  }
}

unsigned grid_for(uint64_t n, int threads = 256) {
  uint64_t g = (n + threads - 1) / threads;
  if (g > 148ull * 64) g = 148ull * 64;
  if (g == 0) g = 1;
  return static_cast<unsigned>(g);
}

}  // namespace

// Does the store's fetched-to-be statistics match the speculated layout
// (own rank span, rank space) and pass validation? Host and device evaluate
// the same predicate on the same StoreStats.
__host__ __device__ inline bool spec_match(const StoreStats& h, int32_t lmin, int32_t lmax,
                                           int32_t R) {
  return h.n_total > 0 && h.min_rank >= 0 && h.min_chan >= 0 && h.max_chan < 4096 &&
         h.n_nan == 0 && h.lmin_rank == lmin && h.lmax_rank == lmax && h.max_rank + 1 == R;
}
__global__ void k_spec_check(const StoreStats* st, int32_t lmin, int32_t lmax, int32_t R,
                             int* go) {
  if (threadIdx.x == 0) *go = spec_match(*st, lmin, lmax, R) ? 1 : 0;
}

void store_build_index(csg_store* s) {
  if (s->indexed) return;
  csg_ctx* c = s->ctx;
  cudaStream_t st = c->stream;
  const uint64_t n = s->n;
  const csg_packed_record* recs = s->recs.as<csg_packed_record>();
  StoreStats h{};
  h.ts_max_key = 0;
  h.min_rank = INT32_MAX;
  h.max_rank = INT32_MIN;
  h.min_chan = INT32_MAX;
  h.max_chan = INT32_MIN;
  h.min_op = INT64_MAX;
  h.max_op = INT64_MIN;
  h.n_total = n;
  h.lmin_rank = INT32_MAX;
  h.lmax_rank = INT32_MIN;
  h.max_seg = 0;
  s->stats_dev.ensure(sizeof(StoreStats));
  CSG_CUDA(cudaMemcpyAsync(s->stats_dev.p, &h, sizeof(h),
                           cudaMemcpyHostToDevice, st));
  s->perm.ensure(n * 4 + 4);
  s->keys.ensure(n * 4 + 4);
  const uint32_t ntiles = static_cast<uint32_t>((n + kTile - 1) / kTile);
  DevBuf& hcnt = c->buf("index.hist");
  hcnt.ensure(static_cast<size_t>(kHistDigits) * ntiles * 4 + 16);
  // CSG_SCATTER_CFG: 0 = block-ranked persistent scatter (k_scatter),
  // 2 = its single-buffered variants, 3 = 2-D tensor-copy scatter
  static const int cfg = std::getenv("CSG_SCATTER_CFG") ? std::atoi(std::getenv("CSG_SCATTER_CFG")) : 0;
  // A store whose last build took the general (wide rank span) path is
  // rebuilt the same way: its first pass writes the statistics together
  // with the (rank, store index) sort pairs, instead of a digit histogram
  // the general path never reads (one pass over the records less). If the
  // statistics then call for the fused path, its histogram pass runs after.
  static const bool spec_on0 = std::getenv("CSG_INDEX_NOSPEC") == nullptr;
  const bool keys_first = spec_on0 && s->spec_general && n > 0 && n <= 0xFFFFFFF0ull;
  auto stats_keys = [&](StoreStats* sdst) {
    ProfScope ps_(c->lc, "k_stats_keys", st);
    const unsigned g = static_cast<unsigned>(std::min<uint64_t>((n + 1023) / 1024, 148ull * 8));
    k_stats_keys<<<g, 256, 0, st>>>(recs, n, sdst, s->keys.as<uint32_t>(),
                                    s->perm.as<uint32_t>());
  };
  HostBuf& hs = c->hbuf("store.stats");
  hs.ensure(sizeof(h));
  FetchArgs fa{};
  fa.add(s->stats_dev.p, hs.p, sizeof(h));
  auto stats_hist = [&](StoreStats* sdst, unsigned long long* flag = nullptr,
                        unsigned long long v = 0, unsigned* fdone = nullptr) {
    ProfScope ps_(c->lc, "k_stats_hist", st);
    k_stats_hist<<<ntiles, kTileThreads, 0, st>>>(recs, n, sdst, hcnt.as<uint32_t>(), fa, flag,
                                                  v, fdone);
  };
  DevBuf& st2 = c->buf("index.stats2");  // statistics of a second pass (discarded)
  st2.ensure(sizeof(StoreStats));
  static const bool stats_fetch = std::getenv("CSG_STATS_FETCH") != nullptr;
  FetchTicket tk;
  if (keys_first) {
    stats_keys(s->stats_dev.as<StoreStats>());
  } else if (n && !comm_active(c) && !stats_fetch) {
    c->sig.ensure(64);
    DevBuf& fdn = c->buf("fetch.done");
    if (fdn.bytes < 16) {
      fdn.ensure(16);
      CSG_CUDA(cudaMemsetAsync(fdn.p, 0, 16, st));
    }
    tk.seq = ++c->sig_seq;
    stats_hist(s->stats_dev.as<StoreStats>(), c->sig.as<unsigned long long>(), tk.seq,
               fdn.as<unsigned>());
    CSG_CUDA(cudaGetLastError());
    if (!c->ev_fetch) CSG_CUDA(cudaEventCreateWithFlags(&c->ev_fetch, cudaEventDisableTiming));
    CSG_CUDA(cudaEventRecord(c->ev_fetch, st));
  } else if (n) {
    stats_hist(s->stats_dev.as<StoreStats>());
  }
  if (comm_active(c)) {
    // global stats over the shards (identical rank space, ticks, op range)
    // one MAX all-reduce over order-preserving u64 images (minima as
    // complements) and one SUM all-reduce for the counts
    DevBuf& pk = c->buf("store.stats_pack");
    const int P = c->nranks;
    pk.ensure((9 + 2 * static_cast<size_t>(P)) * 8);
    {
      ProfScope ps_(c->lc, "k_stats_pack", st);
      k_stats_pack<<<1, 32, 0, st>>>(s->stats_dev.as<StoreStats>(),
                                     pk.as<unsigned long long>(), 0, P, c->rank);
    }
    comm_group_start(c);
    comm_allreduce(c, pk.p, 7 + 2 * static_cast<size_t>(P), ncclUint64, ncclMax);
    comm_allreduce(c, pk.as<unsigned long long>() + 7 + 2 * P, 2, ncclUint64, ncclSum);
    comm_group_end(c);
    {
      ProfScope ps_(c->lc, "k_stats_pack", st);
      k_stats_pack<<<1, 32, 0, st>>>(s->stats_dev.as<StoreStats>(),
                                     pk.as<unsigned long long>(), 1, P, c->rank);
    }
  }
  if (!tk.seq) tk = ctx_fetch_issue(c, fa);
  static const bool force_general = std::getenv("CSG_INDEX_RADIX") != nullptr;
  // Index layout for own rank span [lmin_, lmax_] and rank space R. With
  // go != nullptr the launches are speculative: every kernel first reads
  // *go (k_spec_check) and exits unless the layout holds.
  auto layout = [&](int32_t lmin_, int32_t lmax_, int32_t R, const int* go) {
  s->rank_off.ensure((static_cast<size_t>(R) + 1) * 4);
  s->tso.ensure(n * 16 + 16);
  s->runmax.ensure((n / kCmChunk + static_cast<size_t>(R) + 2) * 8);
  s->meta.ensure(n * 16 + 16);
  const bool fused = n && !force_general &&
                     static_cast<int64_t>(lmax_) - lmin_ < kHistDigits;
  if (fused) {
    if (keys_first) {  // speculated the general path: the histogram is missing
      CSG_CUDA(cudaMemcpyAsync(st2.p, &h, sizeof(h), cudaMemcpyHostToDevice, st));
      stats_hist(st2.as<StoreStats>());
    }
    // one stable counting-sort pass over the rank digits (see k_scatter)
    const int32_t lmin = lmin_;
    const int32_t D = lmax_ - lmin + 1;
    const uint32_t d0 = static_cast<uint32_t>(lmin) & (kHistDigits - 1);
    DevBuf& goff = c->buf("index.goff");
    DevBuf& csum = c->buf("index.csum");
    goff.ensure(static_cast<size_t>(D) * ntiles * 4 + 4);
    const uint32_t tpc = std::max<uint32_t>(1, (ntiles + kHistChunks - 1) / kHistChunks);
    const uint32_t nchunks = (ntiles + tpc - 1) / tpc;
    csum.ensure((static_cast<size_t>(D) * nchunks + kHistDigits) * 4);
    uint32_t* cs = csum.as<uint32_t>();
    uint32_t* tot = cs + static_cast<size_t>(D) * nchunks;
    {
      ProfScope ps_(c->lc, "k_hist_colsum", st);
      launch_pdl(k_hist_colsum, dim3(nchunks), dim3(1024), 0, st, hcnt.as<uint32_t>(), ntiles, tpc, d0, D, cs, go);
    }
    {
      ProfScope ps_(c->lc, "k_hist_chunkscan", st);
      launch_pdl(k_hist_chunkscan, dim3((D + 31) / 32), dim3(256), 0, st, cs, nchunks, D, tot, go);
    }
    {
      ProfScope ps_(c->lc, "k_hist_apply", st);
      launch_pdl(k_hist_apply, dim3(nchunks), dim3(1024), 0, st, hcnt.as<uint32_t>(), cs, tot, ntiles, tpc, d0, D,
                                             goff.as<uint32_t>(), go);
    }
    ScatterOut o{s->tso.as<ulonglong2>(), s->meta.as<uint4>()};
    // Persistent, one CTA per SM, sub-tiles double-buffered by bulk copies:
    // 2048 records for rank spans <= 1024, 1024 records (wider digit tables)
    // up to 2048. CSG_SCATTER_CFG=2: single-buffered variants.
    const bool narrow = D <= 1024;
    const int TR = narrow ? 2048 : 1024;
    const int nbuf = cfg == 2 ? 1 : 2;
    const int Dp = (narrow ? 4 : 8) * kTileThreads;
    const size_t smem = static_cast<size_t>(nbuf) * TR * 48 +
                        (kTileThreads / 32) * static_cast<size_t>(Dp) * 2 +
                        static_cast<size_t>(Dp) * 4;
    smem_optin(k_scatter<8, 2, 4>, 2 * 2048 * 48 + 8 * 1024 * 2 + 1024 * 4);
    smem_optin(k_scatter<4, 2, 8>, 2 * 1024 * 48 + 8 * 2048 * 2 + 2048 * 4);
    smem_optin(k_scatter<8, 1, 4>, 2048 * 48 + 8 * 1024 * 2 + 1024 * 4);
    smem_optin(k_scatter<4, 1, 8>, 1024 * 48 + 8 * 2048 * 2 + 2048 * 4);
    CUtensorMap tm;
    const bool tx = cfg == 3 && record_head_map(recs, n, &tm);
    if (tx) {
      smem_optin(k_scatter_tx<2>, 2 * kTxRows * 32 + 16 * 1024 * 2 + 1024 * 4);
      smem_optin(k_scatter_tx<4>, 2 * kTxRows * 32 + 16 * 2048 * 2 + 2048 * 4);
    }
    {
      ProfScope ps_(c->lc, "k_scatter", st);
      const unsigned grid = std::min<unsigned>(ntiles, kScatterCtas);
      uint32_t* ro = s->rank_off.as<uint32_t>();
      const uint32_t* g = goff.as<uint32_t>();
      if (tx) {
        const int dpt = narrow ? 2 : 4;
        const size_t sm = 2 * kTxRows * 32 + 16 * static_cast<size_t>(dpt) * kTxThreads * 2 +
                          static_cast<size_t>(dpt) * kTxThreads * 4;
        if (narrow)
          k_scatter_tx<2><<<grid, kTxThreads, sm, st>>>(tm, n, g, ntiles, lmin, D, o,
                                                        lmax_, R, ro, go);
        else
          k_scatter_tx<4><<<grid, kTxThreads, sm, st>>>(tm, n, g, ntiles, lmin, D, o,
                                                        lmax_, R, ro, go);
      } else if (nbuf == 2 && narrow) {
        static const bool dbg = std::getenv("CSG_DEBUG_SCATTER") != nullptr;
        if (dbg) {
          const int on = 1;
          unsigned long long z[6] = {0, 0, 0, 0, 0, 0};
          CSG_CUDA(cudaMemcpyToSymbolAsync(g_scatter_prof_on, &on, sizeof(on), 0,
                                           cudaMemcpyHostToDevice, st));
          CSG_CUDA(cudaMemcpyToSymbolAsync(g_scatter_cyc, z, sizeof(z), 0,
                                           cudaMemcpyHostToDevice, st));
        }
        launch_pdl(k_scatter<8, 2, 4>, dim3(grid), dim3(kTileThreads), smem, st, recs, n, g, ntiles, lmin, D, o,
                                                             lmax_, R, ro, go);
        if (dbg) {
          unsigned long long z[6];
          CSG_CUDA(cudaMemcpyFromSymbolAsync(z, g_scatter_cyc, sizeof(z), 0,
                                             cudaMemcpyDeviceToHost, st));
          CSG_CUDA(cudaStreamSynchronize(st));
          const double sub = z[5] ? static_cast<double>(z[5]) : 1.0;
          fprintf(stderr, "k_scatter cycles per sub-tile (thread 0): wait %.0f rank %.0f scan "
                  "%.0f stage %.0f write %.0f over %llu sub-tiles\n", z[0] / sub, z[1] / sub,
                  z[2] / sub, z[3] / sub, z[4] / sub, z[5]);
        }
      }
      else if (nbuf == 2)
        k_scatter<4, 2, 8><<<grid, kTileThreads, smem, st>>>(recs, n, g, ntiles, lmin, D, o,
                                                             lmax_, R, ro, go);
      else if (narrow)
        k_scatter<8, 1, 4><<<grid, kTileThreads, smem, st>>>(recs, n, g, ntiles, lmin, D, o,
                                                             lmax_, R, ro, go);
      else
        k_scatter<4, 1, 8><<<grid, kTileThreads, smem, st>>>(recs, n, g, ntiles, lmin, D, o,
                                                             lmax_, R, ro, go);
    }
  } else {
    // general path: (rank, store index) pairs, LSD radix sort, gather
    if (n && !keys_first) {
      CSG_CUDA(cudaMemcpyAsync(st2.p, &h, sizeof(h), cudaMemcpyHostToDevice, st));
      stats_keys(st2.as<StoreStats>());
    }
    if (n) {
      radix_sort_u32(s->keys.as<uint32_t>(), s->perm.as<uint32_t>(), n,
                     bits_for(static_cast<uint64_t>(R > 0 ? R - 1 : 0)), s->sort,
                     st, c->lc);
      {
        ProfScope ps_(c->lc, "k_gather", st);
        ScatterOut o{s->tso.as<ulonglong2>(), s->meta.as<uint4>()};
        k_gather<<<grid_for(n), 256, 0, st>>>(recs, s->perm.as<uint32_t>(), n, o);
      }
    }
    {
      ProfScope ps_(c->lc, "k_rank_off", st);
      k_rank_off<<<(R + 1 + 255) / 256, 256, 0, st>>>(s->keys.as<uint32_t>(), n, R,
                                                     s->rank_off.as<uint32_t>());
    }
  }
  // flow-index descent flags + work list, filled by k_runmax_blk
  s->fl_unsorted.ensure((static_cast<size_t>(R) + 2) * 4);
  DevBuf& flist = s->fl_list;
  DevBuf& fcnt = s->fl_cnt;
  flist.ensure(static_cast<size_t>(R) * 4 + 4);
  fcnt.ensure(8);
  CSG_CUDA(cudaMemsetAsync(fcnt.p, 0, 8, st));
  if (R) CSG_CUDA(cudaMemsetAsync(s->fl_unsorted.p, 0, static_cast<size_t>(R) * 4, st));
  if (n && R) {
    // ranks outside [lmin, lmax] (a shard's foreign ranks) have no records:
    // their chunk maxima are never read and their flags stay 0
    const int32_t r0 = std::max(lmin_, 0), r1 = std::min(lmax_, R - 1);
    // 128 threads: many blocks per SM overlap one block's scan tail with the
    // others' loads and the ~1000 rank segments fit one wave (43 vs 45 / 51
    // us at 256 / 512 threads on the C2 store, gpurun_out cm1)
    static const int cm_threads =
        std::getenv("CSG_CM_THREADS") ? std::atoi(std::getenv("CSG_CM_THREADS")) : 128;
    ProfScope ps_(c->lc, "k_chunkmax", st);
    if (r1 >= r0)
      launch_pdl(k_chunkmax_blk, dim3(r1 - r0 + 1), dim3(cm_threads), 0, st, 
          s->tso.as<ulonglong2>(), s->rank_off.as<uint32_t>(), s->runmax.as<double>(),
          s->fl_unsorted.as<uint32_t>(), flist.as<uint32_t>(), fcnt.as<unsigned>(),
          &s->stats_dev.as<StoreStats>()->max_seg, r0, go);
  }
  };
  // Speculation: a store rebuilt over the same rank layout (a replay, a
  // re-ingest of the same job) launches its scatter on the last layout while
  // the statistics travel to the host, hiding that round trip.
  static const bool spec_on = std::getenv("CSG_INDEX_NOSPEC") == nullptr;
  const bool spec = spec_on && !force_general && s->spec_ok && n > 0 && n <= 0xFFFFFFF0ull;
  DevBuf& specf = c->buf("index.spec_go");
  if (spec) {
    specf.ensure(16);
    {
      ProfScope ps_(c->lc, "k_spec_check", st);
      k_spec_check<<<1, 32, 0, st>>>(s->stats_dev.as<StoreStats>(), s->sp_lmin, s->sp_lmax,
                                     s->sp_R, specf.as<int>());
    }
    layout(s->sp_lmin, s->sp_lmax, s->sp_R, specf.as<int>());
  }
  ctx_fetch_wait(c, tk);
  std::memcpy(&h, hs.p, sizeof(h));
  s->spec_ok = false;
  const uint64_t ng = h.n_total;
  s->n_global = ng;
  if (h.overlap)
    throw Error(CSG_ERR_RUNTIME,
                "engine: sharded store: shards' rank ranges overlap (records of "
                "one rank must live on one shard; shard by rank range)");
  if (ng && h.min_rank < 0)
    throw Error(CSG_ERR_RUNTIME,
                "engine: negative rank in trace record (ranks must be >= 0)");
  if (ng && h.min_chan < 0)
    throw Error(CSG_ERR_RUNTIME,
                "engine: negative channel in trace record (channels must be >= 0)");
  if (ng && h.max_chan >= 4096)
    throw Error(CSG_ERR_RUNTIME, "engine: channel id >= 4096 unsupported");
  if (h.n_nan)
    throw Error(CSG_ERR_RUNTIME, "engine: NaN timestamp in trace record");
  if (n > 0xFFFFFFF0ull)
    throw Error(CSG_ERR_RUNTIME, "engine: store exceeds 2^32 records");
  const double mx = ng ? dkey_inv(h.ts_max_key) : 0.0;
  s->last_ts = (ng && mx > 0.0) ? mx : 0.0;
  s->own_lo = n ? h.lmin_rank : 0;
  s->own_hi = n ? h.lmax_rank : -1;
  s->min_rank = ng ? h.min_rank : 0;
  s->max_rank = ng ? h.max_rank : -1;
  s->min_chan = ng ? h.min_chan : 0;
  s->max_chan = ng ? h.max_chan : -1;
  s->min_op = ng ? h.min_op : 0;
  s->max_op = ng ? h.max_op : -1;
  s->R = s->max_rank + 1;
  s->nch = s->max_chan + 1;
  const int32_t R = s->R;

  const bool hit = spec && spec_match(h, s->sp_lmin, s->sp_lmax, s->sp_R);
  if (!hit) layout(h.lmin_rank, h.lmax_rank, R, nullptr);
  s->spec_ok = n && !force_general &&
               static_cast<int64_t>(h.lmax_rank) - h.lmin_rank < kHistDigits &&
               spec_match(h, h.lmin_rank, h.lmax_rank, R);
  s->sp_lmin = h.lmin_rank;
  s->sp_lmax = h.lmax_rank;
  s->sp_R = R;
  s->spec_general = n && (force_general ||
                          static_cast<int64_t>(h.lmax_rank) - h.lmin_rank >= kHistDigits);
  // the longest segment stays on the device until the next host round trip
  // (trigger_run picks it up with the trips); shards agree on it over NCCL
  s->max_seg = 0;
  s->max_seg_pending = n && R;
  if (comm_active(c)) {
    // reduced with the next group of collectives (the trigger windows'), read
    // back at the next round trip, on every shard (also shards without records)
    s->max_seg_unreduced = true;
    s->max_seg_pending = true;
  }
  CSG_CUDA(cudaGetLastError());
  s->indexed = true;
  s->op_indexed = false;
  s->flow_indexed = false;
  s->flow_early = false;
}

void store_build_op_index(csg_store* s, int32_t opn) {
  (void)opn;
  if (s->op_indexed) return;
  csg_ctx* c = s->ctx;
  cudaStream_t st = c->stream;
  const uint64_t n = s->n;
  StoreView v = s->view();
  DevBuf& flags = c->buf("opidx.flags");
  flags.ensure(n * 4 + 4);
  uint32_t count = 0;
  if (n) {
    {
      ProfScope ps_(c->lc, "k_opidx_flags", st);
      k_opidx_flags<<<grid_for(n), 256, 0, st>>>(v, flags.as<uint32_t>());
    }
    uint32_t last_flag = 0;
    CSG_CUDA(cudaMemcpyAsync(&last_flag, flags.as<uint32_t>() + n - 1, 4,
                             cudaMemcpyDeviceToHost, st));
    exclusive_scan_u32(flags.as<uint32_t>(), n, c->scratch_a, st, c->lc);
    uint32_t last_off = 0;
    CSG_CUDA(cudaMemcpyAsync(&last_off, flags.as<uint32_t>() + n - 1, 4,
                             cudaMemcpyDeviceToHost, st));
    CSG_CUDA(cudaStreamSynchronize(st));
    count = last_off + last_flag;
  }
  DevBuf& pos = c->buf("opidx.pos");
  s->opidx_keys.ensure(static_cast<size_t>(count) * 8 + 8);
  pos.ensure(static_cast<size_t>(count) * 4 + 4);
  if (count) {
    ProfScope ps_(c->lc, "k_opidx_scatter", st);
    k_opidx_scatter<<<grid_for(n), 256, 0, st>>>(
        v, flags.as<uint32_t>(), s->min_op, s->opidx_keys.as<uint64_t>(),
        pos.as<uint32_t>());
  }
  const uint64_t range = static_cast<uint64_t>(s->max_op - s->min_op);
  if (count)
    radix_sort_u64(s->opidx_keys.as<uint64_t>(), pos.as<uint32_t>(), count,
                   bits_for(range), s->sort, st, c->lc);
  s->opidx_rank.ensure(static_cast<size_t>(count) * 4 + 4);
  s->opidx_ts.ensure(static_cast<size_t>(count) * 8 + 8);
  s->opidx_dur.ensure(static_cast<size_t>(count) * 8 + 8);
  s->opidx_nm.ensure(static_cast<size_t>(count) + 8);
  if (count) {
    ProfScope ps_(c->lc, "k_opidx_fill", st);
    k_opidx_fill<<<grid_for(count), 256, 0, st>>>(
        v, pos.as<uint32_t>(), count, s->opidx_rank.as<int32_t>(),
        s->opidx_ts.as<double>(), s->opidx_dur.as<double>(), s->opidx_nm.as<uint8_t>());
  }
  s->n_opidx = count;
  if (comm_active(c)) {
    // Sharded: every shard needs every rank's completions for the sibling /
    // cohort medians. All-gather the (padded) entry columns, then re-sort.
    DevBuf& dcnt = c->buf("opidx.cnt");
    dcnt.ensure(static_cast<size_t>(c->nranks) * 8);
    unsigned long long mine = count;
    CSG_CUDA(cudaMemcpyAsync(dcnt.as<unsigned long long>() + c->rank, &mine, 8,
                             cudaMemcpyHostToDevice, st));
    comm_allgather(c, dcnt.as<unsigned long long>() + c->rank, dcnt.p, 1, ncclUint64);
    std::vector<unsigned long long> cnts(c->nranks);
    CSG_CUDA(cudaMemcpyAsync(cnts.data(), dcnt.p, c->nranks * 8, cudaMemcpyDeviceToHost, st));
    CSG_CUDA(cudaStreamSynchronize(st));
    unsigned long long cmax = 0, total = 0;
    for (auto x : cnts) {
      cmax = std::max(cmax, x);
      total += x;
    }
    const size_t P = c->nranks;
    DevBuf &gk = c->buf("opidx.gk"), &gr = c->buf("opidx.gr"), &gt = c->buf("opidx.gt"),
           &gd = c->buf("opidx.gd"), &gm = c->buf("opidx.gm"), &gi = c->buf("opidx.gi");
    DevBuf &lk = c->buf("opidx.lk"), &lr = c->buf("opidx.lr"), &lt = c->buf("opidx.lt"),
           &ld = c->buf("opidx.ld"), &lm = c->buf("opidx.lm");
    lk.ensure(cmax * 8 + 8);
    lr.ensure(cmax * 4 + 4);
    lt.ensure(cmax * 8 + 8);
    ld.ensure(cmax * 8 + 8);
    lm.ensure(cmax + 8);
    // padding keys sort after every real key
    CSG_CUDA(cudaMemsetAsync(lk.p, 0xff, cmax * 8 + 8, st));
    if (count) {
      CSG_CUDA(cudaMemcpyAsync(lk.p, s->opidx_keys.p, count * 8ull, cudaMemcpyDeviceToDevice, st));
      CSG_CUDA(cudaMemcpyAsync(lr.p, s->opidx_rank.p, count * 4ull, cudaMemcpyDeviceToDevice, st));
      CSG_CUDA(cudaMemcpyAsync(lt.p, s->opidx_ts.p, count * 8ull, cudaMemcpyDeviceToDevice, st));
      CSG_CUDA(cudaMemcpyAsync(ld.p, s->opidx_dur.p, count * 8ull, cudaMemcpyDeviceToDevice, st));
      CSG_CUDA(cudaMemcpyAsync(lm.p, s->opidx_nm.p, count, cudaMemcpyDeviceToDevice, st));
    }
    gk.ensure(P * cmax * 8 + 8);
    gr.ensure(P * cmax * 4 + 4);
    gt.ensure(P * cmax * 8 + 8);
    gd.ensure(P * cmax * 8 + 8);
    gm.ensure(P * cmax + 8);
    gi.ensure(P * cmax * 4 + 4);
    comm_group_start(c);
    comm_allgather(c, lk.p, gk.p, cmax, ncclUint64);
    comm_allgather(c, lr.p, gr.p, cmax, ncclInt32);
    comm_allgather(c, lt.p, gt.p, cmax, ncclFloat64);
    comm_allgather(c, ld.p, gd.p, cmax, ncclFloat64);
    comm_allgather(c, lm.p, gm.p, cmax, ncclUint8);
    comm_group_end(c);
    const uint64_t ng = P * cmax;
    {
      ProfScope ps_(c->lc, "k_iota", st);
      k_iota<<<grid_for(ng), 256, 0, st>>>(gi.as<uint32_t>(), ng);
    }
    // keys are op - min_op over the global op range; the padding keys'
    // low bits (all ones) still sort after every real key at that width.
    // Stable: equal ops keep shard order, i.e. the global rank-major order.
    const uint64_t grange =
        s->max_op >= s->min_op ? static_cast<uint64_t>(s->max_op - s->min_op) : 0;
    radix_sort_u64(gk.as<uint64_t>(), gi.as<uint32_t>(), ng, bits_for(grange + 1), s->sort, st,
                   c->lc);
    s->opidx_keys.ensure(ng * 8 + 8);
    s->opidx_rank.ensure(ng * 4 + 4);
    s->opidx_ts.ensure(ng * 8 + 8);
    s->opidx_dur.ensure(ng * 8 + 8);
    s->opidx_nm.ensure(ng + 8);
    CSG_CUDA(cudaMemcpyAsync(s->opidx_keys.p, gk.p, ng * 8, cudaMemcpyDeviceToDevice, st));
    {
      ProfScope ps_(c->lc, "k_opidx_permute", st);
      k_opidx_permute<<<grid_for(ng), 256, 0, st>>>(
          gi.as<uint32_t>(), ng, gr.as<int32_t>(), gt.as<double>(), gd.as<double>(),
          gm.as<uint8_t>(), s->opidx_rank.as<int32_t>(), s->opidx_ts.as<double>(),
          s->opidx_dur.as<double>(), s->opidx_nm.as<uint8_t>());
    }
    s->n_opidx = total;  // padding sorted to the end
  }
  {  // dense per-op segment offsets (the straggler self-evidence lookups)
    const uint64_t range = s->max_op >= s->min_op ? static_cast<uint64_t>(s->max_op - s->min_op) : 0;
    s->op_seg_off.ensure((range + 2) * 4 + 16);
    ProfScope ps_(c->lc, "k_opidx_off", st);
    k_opidx_off<<<grid_for(range + 2), 256, 0, st>>>(s->opidx_keys.as<uint64_t>(), s->n_opidx,
                                                     range, s->op_seg_off.as<uint32_t>());
  }
  CSG_CUDA(cudaGetLastError());
  s->op_indexed = true;
}

void store_reduce_max_seg(csg_store* s) {
  if (!s->max_seg_unreduced) return;
  s->max_seg_unreduced = false;
  comm_allreduce(s->ctx, &s->stats_dev.as<StoreStats>()->max_seg, 1, ncclUint64, ncclMax);
}

void store_resolve_max_seg(csg_store* s) {
  store_reduce_max_seg(s);
  if (!s->max_seg_pending) return;
  unsigned long long v = 0;
  CSG_CUDA(cudaMemcpyAsync(&v, &s->stats_dev.as<StoreStats>()->max_seg, 8,
                           cudaMemcpyDeviceToHost, s->ctx->stream));
  CSG_CUDA(cudaStreamSynchronize(s->ctx->stream));
  s->max_seg = v;
  s->max_seg_pending = false;
}

// The flow index's segment fix-up launched ahead of the trip round trip of a
// detection replay: k_flow_fix at the shared-memory cap (the longest segment
// is only known once that round trip returns), so it runs while the host
// reads the trips. store_build_flow_index then only does the overflow check.
void store_flow_index_early(csg_store* s) {
  static const bool off = std::getenv("CSG_FLOW_GLOBAL_SORT") != nullptr ||
                          std::getenv("CSG_DISABLE_FLOW_INDEX") != nullptr ||
                          std::getenv("CSG_FLOW_SMEM_CAP") != nullptr ||
                          std::getenv("CSG_NO_EARLY_FLOW") != nullptr;
  if (off || !s->indexed || s->flow_indexed || s->flow_early || !s->n || !s->R) return;
  csg_ctx* c = s->ctx;
  cudaStream_t st = c->stream;
  s->fl_pos.ensure(s->n * 4 + 4);
  unsigned* d_uns = s->fl_cnt.as<unsigned>();
  smem_optin(k_flow_fix, kFlowSmemMax * 8);
  {
    ProfScope ps_(c->lc, "k_flow_fix", st);
    k_flow_fix<<<static_cast<unsigned>(std::min<int32_t>(s->R, 148)), 1024,
                 static_cast<size_t>(kFlowSmemMax) * 8, st>>>(
        s->view(), s->fl_list.as<uint32_t>(), d_uns, kFlowSmemMax, s->fl_pos.as<uint32_t>(),
        d_uns + 1);
  }
  CSG_CUDA(cudaGetLastError());
  s->flow_early = true;
}

bool store_build_flow_index(csg_store* s) {
  store_build_index(s);
  if (s->flow_indexed) return true;
  tl_mark("flow index entry");
  store_resolve_max_seg(s);
  csg_ctx* c = s->ctx;
  cudaStream_t st = c->stream;
  const uint64_t n = s->n;
  const int32_t R = s->R;
  s->fl_pos.ensure(n * 4 + 4);
  if (!n || !R) {
    s->flow_indexed = true;
    return true;
  }
  // descent flags, work list and its count come from k_runmax_blk
  DevBuf& cnt = s->fl_cnt;
  DevBuf& list = s->fl_list;
  unsigned* d_uns = cnt.as<unsigned>();
  unsigned* d_ovf = d_uns + 1;
  static const bool force_global = std::getenv("CSG_FLOW_GLOBAL_SORT") != nullptr;
  const uint64_t span = static_cast<uint64_t>(s->max_op - s->min_op);
  bool global = force_global;
  if (!global) {
    // CSG_FLOW_SMEM_CAP (power of two) lowers the shared-memory segment cap
    // so tests can drive the overflow -> device-wide fallback on small traces
    static const int32_t cap = [] {
      const char* e = std::getenv("CSG_FLOW_SMEM_CAP");
      int32_t v = e ? std::atoi(e) : kFlowSmemMax;
      return (v >= 64 && v <= kFlowSmemMax) ? v : kFlowSmemMax;
    }();
    int32_t P = 64;
    while (static_cast<uint64_t>(P) < s->max_seg && P < cap) P <<= 1;
    if (s->flow_early) {
      P = kFlowSmemMax;  // already launched at the cap (store_flow_index_early)
    } else {
      const size_t smem = static_cast<size_t>(P) * 8;
      smem_optin(k_flow_fix, kFlowSmemMax * 8);
      ProfScope ps_(c->lc, "k_flow_fix", st);
      k_flow_fix<<<static_cast<unsigned>(std::min<int32_t>(R, 148)), 1024, smem, st>>>(
          s->view(), list.as<uint32_t>(), d_uns, P, s->fl_pos.as<uint32_t>(), d_ovf);
    }
    // Without a segment longer than the shared-memory sort or a huge op
    // span nothing can overflow: no host round trip on the common path.
    if (s->max_seg > static_cast<uint64_t>(P) || span >= (1ull << 49)) {
      unsigned h[2];
      CSG_CUDA(cudaMemcpyAsync(h, cnt.p, 8, cudaMemcpyDeviceToHost, st));
      CSG_CUDA(cudaStreamSynchronize(st));
      global = h[1] != 0;
    }
  }
  if (global) {
    // Device-wide stable radix sort by (rank, op): every segment permuted.
    const int ob = bits_for(span);
    const int rb = bits_for(static_cast<uint64_t>(std::max(R, 1) - 1));
    if (ob + rb > 64) return false;
    {
      ProfScope ps_(c->lc, "k_fill_u32", st);
      k_fill_u32<<<grid_for(R), 256, 0, st>>>(s->fl_unsorted.as<uint32_t>(), R, 1u);
    }
    if (ob + rb <= 32) {
      s->fl_keys.ensure(n * 4 + 4);
      {
        ProfScope ps_(c->lc, "k_flow_keys", st);
        k_flow_keys<uint32_t><<<grid_for(n), 256, 0, st>>>(
            s->view(), s->min_op, ob, s->fl_keys.as<uint32_t>(), s->fl_pos.as<uint32_t>());
      }
      radix_sort_u32(s->fl_keys.as<uint32_t>(), s->fl_pos.as<uint32_t>(), n, ob + rb,
                     s->sort, st, c->lc);
    } else {
      s->fl_keys.ensure(n * 8 + 8);
      {
        ProfScope ps_(c->lc, "k_flow_keys", st);
        k_flow_keys<unsigned long long><<<grid_for(n), 256, 0, st>>>(
            s->view(), s->min_op, ob, s->fl_keys.as<unsigned long long>(),
            s->fl_pos.as<uint32_t>());
      }
      radix_sort_u64(s->fl_keys.as<uint64_t>(), s->fl_pos.as<uint32_t>(), n, ob + rb,
                     s->sort, st, c->lc);
    }
  }
  CSG_CUDA(cudaGetLastError());
  s->flow_indexed = true;
  return true;
}

// ---- query / last_log host entry points --------------------------------------

void store_query(csg_store* s, const int32_t* ranks, size_t nr, double t0,
                 double t1, std::vector<uint64_t>& out) {
  if (t0 > t1) throw Error(CSG_ERR_RUNTIME, "query: t0 > t1");
  store_build_index(s);
  out.clear();
  // Set semantics (std::find over the rank span): unique ranks, ascending,
  // so the compaction yields (rank, store index) order before the ts sort.
  std::vector<int32_t> rs(ranks, ranks + nr);
  std::sort(rs.begin(), rs.end());
  rs.erase(std::unique(rs.begin(), rs.end()), rs.end());
  rs.erase(std::remove_if(rs.begin(), rs.end(),
                          [&](int32_t r) { return r < 0 || r >= s->R; }),
           rs.end());
  if (rs.empty() || s->n == 0) return;
  csg_ctx* c = s->ctx;
  cudaStream_t st = c->stream;
  const int32_t k = static_cast<int32_t>(rs.size());
  DevBuf d_ranks, d_counts;
  d_ranks.ensure(k * 4);
  d_counts.ensure((k + 1) * 4);
  CSG_CUDA(cudaMemcpyAsync(d_ranks.p, rs.data(), k * 4, cudaMemcpyHostToDevice, st));
  StoreView v = s->view();
  const unsigned g = static_cast<unsigned>((static_cast<uint64_t>(k) * 32 + 255) / 256);
  {
    ProfScope ps_(c->lc, "k_query_count", st);
    k_query_count<<<g, 256, 0, st>>>(v, d_ranks.as<int32_t>(), k, t0, t1,
                                     d_counts.as<uint32_t>());
  }
  CSG_CUDA(cudaMemsetAsync(d_counts.as<uint32_t>() + k, 0, 4, st));
  exclusive_scan_u32(d_counts.as<uint32_t>(), k + 1, c->scratch_a, st, c->lc);
  uint32_t total = 0;
  CSG_CUDA(cudaMemcpyAsync(&total, d_counts.as<uint32_t>() + k, 4,
                           cudaMemcpyDeviceToHost, st));
  CSG_CUDA(cudaStreamSynchronize(st));
  if (!total) return;
  DevBuf keys, vals;
  keys.ensure(total * 8);
  vals.ensure(total * 4);
  {
    ProfScope ps_(c->lc, "k_query_write", st);
    k_query_write<<<g, 256, 0, st>>>(v, d_ranks.as<int32_t>(), k, t0, t1,
                                     d_counts.as<uint32_t>(), keys.as<uint64_t>(),
                                     vals.as<uint32_t>());
  }
  SortScratch ss;
  radix_sort_u64(keys.as<uint64_t>(), vals.as<uint32_t>(), total, 64, ss, st,
                 c->lc);
  std::vector<uint32_t> h(total);
  CSG_CUDA(cudaMemcpyAsync(h.data(), vals.p, total * 4, cudaMemcpyDeviceToHost, st));
  CSG_CUDA(cudaStreamSynchronize(st));
  out.assign(h.begin(), h.end());
}

void store_last_log(csg_store* s, const int32_t* members, size_t nm, double t,
                    std::vector<std::pair<int32_t, uint64_t>>& out) {
  if (nm == 0) throw Error(CSG_ERR_RUNTIME, "last_log_per_rank: empty group");
  store_build_index(s);
  out.clear();
  csg_ctx* c = s->ctx;
  cudaStream_t st = c->stream;
  DevBuf d_m, d_o;
  d_m.ensure(nm * 4);
  d_o.ensure(nm * 8);
  CSG_CUDA(cudaMemcpyAsync(d_m.p, members, nm * 4, cudaMemcpyHostToDevice, st));
  const unsigned g = static_cast<unsigned>((nm * 32 + 255) / 256);
  {
    ProfScope ps_(c->lc, "k_last_log", st);
    k_last_log<<<g, 256, 0, st>>>(s->view(), d_m.as<int32_t>(),
                                  static_cast<int32_t>(nm), t, d_o.as<uint64_t>());
  }
  std::vector<uint64_t> h(nm);
  CSG_CUDA(cudaMemcpyAsync(h.data(), d_o.p, nm * 8, cudaMemcpyDeviceToHost, st));
  CSG_CUDA(cudaStreamSynchronize(st));
  for (size_t i = 0; i < nm; ++i)
    if (h[i] != ~0ull) out.emplace_back(members[i], h[i]);
}

}  // namespace csg
