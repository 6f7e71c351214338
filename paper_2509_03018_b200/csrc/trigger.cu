// trigger.cu — Algorithm 1 (the trigger) on the device.
//
// Reference: evaluate (proj/src/trigger.cpp:57-136) runs one full-store
// TraceStore::query per sampled rank per tick (trace.cpp:101-119) and folds
// the window into an EMA baseline. Here every (tick, sampled rank) window is
// reduced in parallel from the rank-major columns (one warp each; the window
// is a FILTER over the rank's records, so order does not matter for the
// statistics used: count, has-state, completion count, byte sum, min/max
// end), and the EMA recurrence runs as one thread per sampled rank over all
// ticks. Baselines of distinct ranks never interact; ticks couple them only
// through "lowest tripped rank wins", resolved per tick afterwards.
//
// Floating point: the EMA and threshold products use explicit _rn intrinsics
// (and the file is built with -fmad=false) so no FMA contraction happens,
// matching the reference's SSE2 build.
#include <algorithm>
#include <cstring>

#include "comm.cuh"
#include "objects.h"
#include "trigger.cuh"

namespace csg {
namespace {

// Window statistics (TraceStore::query per sampled rank and tick,
// trace.cpp:101-119, reduced as evaluate does, trigger.cpp:62-104) with one
// pass over each sampled rank's records per tile of ticks: block (si, tile)
// bins every record into the (few) windows of its tile that contain it,
// accumulating in shared memory. Window k holds x iff !(x < t_k - delta) &&
// !(x > t_k) (trace.cpp:107 with t0 = t_k - delta). Tiles of TT ticks keep
// the bins in shared memory for any tick count: a segment is read once per
// tile, not once per tick.
__global__ void k_window_bins(StoreView s, const double* __restrict__ ticks_all,
                              int32_t T_all, int32_t TT,
                              const int32_t* __restrict__ sampled,
                              int32_t S, double delta,
                              WinStat* __restrict__ out_all) {
  const int32_t k0 = blockIdx.y * TT;
  const int32_t T = min(TT, T_all - k0);
  const double* ticks = ticks_all + k0;
  WinStat* out = out_all + static_cast<int64_t>(k0) * S;
  extern __shared__ __align__(16) unsigned char wb_dyn[];
  double* st = reinterpret_cast<double*>(wb_dyn);                       // [T]
  unsigned long long* bytes = reinterpret_cast<unsigned long long*>(st + T);
  unsigned long long* mn = bytes + T;
  unsigned long long* mx = mn + T;
  uint32_t* nrec = reinterpret_cast<uint32_t*>(mx + T);
  uint32_t* ncomp = nrec + T;
  uint32_t* hstate = ncomp + T;
  const int32_t si = blockIdx.x;
  for (int32_t k = threadIdx.x; k < T; k += blockDim.x) {
    st[k] = ticks[k];
    bytes[k] = 0;
    mn[k] = ~0ull;
    mx[k] = 0;
    nrec[k] = ncomp[k] = hstate[k] = 0;
  }
  __syncthreads();
  const int32_t r = sampled[si];
  if (r >= 0 && r < s.R) {
    const uint32_t e = s.rank_off[r + 1];
    for (uint32_t p = s.rank_off[r] + threadIdx.x; p < e; p += blockDim.x) {
      const double x = s.ts[p];
      int32_t lo = 0, hi = T;  // first tick with t_k >= x
      while (lo < hi) {
        const int32_t md = (lo + hi) >> 1;
        if (st[md] < x) lo = md + 1; else hi = md;
      }
      const bool comp = ko_kind(s.ko[p]) == CSG_KIND_COMPLETION;
      for (int32_t k = lo; k < T && !(x < st[k] - delta); ++k) {
        if (x > st[k]) continue;
        atomicAdd(&nrec[k], 1u);
        if (comp) {
          atomicAdd(&ncomp[k], 1u);
          atomicAdd(&bytes[k], static_cast<unsigned long long>(s.pb[p]));
          const unsigned long long kk = dkey(x);
          atomicMin(&mn[k], kk);
          atomicMax(&mx[k], kk);
        } else {
          hstate[k] = 1;
        }
      }
    }
  }
  __syncthreads();
  for (int32_t k = threadIdx.x; k < T; k += blockDim.x) {
    // an empty window is all zeros: shards that do not own the sampled rank
    // contribute nothing to the sum all-reduce
    WinStat w;
    w.n_rec = nrec[k];
    w.n_comp = ncomp[k];
    w.has_state = hstate[k];
    w.pad = 0;
    w.bytes = bytes[k];
    w.min_end = ncomp[k] ? dkey_inv(mn[k]) : 0.0;
    w.max_end = ncomp[k] ? dkey_inv(mx[k]) : 0.0;
    out[static_cast<int64_t>(k) * S + si] = w;
  }
}

// One baseline step (trigger.cpp:76-133). Returns 0 none, 1 failure,
// 2 straggler.
__device__ int ema_step(TrigSlot& b, const WinStat& w, const TrigParams& p) {
  const bool had_prev = b.had_prev != 0;
  b.had_prev = w.n_rec > 0 ? 1 : 0;
  if (w.n_comp == 0) {
    const bool failure = w.has_state || (w.n_rec == 0 && had_prev);
    return failure ? 1 : 0;
  }
  // Σ (double)msg_bytes: integer-valued, exact below 2^53 in any order.
  const double window_bytes = static_cast<double>(w.bytes);
  const double throughput = __ddiv_rn(window_bytes, p.delta);
  double mean_interval = 0;
  bool interval_defined = false;
  if (w.n_comp >= 2) {
    mean_interval = __ddiv_rn(__dsub_rn(w.max_end, w.min_end),
                              static_cast<double>(w.n_comp - 1));
    interval_defined = true;
  }
  const bool warmed = b.updates >= p.warmup;
  bool straggler = false;
  if (warmed && b.throughput > 0 &&
      throughput <= __dmul_rn(p.drop, b.throughput))
    straggler = true;
  if (warmed && !straggler && interval_defined && b.interval_defined &&
      b.op_interval_ms > 0 &&
      mean_interval >= __dmul_rn(p.inflate, b.op_interval_ms))
    straggler = true;
  if (straggler) return 2;
  const double keep = __dsub_rn(1.0, p.alpha);
  b.throughput = b.updates == 0
                     ? throughput
                     : __dadd_rn(__dmul_rn(keep, b.throughput),
                                 __dmul_rn(p.alpha, throughput));
  if (interval_defined) {
    b.op_interval_ms = !b.interval_defined
                           ? mean_interval
                           : __dadd_rn(__dmul_rn(keep, b.op_interval_ms),
                                       __dmul_rn(p.alpha, mean_interval));
    b.interval_defined = 1;
  }
  b.updates += 1;
  return 0;
}

// run_detection: thread per sampled rank, sequential over ticks.
__global__ void k_ema_ticks(const WinStat* __restrict__ ws, int32_t T, int32_t S,
                            TrigParams p, uint8_t* __restrict__ trip) {
  const int32_t si = blockIdx.x * blockDim.x + threadIdx.x;
  if (si >= S) return;
  TrigSlot b{0, 0, 0, 0, 0, 0};
  for (int32_t k = 0; k < T; ++k)
    trip[static_cast<int64_t>(k) * S + si] =
        static_cast<uint8_t>(ema_step(b, ws[static_cast<int64_t>(k) * S + si], p));
}

// Lowest tripped sampled rank wins (sampled is ascending); compact the
// tripped ticks in tick order. One block.
__global__ void k_pick_trips(const uint8_t* __restrict__ trip,
                             const double* __restrict__ ticks, int32_t T,
                             const int32_t* __restrict__ sampled, int32_t S,
                             csg_trigger_event* __restrict__ events,
                             int32_t* __restrict__ n_events) {
  __shared__ int32_t base;
  __shared__ int32_t wsum[32];
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int32_t k0 = 0; k0 < T; k0 += blockDim.x) {
    const int32_t k = k0 + threadIdx.x;
    int kind = -1, rank = -1;
    if (k < T) {
      for (int32_t s = 0; s < S; ++s) {
        const uint8_t c = trip[static_cast<int64_t>(k) * S + s];
        if (c) {
          kind = c == 1 ? CSG_TRIGGER_FAILURE : CSG_TRIGGER_STRAGGLER;
          rank = sampled[s];
          break;
        }
      }
    }
    const int hit = kind >= 0;
    // block exclusive scan of hit
    int x = hit;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int v = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      wsum[lane] = v;
    }
    __syncthreads();
    const int excl = (warp ? wsum[warp - 1] : 0) + x - hit;
    if (hit) {
      csg_trigger_event e;
      e.kind = kind;
      e.suspect_rank = rank;
      e.time_ms = ticks[k];
      events[base + excl] = e;
    }
    __syncthreads();
    if (threadIdx.x == 0) base += wsum[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_events = base;
}

// Whole trigger stage of run_detection in one launch (unsharded stores):
//   1. window statistics: grid (B, S); block (b, s) bins chunk b of sampled
//      rank s's segment into per-tick shared-memory bins (as k_window_bins)
//      and merges them into zero-initialised global accumulators (ordered
//      timestamp keys: max via atomicMax, min via atomicMax of the
//      complemented key);
//   2. the last block of each sampled rank runs its EMA recurrence over all
//      ticks (evaluate, trigger.cpp:57-136) from the accumulators staged in
//      shared memory;
//   3. the last rank to finish picks the lowest tripped rank of every tick
//      and compacts the trips in tick order (runner.cpp:72-79).
// Accumulators of the trigger windows, zero-initialised; split by the
// reduction they need so a sharded store combines them with one SUM and one
// MAX all-reduce (complemented min key: max = min).
struct WinSum {
  unsigned int n_rec, n_comp, has_state, pad;
  unsigned long long bytes;
};
struct WinMax {
  unsigned long long mn_inv, mx;
};

// Mapped-memory publication of the trip list by the block that compacts it
// (the fused single-GPU trigger): [0] trip count, [8] longest store segment
// (when pending), [16..) the events, then the completion word — what the
// k_fetch of ctx_fetch_issue would copy, without its launch.
struct TrigPublish {
  unsigned char* h = nullptr;
  const unsigned long long* max_seg = nullptr;
  unsigned long long* flag = nullptr;
  unsigned long long seq = 0;
};

// EMA of sampled rank si over all ticks (evaluate, trigger.cpp:57-136) from
// the accumulated windows staged in shared memory, then — in the last block
// to finish (done[S] ticket) — the lowest tripped rank of every tick,
// compacted in tick order (runner.cpp:72-79). Block-collective.
__device__ void trigger_ema_pick(int32_t si, int32_t T, const double* st, int32_t S,
                                 const int32_t* __restrict__ sampled, const TrigParams& p,
                                 const WinSum* __restrict__ asum,
                                 const WinMax* __restrict__ amax, unsigned* __restrict__ done,
                                 uint8_t* __restrict__ trip,
                                 csg_trigger_event* __restrict__ events,
                                 int32_t* __restrict__ n_events, WinStat* ws,
                                 TrigPublish pub = TrigPublish{}) {
  __shared__ int last;
  __threadfence();
  for (int32_t k = threadIdx.x; k < T; k += blockDim.x) {
    const WinSum* a = asum + static_cast<int64_t>(k) * S + si;
    const WinMax* m = amax + static_cast<int64_t>(k) * S + si;
    WinStat w;
    w.n_rec = __ldcg(&a->n_rec);
    w.n_comp = __ldcg(&a->n_comp);
    w.has_state = __ldcg(&a->has_state);
    w.pad = 0;
    w.bytes = __ldcg(&a->bytes);
    w.min_end = w.n_comp ? dkey_inv(~__ldcg(&m->mn_inv)) : 0.0;
    w.max_end = w.n_comp ? dkey_inv(__ldcg(&m->mx)) : 0.0;
    ws[k] = w;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    TrigSlot b{0, 0, 0, 0, 0, 0};
    for (int32_t k = 0; k < T; ++k)
      trip[static_cast<int64_t>(k) * S + si] = static_cast<uint8_t>(ema_step(b, ws[k], p));
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&done[S], 1u) == static_cast<unsigned>(S - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ int32_t base;
  __shared__ int32_t wsum[32];
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int32_t k0 = 0; k0 < T; k0 += blockDim.x) {
    const int32_t k = k0 + threadIdx.x;
    int kind = -1, rank = -1;
    if (k < T) {
      for (int32_t q = 0; q < S; ++q) {
        const uint8_t c = __ldcg(trip + static_cast<int64_t>(k) * S + q);
        if (c) {
          kind = c == 1 ? CSG_TRIGGER_FAILURE : CSG_TRIGGER_STRAGGLER;
          rank = sampled[q];
          break;
        }
      }
    }
    const int hit = kind >= 0;
    int x = hit;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int v = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      wsum[lane] = v;
    }
    __syncthreads();
    const int excl = (warp ? wsum[warp - 1] : 0) + x - hit;
    if (hit) {
      csg_trigger_event e;
      e.kind = kind;
      e.suspect_rank = rank;
      e.time_ms = st[k];
      events[base + excl] = e;
    }
    __syncthreads();
    if (threadIdx.x == 0) base += wsum[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_events = base;
  if (pub.h) {
    __threadfence();
    __syncthreads();
    const int32_t ne = base;
    const uint32_t* e4 = reinterpret_cast<const uint32_t*>(events);
    uint32_t* d4 = reinterpret_cast<uint32_t*>(pub.h + 16);
    const uint32_t words = static_cast<uint32_t>(ne) * (sizeof(csg_trigger_event) / 4);
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) d4[i] = __ldcg(e4 + i);
    if (threadIdx.x == 0) {
      *reinterpret_cast<int32_t*>(pub.h) = ne;
      if (pub.max_seg)
        *reinterpret_cast<unsigned long long*>(pub.h + 8) = __ldcg(pub.max_seg);
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      *reinterpret_cast<volatile unsigned long long*>(pub.flag) = pub.seq;
      __threadfence_system();
    }
  }
}

// Whole trigger stage of run_detection in one launch:
//   1. window statistics: grid (B, S); block (b, s) bins chunk b of sampled
//      rank s's segment into per-tick shared-memory bins (as k_window_bins)
//      and merges them into the zero-initialised accumulators;
//   2. (chain != 0) the last block of each sampled rank runs trigger_ema_pick
//      for it. Sharded stores stop after step 1 (chain == 0), all-reduce the
//      accumulators and finish with k_trigger_ema.
__global__ void __launch_bounds__(512)
    k_trigger(StoreView s, const double* __restrict__ ticks, int32_t T,
              const int32_t* __restrict__ sampled, int32_t S, TrigParams p, int32_t B,
              WinSum* __restrict__ asum, WinMax* __restrict__ amax, unsigned* __restrict__ done,
              uint8_t* __restrict__ trip, csg_trigger_event* __restrict__ events,
              int32_t* __restrict__ n_events, int chain, TrigPublish pub) {
  extern __shared__ __align__(16) unsigned char tg_dyn[];
  double* st = reinterpret_cast<double*>(tg_dyn);                       // [T]
  unsigned long long* bytes = reinterpret_cast<unsigned long long*>(st + T);
  unsigned long long* mn = bytes + T;  // complemented keys (max = min)
  unsigned long long* mx = mn + T;
  uint32_t* nrec = reinterpret_cast<uint32_t*>(mx + T);
  uint32_t* ncomp = nrec + T;
  uint32_t* hstate = ncomp + T;
  __shared__ int last;
  const int32_t si = blockIdx.y, bi = blockIdx.x;
  for (int32_t k = threadIdx.x; k < T; k += blockDim.x) {
    st[k] = ticks[k];
    bytes[k] = mn[k] = mx[k] = 0;
    nrec[k] = ncomp[k] = hstate[k] = 0;
  }
  __syncthreads();
  const double delta = p.delta;
  const int32_t r = sampled[si];
  if (r >= 0 && r < s.R) {
    const uint32_t b0 = s.rank_off[r], L = s.rank_off[r + 1] - b0;
    const uint32_t cb = b0 + static_cast<uint32_t>(static_cast<uint64_t>(L) * bi / B);
    const uint32_t ce = b0 + static_cast<uint32_t>(static_cast<uint64_t>(L) * (bi + 1) / B);
    for (uint32_t q = cb + threadIdx.x; q < ce; q += blockDim.x) {
      const double x = s.ts[q];
      int32_t lo = 0, hi = T;  // first tick with t_k >= x
      while (lo < hi) {
        const int32_t md = (lo + hi) >> 1;
        if (st[md] < x) lo = md + 1; else hi = md;
      }
      const bool comp = ko_kind(s.ko[q]) == CSG_KIND_COMPLETION;
      for (int32_t k = lo; k < T && !(x < st[k] - delta); ++k) {
        if (x > st[k]) continue;
        atomicAdd(&nrec[k], 1u);
        if (comp) {
          atomicAdd(&ncomp[k], 1u);
          atomicAdd(&bytes[k], static_cast<unsigned long long>(s.pb[q]));
          const unsigned long long kk = dkey(x);
          atomicMax(&mn[k], ~kk);
          atomicMax(&mx[k], kk);
        } else {
          hstate[k] = 1;
        }
      }
    }
  }
  __syncthreads();
  for (int32_t k = threadIdx.x; k < T; k += blockDim.x) {
    if (!nrec[k]) continue;
    WinSum& a = asum[static_cast<int64_t>(k) * S + si];
    WinMax& m = amax[static_cast<int64_t>(k) * S + si];
    atomicAdd(&a.n_rec, nrec[k]);
    if (hstate[k]) atomicOr(&a.has_state, 1u);
    if (ncomp[k]) {
      atomicAdd(&a.n_comp, ncomp[k]);
      atomicAdd(&a.bytes, bytes[k]);
      atomicMax(&m.mn_inv, mn[k]);
      atomicMax(&m.mx, mx[k]);
    }
  }
  if (!chain) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&done[si], 1u) == static_cast<unsigned>(B - 1);
  __syncthreads();
  if (!last) return;
  // the bins are merged: the 40 T bytes behind the tick times (launched with
  // T * (8 + sizeof(WinStat)) bytes) stage the T window statistics
  trigger_ema_pick(si, T, st, S, sampled, p, asum, amax, done, trip, events, n_events,
                   reinterpret_cast<WinStat*>(bytes), pub);
}

// Sharded finish: one block per sampled rank over the all-reduced windows.
__global__ void __launch_bounds__(512)
    k_trigger_ema(const double* __restrict__ ticks, int32_t T,
                  const int32_t* __restrict__ sampled, int32_t S, TrigParams p,
                  const WinSum* __restrict__ asum, const WinMax* __restrict__ amax,
                  unsigned* __restrict__ done, uint8_t* __restrict__ trip,
                  csg_trigger_event* __restrict__ events, int32_t* __restrict__ n_events,
                  TrigPublish pub) {
  extern __shared__ __align__(16) unsigned char te_dyn[];
  double* st = reinterpret_cast<double*>(te_dyn);       // [T]
  WinStat* ws = reinterpret_cast<WinStat*>(st + T);      // [T]
  for (int32_t k = threadIdx.x; k < T; k += blockDim.x) st[k] = ticks[k];
  __syncthreads();
  trigger_ema_pick(blockIdx.x, T, st, S, sampled, p, asum, amax, done, trip, events,
                   n_events, ws, pub);
}

// csg_evaluate: one tick, the caller's sampled list in order (duplicates
// allowed, exactly like the reference loop), baselines persisted in the
// state's per-rank slots.
__global__ void k_ema_single(const WinStat* __restrict__ ws,
                             const int32_t* __restrict__ sampled, int32_t S,
                             TrigParams p, double t, TrigSlot* __restrict__ slots,
                             csg_trigger_event* __restrict__ ev,
                             int32_t* __restrict__ tripped) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int32_t hit = 0;
  for (int32_t s = 0; s < S; ++s) {
    const int32_t r = sampled[s];
    const int c = ema_step(slots[r], ws[s], p);
    if (c && !hit) {
      hit = 1;
      ev->kind = c == 1 ? CSG_TRIGGER_FAILURE : CSG_TRIGGER_STRAGGLER;
      ev->suspect_rank = r;
      ev->time_ms = t;
    }
  }
  *tripped = hit;
}

}  // namespace

void trigger_window_stats(csg_store* s, const double* d_ticks, int32_t T,
                          const int32_t* d_sampled, int32_t S, double delta,
                          WinStat* d_out) {
  if (T <= 0 || S <= 0) return;
  csg_ctx* c = s->ctx;
  constexpr int32_t kTileTicks = 4096;  // 44 B of bins per tick: 176 KB
  const int32_t TT = std::min(T, kTileTicks);
  const size_t smem = static_cast<size_t>(TT) * 44;
  smem_optin(k_window_bins, smem);
  ProfScope ps_(c->lc, "k_window_bins", c->stream);
  k_window_bins<<<dim3(S, (T + TT - 1) / TT), 512, smem, c->stream>>>(
      s->view(), d_ticks, T, TT, d_sampled, S, delta, d_out);
  CSG_CUDA(cudaGetLastError());
}

// Tick times by FP accumulation exactly as runner.cpp:69-71:
// for (t = I; t <= last_ts; t += I) if (t >= delta) evaluate.
// Computed on the host (plain IEEE adds, no contraction: the same doubles as
// the reference's SSE2 loop) and uploaded without a device round trip.
int32_t trigger_ticks(csg_store* s, double I, double delta, DevBuf& ticks) {
  csg_ctx* c = s->ctx;
  const double est = s->last_ts / I;
  if (!(est < 5e7))
    throw Error(CSG_ERR_RUNTIME, "run_detection: too many detection ticks");
  std::vector<double>& h = c->h_ticks;
  h.clear();
  for (double t = I; t <= s->last_ts; t += I) {
    if (t < delta) continue;
    h.push_back(t);
  }
  ticks.ensure(h.size() * 8 + 8);
  if (!h.empty())
    CSG_CUDA(cudaMemcpyAsync(ticks.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice,
                             c->stream));
  return static_cast<int32_t>(h.size());
}

int32_t trigger_run(csg_store* s, const double* d_ticks, int32_t T,
                    const int32_t* d_sampled, int32_t S, const TrigParams& p,
                    DevBuf& events) {
  csg_ctx* c = s->ctx;
  events.ensure(static_cast<size_t>(T + 1) * sizeof(csg_trigger_event));
  if (T <= 0 || S <= 0) return 0;
  DevBuf& ws = c->buf("trig.ws");
  DevBuf& trip = c->buf("trig.trip");
  DevBuf& dn = c->buf("trig.n");
  ws.ensure(static_cast<size_t>(T) * S * sizeof(WinStat));
  trip.ensure(static_cast<size_t>(T) * S);
  dn.ensure(4);
  static const bool no_publish = std::getenv("CSG_TRIG_FETCH") != nullptr;
  FetchTicket published;  // seq 0: the trips come back through k_fetch
  // bins need 44 B per tick; after the merge the last block of a sampled
  // rank stages its window statistics behind the tick times (8 + 40 B)
  static_assert(sizeof(WinStat) == 40, "WinStat layout");
  const size_t tsmem = static_cast<size_t>(T) * (8 + sizeof(WinStat));
  if (tsmem <= 200 * 1024) {
    DevBuf& acc = c->buf("trig.acc");
    const size_t sb = static_cast<size_t>(T) * S * sizeof(WinSum);
    const size_t mb = static_cast<size_t>(T) * S * sizeof(WinMax);
    const size_t db = (static_cast<size_t>(S) + 1) * 4;
    acc.ensure(sb + mb + db + 16);
    CSG_CUDA(cudaMemsetAsync(acc.p, 0, sb + mb + db, c->stream));
    WinSum* asum = acc.as<WinSum>();
    WinMax* amax = reinterpret_cast<WinMax*>(acc.as<unsigned char>() + sb);
    unsigned* done = reinterpret_cast<unsigned*>(acc.as<unsigned char>() + sb + mb);
    // about 512 records per block of a sampled rank's (average) segment
    const uint64_t avg = s->R > 0 ? s->n / static_cast<uint64_t>(s->R) : 0;
    const int32_t B = static_cast<int32_t>(std::min<uint64_t>(64, std::max<uint64_t>(1, avg / 512)));
    smem_optin(k_trigger, 200 * 1024);
    smem_optin(k_trigger_ema, 200 * 1024);
    const bool sharded = comm_active(c);
    TrigPublish pub;
    if (!no_publish) {  // the compacting block publishes the trips
      HostBuf& hb = c->hbuf("trig.out");
      hb.ensure(16 + static_cast<size_t>(T) * sizeof(csg_trigger_event));
      c->sig.ensure(64);
      pub.h = hb.as<unsigned char>();
      pub.max_seg = s->max_seg_pending ? &s->stats_dev.as<StoreStats>()->max_seg : nullptr;
      pub.flag = c->sig.as<unsigned long long>();
      pub.seq = ++c->sig_seq;
    }
    {
      ProfScope ps_(c->lc, "k_trigger", c->stream);
      k_trigger<<<dim3(B, S), 512, tsmem, c->stream>>>(
          s->view(), d_ticks, T, d_sampled, S, p, B, asum, amax, done, trip.as<uint8_t>(),
          events.as<csg_trigger_event>(), dn.as<int32_t>(), sharded ? 0 : 1,
          sharded ? TrigPublish{} : pub);
    }
    if (pub.h && !sharded) {
      CSG_CUDA(cudaGetLastError());
      if (!c->ev_fetch) CSG_CUDA(cudaEventCreateWithFlags(&c->ev_fetch, cudaEventDisableTiming));
      CSG_CUDA(cudaEventRecord(c->ev_fetch, c->stream));
      published = FetchTicket{pub.seq};
    }
    if (sharded) {
      // shards own disjoint rank ranges: windows combine by sum / max
      comm_group_start(c);
      comm_allreduce(c, asum, sb / 8, ncclUint64, ncclSum);
      comm_allreduce(c, amax, mb / 8, ncclUint64, ncclMax);
      store_reduce_max_seg(s);
      comm_group_end(c);
      ProfScope ps_(c->lc, "k_trigger_ema", c->stream);
      k_trigger_ema<<<S, 512, tsmem, c->stream>>>(
          d_ticks, T, d_sampled, S, p, asum, amax, done, trip.as<uint8_t>(),
          events.as<csg_trigger_event>(), dn.as<int32_t>(), pub);
      if (pub.h) {
        CSG_CUDA(cudaGetLastError());
        if (!c->ev_fetch)
          CSG_CUDA(cudaEventCreateWithFlags(&c->ev_fetch, cudaEventDisableTiming));
        CSG_CUDA(cudaEventRecord(c->ev_fetch, c->stream));
        published = FetchTicket{pub.seq};
      }
    }
  } else {
  trigger_window_stats(s, d_ticks, T, d_sampled, S, p.delta, ws.as<WinStat>());
  comm_group_start(c);
  comm_allreduce(c, ws.p, static_cast<size_t>(T) * S * sizeof(WinStat) / 8, ncclUint64,
                 ncclSum);
  store_reduce_max_seg(s);
  comm_group_end(c);
  {
    ProfScope ps_(c->lc, "k_ema_ticks", c->stream);
    k_ema_ticks<<<(S + 127) / 128, 128, 0, c->stream>>>(ws.as<WinStat>(), T, S, p,
                                                        trip.as<uint8_t>());
  }
  {
    ProfScope ps_(c->lc, "k_pick_trips", c->stream);
    k_pick_trips<<<1, 1024, 0, c->stream>>>(trip.as<uint8_t>(), d_ticks, T,
                                            d_sampled, S,
                                            events.as<csg_trigger_event>(),
                                            dn.as<int32_t>());
  }
  }
  // one round trip: the trip count and every possible event slot together
  // pinned: [0] trip count, [8] longest store segment, [16..) event slots
  HostBuf& hb = c->hbuf("trig.out");
  hb.ensure(16 + static_cast<size_t>(T) * sizeof(csg_trigger_event));
  unsigned char* h = hb.as<unsigned char>();
  FetchArgs fa{};
  fa.add(dn.p, h, 4);
  fa.add(events.p, h + 16, static_cast<size_t>(T) * sizeof(csg_trigger_event));
  const bool ms = s->max_seg_pending;  // rides on the same round trip
  if (ms) fa.add(&s->stats_dev.as<StoreStats>()->max_seg, h + 8, 8);
  // the flow index's fix-up queues behind the fetch: the GPU runs it while
  // the host reads the trips (RCA needs it for any trip)
  const FetchTicket tk = published.seq ? published : ctx_fetch_issue(c, fa);
  store_flow_index_early(s);
  ctx_fetch_wait(c, tk);
  tl_mark("trigger sync returned");
  if (ms) {
    std::memcpy(&s->max_seg, h + 8, 8);
    s->max_seg_pending = false;
  }
  int32_t n = 0;
  std::memcpy(&n, h, 4);
  const csg_trigger_event* ev = reinterpret_cast<const csg_trigger_event*>(h + 16);
  c->h_events.assign(ev, ev + n);
  return n;
}

void trigger_evaluate_single(csg_store* s, const int32_t* sampled, int32_t S,
                             double t, csg_trigger_state* state,
                             const TrigParams& p, int* tripped,
                             csg_trigger_event* event) {
  csg_ctx* c = s->ctx;
  *tripped = 0;
  if (S <= 0) return;
  int32_t mx = 0;
  for (int32_t i = 0; i < S; ++i) {
    if (sampled[i] < 0)
      throw Error(CSG_ERR_ARG, "evaluate: negative sampled rank");
    mx = std::max(mx, sampled[i]);
  }
  state->ensure(mx + 1);
  // scratch reused across ticks (csg_evaluate is the per-tick API): the
  // sampled list and tick time travel in one upload, the trip flag and the
  // event come back in one mapped-memory round trip
  DevBuf& in = c->buf("eval.in");
  DevBuf& ws = c->buf("eval.ws");
  DevBuf& out = c->buf("eval.out");
  const size_t in_bytes = 8 + static_cast<size_t>(S) * 4;
  in.ensure(in_bytes);
  HostBuf& hin = c->hbuf("eval.in");
  hin.ensure(in_bytes);
  std::memcpy(hin.p, &t, 8);
  std::memcpy(hin.as<unsigned char>() + 8, sampled, static_cast<size_t>(S) * 4);
  CSG_CUDA(cudaMemcpyAsync(in.p, hin.p, in_bytes, cudaMemcpyHostToDevice, c->stream));
  ws.ensure(static_cast<size_t>(S) * sizeof(WinStat));
  out.ensure(16 + sizeof(csg_trigger_event));
  const double* d_t = in.as<double>();
  const int32_t* d_s = reinterpret_cast<const int32_t*>(in.as<unsigned char>() + 8);
  int32_t* d_tr = out.as<int32_t>();
  csg_trigger_event* d_ev = reinterpret_cast<csg_trigger_event*>(out.as<unsigned char>() + 16);
  trigger_window_stats(s, d_t, 1, d_s, S, p.delta, ws.as<WinStat>());
  if (comm_active(c)) {
    // a sampled rank lives on one shard; the others contribute empty
    // (all-zero) windows, so a SUM all-reduce yields the owner's window and
    // every rank evaluates (and persists) the same baselines
    comm_group_start(c);
    comm_allreduce(c, ws.p, static_cast<size_t>(S) * sizeof(WinStat) / 8, ncclUint64,
                   ncclSum);
    comm_group_end(c);
  }
  {
    ProfScope ps_(c->lc, "k_ema_single", c->stream);
    k_ema_single<<<1, 32, 0, c->stream>>>(ws.as<WinStat>(), d_s, S, p, t,
                                          state->slots.as<TrigSlot>(), d_ev, d_tr);
  }
  HostBuf& hb = c->hbuf("eval.out");
  hb.ensure(16 + sizeof(csg_trigger_event));
  FetchArgs fa{};
  fa.add(out.p, hb.p, 16 + sizeof(csg_trigger_event));
  ctx_sync(c, &fa);
  std::memcpy(tripped, hb.p, 4);
  std::memcpy(event, hb.as<unsigned char>() + 16, sizeof(*event));
}

}  // namespace csg

void csg_trigger_state::ensure(int32_t ranks) {
  if (ranks <= cap) return;
  int32_t nc = cap ? cap : 64;
  while (nc < ranks) nc *= 2;
  csg::DevBuf nb;
  nb.ensure(static_cast<size_t>(nc) * sizeof(TrigSlot));
  CSG_CUDA(cudaMemsetAsync(nb.p, 0, static_cast<size_t>(nc) * sizeof(TrigSlot),
                           ctx->stream));
  if (cap)
    CSG_CUDA(cudaMemcpyAsync(nb.p, slots.p, static_cast<size_t>(cap) * sizeof(TrigSlot),
                             cudaMemcpyDeviceToDevice, ctx->stream));
  std::swap(slots.p, nb.p);
  std::swap(slots.bytes, nb.bytes);
  cap = nc;
}
