// synth_gpu.cu — device expansion of the synthetic generator's flows
// (SURVEY.md §8(f) "trace generator at scale").
//
// The host (host/synth.cpp, synth_plan) schedules the op instances — a
// sequential pass over (iteration, op) with O(executing ranks) work each —
// and hands over one Flow per (instance, rank). Every flow expands, per
// channel, into its state snapshots, flush and completion (synth_flow.h,
// the same code the host generator runs); the store order is emission time,
// ties in emission sequence. On the device that is:
//   k_syn_count   thread per (flow, channel): records it emits (filters)
//   scan          exclusive offsets = emission sequence numbers
//   k_syn_write   thread per (flow, channel): records into a scratch array,
//                 their ordered time keys and sequence numbers alongside
//   radix sort    stable LSD sort of (time key, sequence) pairs, 64 bits
//   k_syn_gather  the first `target` records, in order, onto the store
// which replaces the host generator's O(N log N) sort of 64-byte tuples
// (minutes at 1e9 records) with a few HBM passes.
#include <algorithm>

#include "objects.h"
#include "sort.cuh"
#include "synth_flow.h"

namespace csg {
namespace {

__device__ __forceinline__ unsigned long long time_key(double d) {
  unsigned long long u;
  memcpy(&u, &d, 8);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void k_syn_count(const csg_synth::Flow* __restrict__ flows, uint64_t nf,
                            csg_synth::Params P, uint32_t* __restrict__ cnt) {
  const uint64_t total = nf * static_cast<uint64_t>(P.cpp);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const csg_synth::Flow f = flows[i / P.cpp];
    const int ch = static_cast<int>(i % P.cpp);
    uint32_t c = 0;
    csg_synth::expand(P, f, ch, [&](double key, const csg_packed_record& r) {
      if (csg_synth::keep(P, key, r.rank)) ++c;
    });
    cnt[i] = c;
  }
}

__global__ void k_syn_sum(const uint32_t* __restrict__ cnt, uint64_t n,
                          unsigned long long* __restrict__ tot) {
  unsigned long long acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    acc += cnt[i];
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(tot, acc);
}

__global__ void k_syn_write(const csg_synth::Flow* __restrict__ flows, uint64_t nf,
                            csg_synth::Params P, const uint32_t* __restrict__ off,
                            csg_packed_record* __restrict__ out,
                            unsigned long long* __restrict__ keys,
                            uint32_t* __restrict__ seq) {
  const uint64_t total = nf * static_cast<uint64_t>(P.cpp);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const csg_synth::Flow f = flows[i / P.cpp];
    const int ch = static_cast<int>(i % P.cpp);
    uint32_t at = off[i];
    csg_synth::expand(P, f, ch, [&](double key, const csg_packed_record& r) {
      if (!csg_synth::keep(P, key, r.rank)) return;
      out[at] = r;
      keys[at] = time_key(key);
      seq[at] = at;
      ++at;
    });
  }
}

__global__ void k_syn_gather(const csg_packed_record* __restrict__ src,
                             const uint32_t* __restrict__ seq, uint64_t n,
                             csg_packed_record* __restrict__ dst) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const ulonglong2* s = reinterpret_cast<const ulonglong2*>(src + seq[i]);
    ulonglong2* d = reinterpret_cast<ulonglong2*>(dst + i);
    d[0] = s[0];
    d[1] = s[1];
    d[2] = s[2];
  }
}

unsigned grid_of(uint64_t n) {
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148ull * 32)));
}

}  // namespace

uint64_t synth_append_device(csg_store* s, const csg_synth::Flow* flows, size_t n_flows,
                             const csg_synth::Params& P, uint64_t target) {
  csg_ctx* c = s->ctx;
  cudaStream_t st = c->stream;
  CSG_CUDA(cudaSetDevice(c->device));
  if (n_flows == 0 || P.cpp <= 0) return 0;
  const uint64_t items = static_cast<uint64_t>(n_flows) * P.cpp;
  DevBuf fl, cnt, recs, keys, seq;
  fl.ensure(n_flows * sizeof(csg_synth::Flow));
  CSG_CUDA(cudaMemcpyAsync(fl.p, flows, n_flows * sizeof(csg_synth::Flow),
                           cudaMemcpyHostToDevice, st));
  cnt.ensure((items + 1) * 4);
  CSG_CUDA(cudaMemsetAsync(cnt.as<uint32_t>() + items, 0, 4, st));
  k_syn_count<<<grid_of(items), 256, 0, st>>>(fl.as<csg_synth::Flow>(), n_flows, P,
                                             cnt.as<uint32_t>());
  // the records' total must fit the scan's u32 offsets (sequence numbers)
  {
    DevBuf tot;
    tot.ensure(8);
    CSG_CUDA(cudaMemsetAsync(tot.p, 0, 8, st));
    k_syn_sum<<<grid_of(items), 256, 0, st>>>(cnt.as<uint32_t>(), items,
                                             tot.as<unsigned long long>());
    unsigned long long t64 = 0;
    CSG_CUDA(cudaMemcpyAsync(&t64, tot.p, 8, cudaMemcpyDeviceToHost, st));
    CSG_CUDA(cudaStreamSynchronize(st));
    if (t64 > 0xFFFFFFF0ull)
      throw Error(CSG_ERR_RUNTIME, "synth: more than 2^32 records in one call (shard the ranks)");
    exclusive_scan_u32(cnt.as<uint32_t>(), items + 1, c->buf("synth.scan"), st, c->lc);
  }
  uint32_t n32 = 0;
  CSG_CUDA(cudaMemcpyAsync(&n32, cnt.as<uint32_t>() + items, 4, cudaMemcpyDeviceToHost, st));
  CSG_CUDA(cudaStreamSynchronize(st));
  const uint64_t n = n32;
  if (n == 0) return 0;
  recs.ensure(n * sizeof(csg_packed_record));
  keys.ensure(n * 8);
  seq.ensure(n * 4);
  k_syn_write<<<grid_of(items), 256, 0, st>>>(fl.as<csg_synth::Flow>(), n_flows, P,
                                             cnt.as<uint32_t>(), recs.as<csg_packed_record>(),
                                             keys.as<unsigned long long>(), seq.as<uint32_t>());
  fl.release();
  cnt.release();
  {
    SortScratch sc;
    radix_sort_u64(keys.as<uint64_t>(), seq.as<uint32_t>(), n, 64, sc, st, c->lc);
  }
  keys.release();
  const uint64_t m = target && target < n ? target : n;
  const size_t need = (s->n + m) * sizeof(csg_packed_record);
  if (need > s->recs.bytes) {
    DevBuf nb;
    nb.ensure(need);
    if (s->n)
      CSG_CUDA(cudaMemcpyAsync(nb.p, s->recs.p, s->n * sizeof(csg_packed_record),
                               cudaMemcpyDeviceToDevice, st));
    CSG_CUDA(cudaStreamSynchronize(st));
    std::swap(nb.p, s->recs.p);
    std::swap(nb.bytes, s->recs.bytes);
  }
  k_syn_gather<<<grid_of(m), 256, 0, st>>>(recs.as<csg_packed_record>(), seq.as<uint32_t>(), m,
                                          s->recs.as<csg_packed_record>() + s->n);
  CSG_CUDA(cudaGetLastError());
  CSG_CUDA(cudaStreamSynchronize(st));
  s->n += m;
  s->indexed = false;
  s->op_indexed = false;
  s->flow_indexed = false;
  return m;
}

}  // namespace csg
