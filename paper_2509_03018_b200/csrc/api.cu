// api.cu — the engine's C ABI (include/csg_engine.h): handles, model
// tables, run_detection orchestration and result packaging. No exception
// crosses this boundary; every entry point maps failures to csg_status and
// the thread-local message of csg_last_error().
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <unordered_map>
#include <string>
#include <vector>

#include "comm.cuh"
#include "objects.h"
#include "fetch.cuh"
#include "rca.cuh"
#include "rca_table.h"
#include "trigger.cuh"

namespace csg {

namespace {
thread_local std::string g_err;

template <typename Fn>
csg_status guarded(Fn&& fn) {
  try {
    return fn();
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<csg_status>(e.status);
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return CSG_ERR_RUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CSG_ERR_RUNTIME;
  }
}

csg_status fail(csg_status s, const char* msg) {
  g_err = msg;
  return s;
}

// splitmix64 finalizer: the reference's counter-based mixing
// (proj/include/collsight/types.hpp:78-87).
inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
inline uint64_t mix64(uint64_t a, uint64_t b) { return mix64(a ^ mix64(b)); }

struct UnionFind {
  std::vector<int32_t> p;
  explicit UnionFind(int32_t n) : p(n) { std::iota(p.begin(), p.end(), 0); }
  int32_t find(int32_t x) {
    while (p[x] != x) x = p[x] = p[p[x]];
    return x;
  }
  void unite(int32_t a, int32_t b) {
    a = find(a);
    b = find(b);
    if (a != b) p[std::max(a, b)] = std::min(a, b);
  }
};

template <typename T>
void put(DevBuf& b, const std::vector<T>& v, cudaStream_t st) {
  b.ensure(v.size() * sizeof(T) + sizeof(T));
  if (!v.empty())
    CSG_CUDA(cudaMemcpyAsync(b.p, v.data(), v.size() * sizeof(T),
                             cudaMemcpyHostToDevice, st));
}

}  // namespace

void set_error(const std::string& msg) { g_err = msg; }

std::vector<int32_t> sample_ranks_host(const csg_model* m, int32_t cap_i,
                                       uint64_t seed) {
  // sample_ranks (proj/src/trigger.cpp:29-55): one rank per DP group; a
  // seeded subset of groups when there are more groups than the cap.
  std::vector<int32_t> dp;
  for (int32_t g = 0; g < m->n_groups; ++g)
    if (m->h_kind[g] == CSG_GROUP_DP) dp.push_back(g);
  const size_t cap = static_cast<size_t>(std::max(cap_i, 0));
  if (dp.size() > cap) {
    std::sort(dp.begin(), dp.end(), [&](int32_t a, int32_t b) {
      const uint64_t ka = mix64(seed, static_cast<uint64_t>(a) | (1ull << 32));
      const uint64_t kb = mix64(seed, static_cast<uint64_t>(b) | (1ull << 32));
      if (ka != kb) return ka < kb;
      return a < b;
    });
    dp.resize(cap);
  }
  std::vector<int32_t> out;
  for (int32_t g : dp) {
    const uint32_t b = m->h_member_off[g], e = m->h_member_off[g + 1];
    if (e == b) continue;
    const uint64_t pick = mix64(seed, static_cast<uint64_t>(g)) % (e - b);
    out.push_back(m->h_members[b + pick]);
  }
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  return out;
}

void store_append_jsonl_mem(csg_store* s, const char* text, uint64_t len, int* accepted);
void store_append_jsonl_file(csg_store* s, const char* path, int* accepted);
void store_query(csg_store* s, const int32_t* ranks, size_t nr, double t0,
                 double t1, std::vector<uint64_t>& out);
void store_last_log(csg_store* s, const int32_t* members, size_t nm, double t,
                    std::vector<std::pair<int32_t, uint64_t>>& out);

}  // namespace csg

using namespace csg;

void csg_results::finalize() {
  views.resize(ofs.size());
  for (size_t i = 0; i < ofs.size(); ++i) {
    csg_report_view& v = views[i];
    const Ofs& o = ofs[i];
    v.suspects = o.nsus ? suspects.data() + o.sus : nullptr;
    v.n_suspects = o.nsus;
    v.exonerated = o.nexo ? suspects.data() + o.exo : nullptr;
    v.n_exonerated = o.nexo;
    v.affected_groups = o.naff ? affected.data() + o.aff : nullptr;
    v.n_affected = o.naff;
    v.evidence = o.nev ? evidence.data() + o.ev : nullptr;
    v.n_evidence = o.nev;
  }
}

namespace {

// RcaResult (device pools) -> csg_results (host, one report per trip).
csg_results* package(const RcaResult& r, const csg_trigger_event* trips,
                     int32_t J) {
  auto* res = new csg_results();
  res->ofs.resize(J);
  res->views.resize(J);
  for (int32_t j = 0; j < J; ++j) {
    const TripOut& t = r.trips[j];
    csg_results::Ofs o;
    o.sus = res->suspects.size();
    o.nsus = t.n_sus;
    for (uint32_t i = 0; i < t.n_sus; ++i)
      res->suspects.push_back(r.sus[t.sus_off + i]);
    o.exo = res->suspects.size();
    o.nexo = t.n_exo;
    for (uint32_t i = 0; i < t.n_exo; ++i)
      res->suspects.push_back(r.sus[t.exo_off + i]);
    o.aff = res->affected.size();
    o.naff = t.n_aff;
    for (int32_t i = 0; i < t.n_aff; ++i)
      res->affected.push_back(r.aff[static_cast<size_t>(j) * r.G + i]);
    o.ev = res->evidence.size();
    o.nev = t.n_ev;
    for (uint32_t i = 0; i < t.n_ev; ++i)
      res->evidence.push_back(r.ev[t.ev_off + i]);
    res->ofs[j] = o;
    csg_report_view& v = res->views[j];
    std::memset(&v, 0, sizeof(v));
    v.verdict = t.verdict;
    v.trigger = trips[j];
    v.records_scanned = t.scanned;
  }
  res->finalize();
  return res;
}

}  // namespace

namespace csg {
namespace {
// Copies up to kFetchSegs small device regions into mapped pinned host
// memory, then publishes the sequence number: one launch instead of one
// DMA copy per region plus a wait (each copy-engine transfer costs several
// microseconds of latency on the path between two analysis phases).
// Copies the fetch segments into mapped pinned host memory, then raises the
// completion word the host polls. Several blocks share the copies (PCIe
// writes from one SM were ~10 us for the affected-group rows); the last
// block to finish (device-side counter) fences and raises the flag.
constexpr unsigned kFetchBlocks = 8;
__global__ void k_fetch(FetchArgs a, unsigned long long* flag, unsigned long long v,
                        unsigned* __restrict__ done) {
  const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nt = gridDim.x * blockDim.x;
  fetch_copy(a, gt, nt);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(done, 1u);
    if (prev == gridDim.x - 1) {
      *done = 0;  // ready for the next fetch
      __threadfence_system();
      *reinterpret_cast<volatile unsigned long long*>(flag) = v;
      __threadfence_system();
    }
  }
}
}  // namespace

bool pdl_enabled() {
  static const bool on = std::getenv("CSG_NO_PDL") == nullptr;
  return on;
}

void smem_optin_raw(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> granted;
  int dev = 0;
  CSG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& g = granted[{dev, func}];
  if (g >= bytes) return;
  CSG_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(bytes)));
  g = bytes;
}

void ctx_sync(csg_ctx* c, const FetchArgs* fetch) {
  c->sig.ensure(64);
  volatile unsigned long long* f = c->sig.as<volatile unsigned long long>();
  const unsigned long long v = ++c->sig_seq;
  FetchArgs none{};
  DevBuf& dn = c->buf("fetch.done");
  if (dn.bytes < 16) {
    dn.ensure(16);
    CSG_CUDA(cudaMemsetAsync(dn.p, 0, 16, c->stream));
  }
  k_fetch<<<kFetchBlocks, 256, 0, c->stream>>>(fetch ? *fetch : none,
                                               c->sig.as<unsigned long long>(), v,
                                               dn.as<unsigned>());
  CSG_CUDA(cudaGetLastError());
  ++c->lc.launches;
  // spin briefly (the short waits of the analysis path), then let the
  // driver block; either way surface stream errors
  const auto t0 = std::chrono::steady_clock::now();
  while (*f < v) {
    if (std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(500)) {
      CSG_CUDA(cudaStreamSynchronize(c->stream));
      break;
    }
  }
  const cudaError_t e = cudaStreamQuery(c->stream);
  if (e != cudaSuccess && e != cudaErrorNotReady) CSG_CUDA(e);
  if (e == cudaErrorNotReady) CSG_CUDA(cudaStreamSynchronize(c->stream));
}
FetchTicket ctx_fetch_issue(csg_ctx* c, const FetchArgs& fetch) {
  c->sig.ensure(64);
  const unsigned long long v = ++c->sig_seq;
  DevBuf& dn = c->buf("fetch.done");
  if (dn.bytes < 16) {
    dn.ensure(16);
    CSG_CUDA(cudaMemsetAsync(dn.p, 0, 16, c->stream));
  }
  k_fetch<<<kFetchBlocks, 256, 0, c->stream>>>(fetch, c->sig.as<unsigned long long>(), v,
                                               dn.as<unsigned>());
  CSG_CUDA(cudaGetLastError());
  ++c->lc.launches;
  if (!c->ev_fetch) CSG_CUDA(cudaEventCreateWithFlags(&c->ev_fetch, cudaEventDisableTiming));
  CSG_CUDA(cudaEventRecord(c->ev_fetch, c->stream));
  return FetchTicket{v};
}

void ctx_fetch_wait(csg_ctx* c, const FetchTicket& t) {
  volatile unsigned long long* f = c->sig.as<volatile unsigned long long>();
  const auto t0 = std::chrono::steady_clock::now();
  while (*f < t.seq) {
    if (std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(500)) {
      CSG_CUDA(cudaEventSynchronize(c->ev_fetch));
      break;
    }
  }
  const cudaError_t e = cudaEventQuery(c->ev_fetch);
  if (e != cudaSuccess && e != cudaErrorNotReady) CSG_CUDA(e);
}
}  // namespace csg

extern "C" {

const char* csg_version(void) { return "0.1.0-b200"; }
const char* csg_last_error(void) { return g_err.c_str(); }

void csg_trigger_config_default(csg_trigger_config* o) {
  if (!o) return;
  o->delta_ms = 200.0;
  o->detect_interval_ms = 500.0;
  o->throughput_drop_factor = 0.5;
  o->interval_inflation_factor = 2.0;
  o->max_sampled_ranks = 10;
  o->warmup_windows = 3;
  o->ema_alpha = 0.3;
}

void csg_analysis_config_default(csg_analysis_config* o) {
  if (!o) return;
  o->straggler_threshold_ms = 1000.0;
  o->delta_ms = 200.0;
  o->flow_skew_factor = 2.0;
  o->consecutive_iterations_k = 3;
  o->reserved = 0;
}

csg_status csg_ctx_create(int device, csg_ctx** out) {
  if (!out) return fail(CSG_ERR_ARG, "null argument");
  return guarded([&] {
    int n = 0;
    CSG_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n)
      throw Error(CSG_ERR_ARG, "csg_ctx_create: no such CUDA device");
    CSG_CUDA(cudaSetDevice(device));
    auto* c = new csg_ctx();
    c->device = device;
    CSG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CSG_CUDA(cudaEventCreate(&c->ev_start));
    CSG_CUDA(cudaEventCreate(&c->ev_stop));
    *out = c;
    return CSG_OK;
  });
}

void csg_ctx_free(csg_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  csg_comm_release(c);
  c->scratch_a.release();
  c->scratch_b.release();
  c->scratch_c.release();
  cudaEventDestroy(c->ev_start);
  if (c->ev_fetch) cudaEventDestroy(c->ev_fetch);
  cudaEventDestroy(c->ev_stop);
  cudaStreamDestroy(c->stream);
  delete c;
}

csg_status csg_ctx_stats(csg_ctx* c, double* device_ms, uint64_t* launches) {
  if (!c) return fail(CSG_ERR_ARG, "null argument");
  if (device_ms) *device_ms = c->device_ms;
  if (launches) *launches = c->lc.launches;
  return CSG_OK;
}

void csg_ctx_reset_stats(csg_ctx* c) {
  if (!c) return;
  c->device_ms = 0;
  c->lc.launches = 0;
  c->h2d_bytes = c->d2h_bytes = 0;
  c->lc.prof.totals.clear();
}

csg_status csg_ctx_profile(csg_ctx* c, int enable) {
  if (!c) return fail(CSG_ERR_ARG, "null argument");
  c->lc.prof.enabled = enable != 0;
  return CSG_OK;
}

csg_status csg_ctx_kernel_stats(csg_ctx* c, char* json, size_t cap,
                                uint64_t* h2d, uint64_t* d2h) {
  if (!c) return fail(CSG_ERR_ARG, "null argument");
  return guarded([&] {
    CSG_CUDA(cudaStreamSynchronize(c->stream));
    c->lc.prof.collect();
    std::string o = "{";
    bool first = true;
    for (const auto& [name, t] : c->lc.prof.totals) {
      if (!first) o += ",";
      first = false;
      char buf[160];
      snprintf(buf, sizeof(buf), "\"%s\":[%.6f,%llu]", name.c_str(), t.first,
               static_cast<unsigned long long>(t.second));
      o += buf;
    }
    o += "}";
    if (json && cap) {
      const size_t k = std::min(cap - 1, o.size());
      std::memcpy(json, o.data(), k);
      json[k] = 0;
    }
    if (h2d) *h2d = c->h2d_bytes;
    if (d2h) *d2h = c->d2h_bytes;
    return CSG_OK;
  });
}

csg_status csg_store_invalidate(csg_store* s) {
  if (!s) return fail(CSG_ERR_ARG, "null argument");
  s->indexed = false;
  s->op_indexed = false;
  s->flow_indexed = false;
  s->flow_early = false;
  return CSG_OK;
}

csg_status csg_store_create(csg_ctx* ctx, csg_store** out) {
  if (!ctx || !out) return fail(CSG_ERR_ARG, "null argument");
  return guarded([&] {
    auto* s = new csg_store();
    s->ctx = ctx;
    *out = s;
    return CSG_OK;
  });
}

csg_status csg_store_reserve(csg_store* s, size_t cap) {
  if (!s) return fail(CSG_ERR_ARG, "null argument");
  return guarded([&] {
    CSG_CUDA(cudaSetDevice(s->ctx->device));
    if (cap * sizeof(csg_packed_record) > s->recs.bytes) {
      DevBuf nb;
      nb.ensure(cap * sizeof(csg_packed_record));
      if (s->n)
        CSG_CUDA(cudaMemcpyAsync(nb.p, s->recs.p, s->n * sizeof(csg_packed_record),
                                 cudaMemcpyDeviceToDevice, s->ctx->stream));
      CSG_CUDA(cudaStreamSynchronize(s->ctx->stream));
      std::swap(nb.p, s->recs.p);
      std::swap(nb.bytes, s->recs.bytes);
    }
    return CSG_OK;
  });
}

static csg_status append_impl(csg_store* s, const csg_packed_record* src,
                              size_t n, cudaMemcpyKind kind) {
  if (!s || (!src && n)) return fail(CSG_ERR_ARG, "null argument");
  return guarded([&] {
    if (!n) return CSG_OK;
    CSG_CUDA(cudaSetDevice(s->ctx->device));
    const size_t need = (s->n + n) * sizeof(csg_packed_record);
    if (need > s->recs.bytes) {
      size_t cap = std::max(need, s->recs.bytes * 2);
      DevBuf nb;
      nb.ensure(cap);
      if (s->n)
        CSG_CUDA(cudaMemcpyAsync(nb.p, s->recs.p, s->n * sizeof(csg_packed_record),
                                 cudaMemcpyDeviceToDevice, s->ctx->stream));
      CSG_CUDA(cudaStreamSynchronize(s->ctx->stream));
      std::swap(nb.p, s->recs.p);
      std::swap(nb.bytes, s->recs.bytes);
    }
    CSG_CUDA(cudaMemcpyAsync(s->recs.as<csg_packed_record>() + s->n, src,
                             n * sizeof(csg_packed_record), kind, s->ctx->stream));
    if (kind == cudaMemcpyHostToDevice) s->ctx->h2d_bytes += n * sizeof(csg_packed_record);
    s->n += n;
    s->indexed = false;
    s->op_indexed = false;
    s->flow_indexed = false;
    s->flow_early = false;
    return CSG_OK;
  });
}

csg_status csg_store_append(csg_store* s, const csg_packed_record* host,
                            size_t n) {
  return append_impl(s, host, n, cudaMemcpyHostToDevice);
}

csg_status csg_store_append_device(csg_store* s, const csg_packed_record* dev,
                                   size_t n) {
  return append_impl(s, dev, n, cudaMemcpyDeviceToDevice);
}

csg_status csg_store_append_jsonl(csg_store* s, const char* text, size_t len,
                                  int* accepted) {
  if (!s || (!text && len) || !accepted) return fail(CSG_ERR_ARG, "null argument");
  return guarded([&] {
    CSG_CUDA(cudaSetDevice(s->ctx->device));
    csg_ctx::Timed tm(s->ctx);
    store_append_jsonl_mem(s, text, len, accepted);
    return CSG_OK;
  });
}

csg_status csg_store_append_jsonl_file(csg_store* s, const char* path, int* accepted) {
  if (!s || !path || !accepted) return fail(CSG_ERR_ARG, "null argument");
  return guarded([&] {
    CSG_CUDA(cudaSetDevice(s->ctx->device));
    csg_ctx::Timed tm(s->ctx);
    store_append_jsonl_file(s, path, accepted);
    return CSG_OK;
  });
}

csg_status csg_store_records(const csg_store* s, csg_packed_record* host, size_t n) {
  if (!s || (!host && n)) return fail(CSG_ERR_ARG, "null argument");
  return guarded([&] {
    if (n > s->n) throw Error(CSG_ERR_ARG, "csg_store_records: n exceeds the store size");
    CSG_CUDA(cudaSetDevice(s->ctx->device));
    if (n)
      CSG_CUDA(cudaMemcpyAsync(host, s->recs.p, n * sizeof(csg_packed_record),
                               cudaMemcpyDeviceToHost, s->ctx->stream));
    CSG_CUDA(cudaStreamSynchronize(s->ctx->stream));
    return CSG_OK;
  });
}

csg_status csg_store_clear(csg_store* s) {
  if (!s) return fail(CSG_ERR_ARG, "null argument");
  s->n = 0;
  s->indexed = false;
  s->op_indexed = false;
  s->flow_indexed = false;
  s->flow_early = false;
  return CSG_OK;
}

size_t csg_store_size(const csg_store* s) { return s ? s->n : 0; }

csg_status csg_store_build_index(csg_store* s) {
  if (!s) return fail(CSG_ERR_ARG, "null argument");
  return guarded([&] {
    CSG_CUDA(cudaSetDevice(s->ctx->device));
    csg_ctx::Timed tm(s->ctx);
    store_build_index(s);
    return CSG_OK;
  });
}

void csg_store_free(csg_store* s) {
  if (!s) return;
  cudaSetDevice(s->ctx->device);
  cudaStreamSynchronize(s->ctx->stream);
  delete s;
}

csg_status csg_store_query(csg_store* s, const int32_t* ranks, size_t nr,
                           double t0, double t1, uint64_t* out, size_t cap,
                           size_t* n_out) {
  if (!s || (!ranks && nr) || !n_out) return fail(CSG_ERR_ARG, "null argument");
  return guarded([&] {
    CSG_CUDA(cudaSetDevice(s->ctx->device));
    std::vector<uint64_t> v;
    store_query(s, ranks, nr, t0, t1, v);
    *n_out = v.size();
    for (size_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
    return CSG_OK;
  });
}

csg_status csg_store_last_log_per_rank(csg_store* s, const int32_t* members,
                                       size_t nm, double t, int32_t* out_rank,
                                       uint64_t* out_idx, size_t* n_out) {
  if (!s || (!members && nm) || !n_out) return fail(CSG_ERR_ARG, "null argument");
  return guarded([&] {
    CSG_CUDA(cudaSetDevice(s->ctx->device));
    std::vector<std::pair<int32_t, uint64_t>> v;
    store_last_log(s, members, nm, t, v);
    *n_out = v.size();
    for (size_t i = 0; i < v.size(); ++i) {
      out_rank[i] = v[i].first;
      out_idx[i] = v[i].second;
    }
    return CSG_OK;
  });
}

csg_status csg_model_create(csg_ctx* ctx, const csg_topology_desc* td,
                            const csg_program_desc* pd, csg_model** out) {
  if (!ctx || !td || !pd || !out) return fail(CSG_ERR_ARG, "null argument");
  return guarded([&] {
    CSG_CUDA(cudaSetDevice(ctx->device));
    auto m = std::make_unique<csg_model>();
    m->ctx = ctx;
    static std::atomic<uint64_t> next_uid{1};
    m->uid = next_uid++;
    const int32_t G = td->n_groups;
    const int32_t opn = pd->n_ops;
    if (G < 0 || opn < 0) throw Error(CSG_ERR_ARG, "negative table size");
    m->world_size = td->world_size;
    m->n_groups = G;
    m->opn = opn;
    m->h_kind.assign(td->group_kind, td->group_kind + G);
    m->h_member_off.resize(G + 1);
    int32_t max_member = -1;
    for (int32_t g = 0; g <= G; ++g) {
      if (td->member_off[g] < 0 || td->member_off[g] > 0xFFFFFFF0ll)
        throw Error(CSG_ERR_ARG, "member_off out of range");
      m->h_member_off[g] = static_cast<uint32_t>(td->member_off[g]);
    }
    const uint32_t M = m->h_member_off[G];
    m->h_members.assign(td->members, td->members + M);
    for (int32_t g = 0; g < G; ++g) {
      std::vector<int32_t> mem(m->h_members.begin() + m->h_member_off[g],
                               m->h_members.begin() + m->h_member_off[g + 1]);
      for (int32_t r : mem) {
        if (r < 0) throw Error(CSG_ERR_CONFIG, "engine: negative group member");
        max_member = std::max(max_member, r);
      }
      std::sort(mem.begin(), mem.end());
      if (std::adjacent_find(mem.begin(), mem.end()) != mem.end())
        throw Error(CSG_ERR_CONFIG, "engine: duplicate member in a group");
    }
    m->h_member_slot.resize(M);
    for (uint32_t q = 0; q < M; ++q) m->h_member_slot[q] = q;
    m->rank_space = std::max({m->world_size, max_member + 1, 1});
    const int32_t RS = m->rank_space;
    // rank -> (group, slot), groups ascending (Topology::groups_of order)
    std::vector<std::vector<std::pair<int32_t, uint32_t>>> rg(RS);
    for (int32_t g = 0; g < G; ++g)
      for (uint32_t q = m->h_member_off[g]; q < m->h_member_off[g + 1]; ++q)
        rg[m->h_members[q]].emplace_back(g, q);
    m->h_rg_off.assign(RS + 1, 0);
    std::vector<uint32_t> rg_slot;
    for (int32_t r = 0; r < RS; ++r) {
      m->h_rg_off[r + 1] = m->h_rg_off[r] + static_cast<uint32_t>(rg[r].size());
      for (auto& [g, q] : rg[r]) {
        m->h_rg_group.push_back(g);
        rg_slot.push_back(q);
      }
    }
    // program tables
    m->h_op_name.assign(pd->op_name, pd->op_name + opn);
    std::vector<int64_t> gfo(G, opn);
    for (int32_t s = 0; s < opn; ++s) {
      const int32_t g = pd->group[s];
      if (g < 0 || g >= G)
        throw Error(CSG_ERR_CONFIG, "unknown comm_id " + std::to_string(g));
      gfo[g] = std::min<int64_t>(gfo[g], s);
      for (int64_t e = pd->dep_off[s]; e < pd->dep_off[s + 1]; ++e)
        if (pd->deps[e] < 0 || pd->deps[e] >= s)
          throw Error(CSG_ERR_CONFIG,
                      "program: op " + std::to_string(s) +
                          " depends on non-earlier op " + std::to_string(pd->deps[e]));
    }
    // connected components of the group graph (affected_groups adjacency,
    // proj/src/rca.cpp:427-439): program dependency pairs + groups sharing
    // a rank (ranks 0..world_size-1).
    UnionFind uf(std::max(G, 1));
    for (int32_t s = 0; s < opn; ++s)
      for (int64_t e = pd->dep_off[s]; e < pd->dep_off[s + 1]; ++e)
        uf.unite(pd->group[s], pd->group[pd->deps[e]]);
    for (int32_t r = 0; r < std::min(m->world_size, RS); ++r)
      for (size_t i = 0; i + 1 < rg[r].size(); ++i)
        uf.unite(rg[r][i].first, rg[r][i + 1].first);
    m->h_comp.resize(G);
    for (int32_t g = 0; g < G; ++g) m->h_comp[g] = uf.find(g);
    // DepIndex parents per program op (proj/src/rca.cpp:99-119): explicit
    // depends_on (same iteration) plus each executing rank's previous op,
    // which for its first op of an iteration is its last op of the previous
    // iteration.
    auto exec = [&](int32_t s) {
      std::vector<int32_t> v;
      if (pd->op_name[s] == CSG_OP_SEND) v.push_back(pd->src[s]);
      else if (pd->op_name[s] == CSG_OP_RECV) v.push_back(pd->dst[s]);
      else {
        const int32_t g = pd->group[s];
        for (uint32_t q = m->h_member_off[g]; q < m->h_member_off[g + 1]; ++q)
          v.push_back(m->h_members[q]);
      }
      return v;
    };
    std::vector<std::vector<int32_t>> ex(opn);
    std::unordered_map<int32_t, int32_t> last_of;
    for (int32_t s = 0; s < opn; ++s) {
      ex[s] = exec(s);
      for (int32_t r : ex[s]) last_of[r] = s;
    }
    std::vector<uint32_t> par_off(opn + 1, 0);
    std::vector<int32_t> par_op;
    std::vector<int8_t> par_it;
    std::vector<int32_t> level(opn, 0);
    std::unordered_map<int32_t, int32_t> prev;
    int32_t nlev = 0;
    for (int32_t s = 0; s < opn; ++s) {
      std::vector<std::pair<int8_t, int32_t>> ps;
      for (int64_t e = pd->dep_off[s]; e < pd->dep_off[s + 1]; ++e)
        ps.emplace_back(0, static_cast<int32_t>(pd->deps[e]));
      for (int32_t r : ex[s]) {
        auto it = prev.find(r);
        if (it != prev.end()) ps.emplace_back(0, it->second);
        else ps.emplace_back(-1, last_of[r]);
        prev[r] = s;
      }
      std::sort(ps.begin(), ps.end());
      ps.erase(std::unique(ps.begin(), ps.end()), ps.end());
      int32_t lv = 0;
      for (auto& [di, p] : ps) {
        par_it.push_back(di);
        par_op.push_back(p);
        if (di == 0) lv = std::max(lv, level[p] + 1);
      }
      level[s] = lv;
      nlev = std::max(nlev, lv + 1);
      par_off[s + 1] = static_cast<uint32_t>(par_op.size());
    }
    std::vector<uint32_t> lvl_off(nlev + 1, 0);
    for (int32_t s = 0; s < opn; ++s) ++lvl_off[level[s] + 1];
    for (int32_t l = 0; l < nlev; ++l) lvl_off[l + 1] += lvl_off[l];
    std::vector<int32_t> lvl_ops(opn);
    {
      std::vector<uint32_t> fill(lvl_off.begin(), lvl_off.end() - 1);
      for (int32_t s = 0; s < opn; ++s) lvl_ops[fill[level[s]]++] = s;
    }
    m->n_levels = nlev;
    cudaStream_t st = ctx->stream;
    put(m->group_kind, m->h_kind, st);
    put(m->member_off, m->h_member_off, st);
    put(m->members, m->h_members, st);
    put(m->member_slot, m->h_member_slot, st);
    put(m->comp, m->h_comp, st);
    put(m->group_first_op, gfo, st);
    put(m->rg_off, m->h_rg_off, st);
    put(m->rg_group, m->h_rg_group, st);
    put(m->rg_slot, rg_slot, st);
    put(m->op_name, m->h_op_name, st);
    put(m->par_off, par_off, st);
    put(m->par_op, par_op, st);
    put(m->par_it, par_it, st);
    put(m->lvl_off, lvl_off, st);
    put(m->lvl_ops, lvl_ops, st);
    put(m->op_level, level, st);
    {
      uint32_t md = 0;
      for (int32_t s2 = 0; s2 < opn; ++s2) md = std::max(md, par_off[s2 + 1] - par_off[s2]);
      m->max_deg = static_cast<int32_t>(md);
    }
    CSG_CUDA(cudaStreamSynchronize(st));
    *out = m.release();
    return CSG_OK;
  });
}

void csg_model_free(csg_model* m) { delete m; }

csg_status csg_sample_ranks(const csg_model* m, int32_t max_sampled,
                            uint64_t seed, int32_t* out, size_t cap,
                            size_t* n_out) {
  if (!m || !n_out) return fail(CSG_ERR_ARG, "null argument");
  return guarded([&] {
    const auto v = sample_ranks_host(m, max_sampled, seed);
    *n_out = v.size();
    for (size_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
    return CSG_OK;
  });
}

csg_status csg_trigger_state_create(csg_ctx* ctx, csg_trigger_state** out) {
  if (!ctx || !out) return fail(CSG_ERR_ARG, "null argument");
  return guarded([&] {
    auto* s = new csg_trigger_state();
    s->ctx = ctx;
    *out = s;
    return CSG_OK;
  });
}

void csg_trigger_state_free(csg_trigger_state* s) { delete s; }

csg_status csg_evaluate(csg_store* store, const int32_t* sampled, size_t ns,
                        double t, csg_trigger_state* state,
                        const csg_trigger_config* cfg, int* tripped,
                        csg_trigger_event* ev) {
  if (!store || (!sampled && ns) || !state || !cfg || !tripped || !ev)
    return fail(CSG_ERR_ARG, "null argument");
  return guarded([&] {
    CSG_CUDA(cudaSetDevice(store->ctx->device));
    csg_ctx::Timed tm(store->ctx);
    store_build_index(store);
    trigger_evaluate_single(store, sampled, static_cast<int32_t>(ns), t, state,
                            trig_params(*cfg), tripped, ev);
    return CSG_OK;
  });
}

csg_status csg_analyze(csg_store* store, const csg_model* model,
                       const csg_analysis_config* cfg,
                       const csg_trigger_event* trigger, int mode,
                       csg_results** out) {
  if (!store || !model || !cfg || !trigger || !out)
    return fail(CSG_ERR_ARG, "null argument");
  return guarded([&] {
    CSG_CUDA(cudaSetDevice(store->ctx->device));
    csg_ctx::Timed tm(store->ctx);
    csg_trigger_event t = *trigger;
    if (mode == 1) t.kind = CSG_TRIGGER_FAILURE;
    if (mode == 2) t.kind = CSG_TRIGGER_STRAGGLER;
    RcaResult r;
    rca_batch(store, model, *cfg, &t, 1, false, r);
    // reports carry the caller's trigger (its kind is reported as given)
    *out = package(r, trigger, 1);
    return CSG_OK;
  });
}

csg_status csg_affected_groups(csg_store* store, const csg_model* model,
                               const csg_analysis_config* cfg,
                               const csg_trigger_event* trigger, int32_t* out,
                               size_t cap, size_t* n_out, uint64_t* scanned) {
  if (!store || !model || !cfg || !trigger || !n_out)
    return fail(CSG_ERR_ARG, "null argument");
  return guarded([&] {
    CSG_CUDA(cudaSetDevice(store->ctx->device));
    csg_ctx::Timed tm(store->ctx);
    RcaResult r;
    rca_batch(store, model, *cfg, trigger, 1, true, r);
    const int32_t n = r.trips[0].n_aff;
    *n_out = n;
    for (int32_t i = 0; i < n && static_cast<size_t>(i) < cap; ++i) out[i] = r.aff[i];
    if (scanned) *scanned += store->n_global;  // records over all shards
    return CSG_OK;
  });
}

csg_status csg_run_detection(csg_store* store, const csg_model* model,
                             const csg_trigger_config* tcfg,
                             const csg_analysis_config* acfg, uint64_t seed,
                             csg_results** out, int32_t* sampled_out,
                             size_t sampled_cap, size_t* n_sampled) {
  if (!store || !model || !tcfg || !acfg || !out)
    return fail(CSG_ERR_ARG, "null argument");
  return guarded([&] {
    if (!(tcfg->detect_interval_ms > 0))
      throw Error(CSG_ERR_CONFIG, "trigger: detect_interval_ms must be > 0");
    csg_ctx* c = store->ctx;
    CSG_CUDA(cudaSetDevice(c->device));
    csg_ctx::Timed tm(c);
    const std::vector<int32_t> sampled =
        sample_ranks_host(model, tcfg->max_sampled_ranks, seed);
    if (n_sampled) *n_sampled = sampled.size();
    if (sampled_out)
      for (size_t i = 0; i < sampled.size() && i < sampled_cap; ++i)
        sampled_out[i] = sampled[i];
    store_build_index(store);
    DevBuf& ticks = c->buf("det.ticks");
    DevBuf& events = c->buf("det.events");
    DevBuf& d_s = c->buf("det.sampled");
    const int32_t T = trigger_ticks(store, tcfg->detect_interval_ms,
                                    tcfg->delta_ms, ticks);
    std::vector<csg_trigger_event> trips;
    if (T > 0 && !sampled.empty()) {
      d_s.ensure(sampled.size() * 4);
      CSG_CUDA(cudaMemcpyAsync(d_s.p, sampled.data(), sampled.size() * 4,
                               cudaMemcpyHostToDevice, c->stream));
      const int32_t n = trigger_run(store, ticks.as<double>(), T,
                                    d_s.as<int32_t>(),
                                    static_cast<int32_t>(sampled.size()),
                                    trig_params(*tcfg), events);
      trips.assign(c->h_events.begin(), c->h_events.begin() + n);
      c->d2h_bytes += static_cast<uint64_t>(T) * sizeof(csg_trigger_event) + 4;
    }
    RcaResult r;
    tl_mark("run_detection -> rca_batch");
    rca_batch(store, model, *acfg, trips.data(),
              static_cast<int32_t>(trips.size()), false, r);
    *out = package(r, trips.data(), static_cast<int32_t>(trips.size()));
    return CSG_OK;
  });
}

size_t csg_results_count(const csg_results* r) { return r ? r->views.size() : 0; }

csg_status csg_results_get(const csg_results* r, size_t i, csg_report_view* out) {
  if (!r || !out) return fail(CSG_ERR_ARG, "null argument");
  if (i >= r->views.size()) return fail(CSG_ERR_ARG, "index out of range");
  *out = r->views[i];
  return CSG_OK;
}

void csg_results_free(csg_results* r) { delete r; }

csg_status csg_check_min_op(const int32_t* ranks, const int64_t* ops, size_t n,
                            int32_t* out, size_t* n_out, int* has_min) {
  if ((!ranks || !ops) && n) return fail(CSG_ERR_ARG, "null argument");
  if (!out || !n_out || !has_min) return fail(CSG_ERR_ARG, "null argument");
  // check_min_op (proj/src/rca.cpp:249-261)
  if (n == 0) return fail(CSG_ERR_RUNTIME, "check_min_op: no last logs supplied");
  int64_t mn = ops[0];
  for (size_t i = 0; i < n; ++i) mn = std::min(mn, ops[i]);
  std::vector<int32_t> mins;
  for (size_t i = 0; i < n; ++i)
    if (ops[i] == mn) mins.push_back(ranks[i]);
  if (mins.size() == n) {
    *has_min = 0;
    *n_out = 0;
    return CSG_OK;
  }
  std::sort(mins.begin(), mins.end());
  *has_min = 1;
  *n_out = mins.size();
  std::copy(mins.begin(), mins.end(), out);
  return CSG_OK;
}

csg_status csg_check_min_data(const int32_t* ranks, const csg_progress* p,
                              size_t n, int32_t* out, size_t* n_out) {
  if ((!ranks || !p) && n) return fail(CSG_ERR_ARG, "null argument");
  if (!out || !n_out) return fail(CSG_ERR_ARG, "null argument");
  if (n == 0) return fail(CSG_ERR_RUNTIME, "check_min_data: no progress supplied");
  size_t best = 0;
  for (size_t i = 1; i < n; ++i)
    if (prog_less(p[i].rdma_done, p[i].rdma_transmitted, p[i].gpu_ready,
                  p[best].rdma_done, p[best].rdma_transmitted, p[best].gpu_ready))
      best = i;
  std::vector<int32_t> mins;
  for (size_t i = 0; i < n; ++i)
    if (p[i].rdma_done == p[best].rdma_done &&
        p[i].rdma_transmitted == p[best].rdma_transmitted &&
        p[i].gpu_ready == p[best].gpu_ready)
      mins.push_back(ranks[i]);
  std::sort(mins.begin(), mins.end());
  *n_out = mins.size();
  std::copy(mins.begin(), mins.end(), out);
  return CSG_OK;
}

csg_status csg_check_rc_table(const csg_progress* c, const csg_progress* peer,
                              int* category, int* side) {
  if (!c || !category || !side) return fail(CSG_ERR_ARG, "null argument");
  const bool ok = rc_table(c->gpu_ready, c->rdma_transmitted, c->rdma_done,
                           peer != nullptr, peer ? peer->gpu_ready : 0,
                           peer ? peer->rdma_transmitted : 0,
                           peer ? peer->rdma_done : 0, category, side);
  if (!ok)
    return fail(CSG_ERR_RUNTIME,
                "check_rc_table: counters violate the pipeline invariant");
  return CSG_OK;
}

}  // extern "C"
