// engine_internal.h — shared internals of the B200 trace-analysis engine.
#pragma once

#include <cstring>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "csg_engine.h"

namespace csg {

// Errors thrown inside the engine are mapped to csg_status at the C ABI.
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define CSG_CUDA(call)                                                      \
  do {                                                                      \
    cudaError_t e_ = (call);                                                \
    if (e_ != cudaSuccess)                                                  \
      throw ::csg::Error(CSG_ERR_RUNTIME,                                   \
                         std::string("CUDA: ") + cudaGetErrorString(e_) +   \
                             " at " __FILE__ ":" + std::to_string(__LINE__)); \
  } while (0)

// Programmatic dependent launch (PDL) for the latency-bound kernel chains
// (index scans -> scatter -> chunk maxima, the failure RCA): a kernel
// launched with launch_pdl may be scheduled while its predecessor's last
// blocks still run; it calls pdl_wait() before touching any memory (which
// returns once the predecessor has completed and its writes are visible),
// and every chain kernel calls pdl_trigger() at its start so the next one
// is launched as soon as all of its blocks are resident. Stream order is
// otherwise unchanged; CSG_NO_PDL=1 launches plainly.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#endif
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  CSG_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

// Dynamic shared-memory opt-in for a kernel on the CURRENT device.
// cudaFuncSetAttribute is per device, so the "already set" cache is keyed by
// (device, kernel) and holds the largest size granted; thread-safe.
void smem_optin_raw(const void* func, size_t bytes);
template <typename F>
inline void smem_optin(F* func, size_t bytes) {
  smem_optin_raw(reinterpret_cast<const void*>(func), bytes);
}

// Grow-only pinned host buffer mapped into the device address space
// (kernels write results straight into it; no separate copy-back).
struct HostBuf {
  void* p = nullptr;
  size_t bytes = 0;
  HostBuf() = default;
  HostBuf(const HostBuf&) = delete;
  HostBuf& operator=(const HostBuf&) = delete;
  ~HostBuf() {
    if (p) cudaFreeHost(p);
  }
  void ensure(size_t b) {
    if (b <= bytes) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    const size_t want = b < 4096 ? 4096 : b + b / 2;
    CSG_CUDA(cudaHostAlloc(&p, want, cudaHostAllocMapped | cudaHostAllocPortable));
    // recycled pinned pages keep their old contents: a completion word
    // (csg_ctx::sig) left at another context's sequence number would read
    // as an already-finished fetch (large staging buffers are always
    // written before they are read)
    std::memset(p, 0, want < (64u << 10) ? want : (64u << 10));
    bytes = want;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  HostBuf stage;  // pinned staging for asynchronous uploads (see upload())
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  // Ensures capacity; contents are NOT preserved.
  void ensure(size_t b) {
    if (b <= bytes) return;
    release();
    size_t want = b < 256 ? 256 : b;
    CSG_CUDA(cudaMalloc(&p, want));
    bytes = want;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Error flags raised by device code (bitwise OR into one u32).
enum : uint32_t {
  DEV_ERR_RC_TABLE = 1u << 0,      // check_rc_table invariant (DataError)
  DEV_ERR_POOL = 1u << 1,          // output pool overflow -> retry bigger
  DEV_ERR_TOO_MANY_COMPS = 1u << 2,// > kFlowBuf completions of one (rank,op)
  DEV_ERR_K_TOO_LARGE = 1u << 3,   // consecutive_iterations_k > kMaxK
  DEV_ERR_DAG_SCRATCH = 1u << 4,   // reachability scratch too small
  DEV_ERR_SCRATCH = 1u << 5,       // generic scratch overflow -> retry
};

constexpr int kMaxK = 64;         // consecutive_iterations_k supported
constexpr int kFlowBuf = 256;     // completions per (rank, op) in a window
constexpr uint32_t kNoPos = 0xFFFFFFFFu;

// Rank-major, structure-of-arrays view of the store built by the index.
// Interleaved column: element i is field OFF of a STRIDE-wide rank-major
// record. The index builder writes {ts, op_seq} and {comm, channel, store
// index, kind | op_name} with one 16-byte store each (full sectors on the
// scattered write side when a digit run holds two records); readers index
// columns as before.
template <typename T, int STRIDE, int OFF>
struct ColView {
  const T* p = nullptr;
  __host__ __device__ __forceinline__ T operator[](uint64_t i) const {
    return p[i * STRIDE + OFF];
  }
};

// Payload words read straight from the packed store record of a rank-major
// position (perm): the index does not copy the 16-byte payload, which only
// the window sums, progress lookups and straggler durations touch. Word 1 of
// a state record is rdma_done alone (the reserved lane masked off).
template <int W>
struct PayView {
  const unsigned char* recs = nullptr;  // packed records (48 B each)
  ColView<uint32_t, 4, 2> perm;         // store index (meta word 2)
  __device__ __forceinline__ uint64_t operator[](uint64_t p) const {
    const unsigned char* r = recs + static_cast<uint64_t>(perm[p]) * 48;
    const uint64_t v = *reinterpret_cast<const unsigned long long*>(r + 32 + 8 * W);
    if (W == 1 && (r[28] & 1)) return v & 0xffffffffull;  // CSG_KIND_STATE
    return v;
  }
};

struct StoreView {
  uint64_t n = 0;          // records
  int32_t R = 0;           // rank space [0, R)
  int32_t nch = 0;         // channel space [0, nch)
  const uint32_t* rank_off = nullptr;  // [R+1]
  ColView<uint32_t, 4, 2> perm;        // rank-major pos -> store index (meta word 2)
  const double* cmax = nullptr;        // per-rank chunked prefix max of ts
                                       // (chunk c of rank r at r + off[r]/128 + c)
  ColView<double, 2, 0> ts;            // {ts, op_seq} pairs
  ColView<int64_t, 2, 1> op;
  // 16-byte meta record per position: {comm, channel, store index, kind |
  // op_name << 1} — written by the index with one 16-byte store
  ColView<int32_t, 4, 0> comm;
  ColView<int32_t, 4, 1> chan;
  ColView<uint8_t, 16, 12> ko;         // kind | op_name << 1
  PayView<0> pa;                       // payload: start_ms bits | ready | tx << 32
  PayView<1> pb;                       //          msg_bytes | done
};

constexpr uint32_t kCmChunk = 128;  // records per cmax chunk

// Rank owning rank-major position p (p < n): upper_bound over rank_off.
__device__ inline int32_t rank_at(const StoreView& s, uint32_t p) {
  int32_t lo = 0, hi = s.R;  // rank_off[lo] <= p < rank_off[hi]
  while (hi - lo > 1) {
    const int32_t m = (lo + hi) >> 1;
    if (s.rank_off[m] <= p) lo = m; else hi = m;
  }
  return lo;
}

// Flow index view (see store_build_flow_index): inside each rank segment
// [rank_off[r], rank_off[r+1]) the positions ordered by (op_seq, store
// order). A segment whose op_seq is already non-decreasing in store order
// (every simulator trace) is its own flow order: unsorted[r] == 0 and the
// identity is used; otherwise pos[] holds that segment's permutation.
struct FlowView {
  uint64_t n = 0;                      // 0: no flow index (prefix scans)
  const uint32_t* unsorted = nullptr;  // per rank
  const uint32_t* pos = nullptr;       // rank-major positions
  __device__ uint32_t at(bool uns, uint32_t i) const { return uns ? pos[i] : i; }
};

__host__ __device__ inline int ko_kind(uint8_t ko) { return ko & 1; }
__host__ __device__ inline int ko_opname(uint8_t ko) { return ko >> 1; }

// Device model tables (topology + program), see csg_model_create.
struct ModelView {
  int32_t world_size = 0;
  int32_t n_groups = 0;
  int32_t rank_space = 0;          // max(world, max member + 1)
  const uint8_t* group_kind = nullptr;
  const uint32_t* member_off = nullptr;  // [G+1]
  const int32_t* members = nullptr;
  const uint32_t* member_slot = nullptr; // first-occurrence membership slot
  const int32_t* comp = nullptr;         // connected component per group
  const int64_t* group_first_op = nullptr;  // per group; opn when none
  const uint32_t* rg_off = nullptr;      // rank -> (group, slot) CSR [RS+1]
  const int32_t* rg_group = nullptr;
  const uint32_t* rg_slot = nullptr;
  int32_t opn = 0;
  const uint8_t* op_name = nullptr;      // [opn]
  const uint32_t* par_off = nullptr;     // parents per program op [opn+1]
  const int32_t* par_op = nullptr;
  const int8_t* par_it = nullptr;        // iteration offset 0 or -1
  int32_t n_levels = 0;
  const uint32_t* lvl_off = nullptr;     // [n_levels+1]
  const int32_t* lvl_ops = nullptr;      // ops ordered by level
  const int32_t* op_level = nullptr;     // level of each program op [opn]
  int32_t max_deg = 0;                   // most parents of one program op
};

// Ordered-key transform for doubles (non-NaN): unsigned compare == double
// compare except -0 < +0.
__host__ __device__ inline uint64_t dkey(double d) {
  uint64_t u;
  memcpy(&u, &d, 8);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__host__ __device__ inline double dkey_inv(uint64_t k) {
  uint64_t u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  double d;
  memcpy(&d, &u, 8);
  return d;
}

// C++ truncating division, as static_cast<long>(op_seq / opn) in the
// reference (proj/src/rca.cpp:339, :533, :813, :824).
__host__ __device__ inline int64_t iter_of(int64_t op, int64_t opn) {
  return op / opn;
}

}  // namespace csg
