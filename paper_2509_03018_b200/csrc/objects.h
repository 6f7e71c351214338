// objects.h — the engine's handle types (behind the opaque C ABI handles).
#pragma once

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "engine_internal.h"
#include "sort.cuh"

struct csg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_start = nullptr, ev_stop = nullptr;
  cudaEvent_t ev_fetch = nullptr;  // recorded after an issued fetch (ctx_fetch_issue)
  double device_ms = 0;
  uint64_t h2d_bytes = 0, d2h_bytes = 0;
  // sharded mode (csg_ctx_comm_init): NCCL communicator over nranks GPUs
  void* comm = nullptr;
  int nranks = 1, rank = 0;
  uint64_t collectives = 0;
  int comm_group_depth = 0;   // NCCL group nesting (timeline records)
  size_t group_rec = ~size_t(0);
  csg::LaunchCounter lc;
  std::vector<double> h_ticks;  // detection tick times (host-computed)
  std::vector<csg_trigger_event> h_events;  // trips of the last trigger_run
  // shared scratch
  csg::DevBuf scratch_a, scratch_b, scratch_c, pinned_flag_dev;
  uint32_t* host_flag = nullptr;  // pinned
  // Named grow-only device buffers reused across calls (no cudaMalloc /
  // cudaFree on the analysis path once warm).
  std::map<std::string, csg::DevBuf> arena;
  csg::DevBuf& buf(const char* name) { return arena[name]; }
  std::map<std::string, csg::HostBuf> host_arena;  // mapped pinned buffers
  uint64_t slot_group_uid = 0;
  uint64_t rca_bits_cap = 0;   // op-DAG scratch words that sufficed last time
  uint64_t rca_pool_mult = 1;  // straggler pool growth that sufficed last time
  // low-latency host wait (ctx_sync): a mapped pinned word the stream's
  // last kernel sets; the host polls it instead of sleeping in the driver
  csg::HostBuf sig;
  uint64_t sig_seq = 0;  // model whose slot -> group table is in "rca.slot_group"
  csg::HostBuf& hbuf(const char* name) { return host_arena[name]; }

  // Times an engine phase on the context stream with CUDA events.
  struct Timed {
    csg_ctx* c;
    explicit Timed(csg_ctx* ctx) : c(ctx) {
      cudaEventRecord(c->ev_start, c->stream);
    }
    ~Timed() {
      cudaEventRecord(c->ev_stop, c->stream);
      if (cudaEventSynchronize(c->ev_stop) == cudaSuccess) {
        float ms = 0;
        cudaEventElapsedTime(&ms, c->ev_start, c->ev_stop);
        c->device_ms += ms;
      }
      c->lc.prof.collect();
    }
  };
};

struct StoreStats {
  unsigned long long ts_max_key;  // dkey of max timestamp
  int min_rank, max_rank;
  int min_chan, max_chan;
  long long min_op, max_op;
  unsigned long long n_nan;
  unsigned long long n_total;  // records over all shards
  int lmin_rank, lmax_rank;    // this shard's own rank range (not reduced)
  unsigned long long max_seg;  // longest rank segment (k_runmax_blk)
  unsigned int overlap;        // sharded: two shards' own rank ranges overlap
  unsigned int pad_;
};

struct csg_store {
  csg_ctx* ctx = nullptr;
  csg::DevBuf recs;  // packed AoS in store (emission) order
  uint64_t n = 0;
  uint64_t n_global = 0;  // records over all shards (== n unsharded)
  bool indexed = false;
  // stats (valid when indexed)
  double last_ts = 0;  // max(0, max timestamp), runner.cpp:51-56
  int32_t min_rank = 0, max_rank = -1;
  int32_t own_lo = 0, own_hi = -1;  // this shard's own rank range (local records)
  int32_t min_chan = 0, max_chan = -1;
  int64_t min_op = 0, max_op = -1;
  // rank-major index
  int32_t R = 0, nch = 0;
  uint64_t max_seg = 0;  // longest rank segment
  bool max_seg_pending = false;  // still on the device (stats_dev->max_seg)
  bool max_seg_unreduced = false;  // sharded: not yet MAX-reduced over the shards
  // layout of the last fused index build: the next build launches its
  // scatter on it before the statistics reach the host (store_build_index)
  bool spec_ok = false;
  bool spec_general = false;  // last build took the general path (stats + keys first)
  int32_t sp_lmin = 0, sp_lmax = -1, sp_R = 0;
  csg::DevBuf rank_off, perm, keys;  // perm, keys: general-path sort pairs
  csg::DevBuf runmax;  // chunked prefix max of ts (StoreView::cmax)
  csg::DevBuf tso;  // {ts, op_seq} per rank-major position (16 B)
  csg::DevBuf meta;  // {comm, channel, store index, kind | op_name << 1} (16 B)
  csg::SortScratch sort;
  // op-ordered completion index for the straggler self-evidence pass
  bool op_indexed = false;
  uint64_t n_opidx = 0;
  csg::DevBuf opidx_pos;     // rank-major positions of non-Recv completions,
                             // ordered by (op_seq, store index)
  csg::DevBuf opidx_keys;    // u64 op - min_op (sorted)
  csg::DevBuf opidx_rank;    // rank of each entry
  csg::DevBuf opidx_ts;      // end_ms (timestamp) of each entry
  csg::DevBuf opidx_dur;     // end_ms - start_ms
  csg::DevBuf opidx_nm;      // record op_name
  csg::DevBuf op_seg_off;    // dense [min_op, max_op+1] -> start in opidx
  // flow index: per rank segment, positions ordered by (op_seq, store
  // order); identity for segments already ordered (see FlowView)
  bool flow_indexed = false;
  bool flow_early = false;  // k_flow_fix launched ahead of the trip round trip
  csg::DevBuf fl_unsorted;  // u32 flag per rank
  csg::DevBuf fl_list;      // ranks with a descending op_seq (work list)
  csg::DevBuf fl_cnt;       // [0] list length, [1] overflow count
  csg::DevBuf fl_pos;       // u32 rank-major positions (unsorted segments)
  csg::DevBuf fl_keys;      // global-sort fallback scratch
  csg::DevBuf stats_dev;

  csg::StoreView view() const {
    csg::StoreView v;
    v.n = n;
    v.R = R;
    v.nch = nch;
    v.rank_off = rank_off.as<uint32_t>();
    v.perm.p = meta.as<uint32_t>();
    v.cmax = runmax.as<double>();
    v.ts.p = tso.as<double>();
    v.op.p = tso.as<int64_t>();
    v.comm.p = meta.as<int32_t>();
    v.chan.p = meta.as<int32_t>();
    v.ko.p = meta.as<uint8_t>();
    v.pa.recs = recs.as<unsigned char>();
    v.pa.perm.p = meta.as<uint32_t>();
    v.pb.recs = recs.as<unsigned char>();
    v.pb.perm.p = meta.as<uint32_t>();
    return v;
  }
  csg::FlowView flow_view() const {
    csg::FlowView f;
    f.n = flow_indexed ? n : 0;
    f.unsorted = fl_unsorted.as<uint32_t>();
    f.pos = fl_pos.as<uint32_t>();
    return f;
  }
};

struct csg_model {
  csg_ctx* ctx = nullptr;
  // host copies
  int32_t world_size = 0, n_groups = 0, rank_space = 0, opn = 0;
  std::vector<uint8_t> h_kind;
  std::vector<uint32_t> h_member_off;
  std::vector<int32_t> h_members;
  std::vector<uint32_t> h_member_slot;
  std::vector<int32_t> h_comp;
  std::vector<uint32_t> h_rg_off;
  std::vector<int32_t> h_rg_group;
  std::vector<uint8_t> h_op_name;
  int32_t n_levels = 0;
  int32_t max_deg = 0;  // most parents of one program op
  uint64_t uid = 0;  // unique per model object (context-side table caches)
  // device copies
  csg::DevBuf group_kind, member_off, members, member_slot, comp,
      group_first_op, rg_off, rg_group, rg_slot, op_name, par_off, par_op,
      par_it, lvl_off, lvl_ops, op_level;
  csg::ModelView view() const {
    csg::ModelView v;
    v.world_size = world_size;
    v.n_groups = n_groups;
    v.rank_space = rank_space;
    v.group_kind = group_kind.as<uint8_t>();
    v.member_off = member_off.as<uint32_t>();
    v.members = members.as<int32_t>();
    v.member_slot = member_slot.as<uint32_t>();
    v.comp = comp.as<int32_t>();
    v.group_first_op = group_first_op.as<int64_t>();
    v.rg_off = rg_off.as<uint32_t>();
    v.rg_group = rg_group.as<int32_t>();
    v.rg_slot = rg_slot.as<uint32_t>();
    v.opn = opn;
    v.op_name = op_name.as<uint8_t>();
    v.par_off = par_off.as<uint32_t>();
    v.par_op = par_op.as<int32_t>();
    v.par_it = par_it.as<int8_t>();
    v.n_levels = n_levels;
    v.lvl_off = lvl_off.as<uint32_t>();
    v.lvl_ops = lvl_ops.as<int32_t>();
    v.op_level = op_level.as<int32_t>();
    v.max_deg = max_deg;
    return v;
  }
};

// Trigger baselines (proj/include/collsight/trigger.hpp:29-50), one slot per
// rank id, resident on the device.
struct TrigSlot {
  double throughput;
  double op_interval_ms;
  int32_t interval_defined;
  int32_t updates;
  int32_t had_prev;
  int32_t pad;
};

struct csg_trigger_state {
  csg_ctx* ctx = nullptr;
  int32_t cap = 0;
  csg::DevBuf slots;  // TrigSlot[cap], zero = fresh
  void ensure(int32_t ranks);
};

struct csg_results {
  std::vector<csg_report_view> views;
  std::vector<csg_suspect> suspects;
  std::vector<csg_evidence> evidence;
  std::vector<int32_t> affected;
  // per report: offsets into the vectors above
  struct Ofs {
    size_t sus, nsus, exo, nexo, aff, naff, ev, nev;
  };
  std::vector<Ofs> ofs;
  void finalize();
};

namespace csg {

void store_build_index(csg_store* s);
void store_build_op_index(csg_store* s, int32_t opn);
// Returns false (and builds nothing) when the packed key exceeds 64 bits.
bool store_build_flow_index(csg_store* s);
void store_flow_index_early(csg_store* s);
// Waits until everything enqueued on the context stream has completed
// (spins on a mapped flag, falls back to cudaStreamSynchronize; errors are
// reported like cudaStreamSynchronize's).
// fetch (optional): small device regions copied into mapped host memory by
// the same kernel that publishes completion.
struct FetchSeg {
  const unsigned char* src;
  unsigned char* dst;
  uint32_t bytes;
  // row mode (row_len != nullptr): nrows rows of stride `bytes`, row i holds
  // row_len[i] (device) 4-byte elements — only those are copied
  const int32_t* row_len;
  uint32_t nrows;
};
constexpr int kFetchSegs = 8;
struct FetchArgs {
  FetchSeg seg[kFetchSegs];
  int n;
  void add(const void* src, void* dst, size_t bytes) {
    if (n >= kFetchSegs) throw csg::Error(CSG_ERR_RUNTIME, "fetch: too many segments");
    seg[n++] = FetchSeg{static_cast<const unsigned char*>(src),
                        static_cast<unsigned char*>(dst), static_cast<uint32_t>(bytes),
                        nullptr, 0};
  }
  void add_rows(const void* src, void* dst, size_t stride, const int32_t* lens,
                uint32_t nrows) {
    if (n >= kFetchSegs) throw csg::Error(CSG_ERR_RUNTIME, "fetch: too many segments");
    seg[n++] = FetchSeg{static_cast<const unsigned char*>(src),
                        static_cast<unsigned char*>(dst), static_cast<uint32_t>(stride),
                        lens, nrows};
  }
};
void ctx_sync(csg_ctx* c, const FetchArgs* fetch = nullptr);
// Split round trip: enqueue the fetch now, keep enqueueing work, wait for the
// fetched bytes later (without draining the work queued after the fetch).
struct FetchTicket {
  uint64_t seq = 0;
};
FetchTicket ctx_fetch_issue(csg_ctx* c, const FetchArgs& fetch);
void ctx_fetch_wait(csg_ctx* c, const FetchTicket& t);
// Brings stats_dev->max_seg to the host if still pending (one round trip).
void store_resolve_max_seg(csg_store* s);
// Sharded stores: enqueue the MAX all-reduce of the longest segment if it is
// still local (callers may be inside an NCCL group).
void store_reduce_max_seg(csg_store* s);

// Per-thread error text for csg_last_error.
void set_error(const std::string& msg);

}  // namespace csg
