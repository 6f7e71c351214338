// comm.cu — NCCL plumbing for rank-range sharded stores.
//
// Records are sharded by rank range: shard p holds every record of its ranks
// in their original store order, so every per-rank prefix quantity is local.
// Each per-rank / per-slot table the analysis needs from other shards is
// produced with all-zero (or min/max identity) entries for ranks a shard does
// not own, and one NCCL all-reduce on the engine stream (sum / min / max over
// NVLink) makes it global; the decision kernels then run replicated on every
// GPU on identical inputs. NCCL is loaded with dlopen so single-GPU use never
// needs it.
#include <dlfcn.h>

#include <cstring>
#include <string>

#include "comm.cuh"
#include "objects.h"

namespace csg {
namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                            ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (api.h) return api;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* n : names) {
    api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (api.h) break;
  }
  if (!api.h)
    throw Error(CSG_ERR_RUNTIME, std::string("NCCL not loadable: ") + dlerror());
  auto sym = [&](const char* s) {
    void* p = dlsym(api.h, s);
    if (!p) throw Error(CSG_ERR_RUNTIME, std::string("NCCL symbol missing: ") + s);
    return p;
  };
  api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
  api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
  api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
  api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
  api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
  api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
  api.GetErrorString =
      reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  return api;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(CSG_ERR_RUNTIME,
                std::string("NCCL ") + what + ": " + nccl().GetErrorString(r));
}

}  // namespace

bool comm_active(const csg_ctx* c) { return c->nranks > 1 && c->comm; }

void comm_allreduce(csg_ctx* c, void* ptr, size_t count, ncclDataType_t t,
                    ncclRedOp_t op) {
  if (!comm_active(c) || count == 0) return;
  ++c->collectives;
  ProfScope ps_(c->lc, c->comm_group_depth ? "nccl_in_group" : "nccl_allreduce", c->stream,
                false);
  check(nccl().AllReduce(ptr, ptr, count, t, op, static_cast<ncclComm_t>(c->comm),
                         c->stream),
        "allreduce");
}

void comm_group_start(csg_ctx* c) {
  if (!comm_active(c)) return;
  if (c->comm_group_depth++ == 0 && c->lc.prof.enabled) {
    cudaEvent_t a = c->lc.prof.take();
    cudaEventRecord(a, c->stream);
    c->lc.prof.pending.push_back({"nccl_group", a, nullptr, 0.0});
    c->group_rec = c->lc.prof.pending.size() - 1;
  }
  check(nccl().GroupStart(), "group start");
}
void comm_group_end(csg_ctx* c) {
  if (!comm_active(c)) return;
  check(nccl().GroupEnd(), "group end");
  if (--c->comm_group_depth == 0 && c->lc.prof.enabled && c->group_rec < c->lc.prof.pending.size()) {
    cudaEvent_t b = c->lc.prof.take();
    cudaEventRecord(b, c->stream);
    c->lc.prof.pending[c->group_rec].b = b;
  }
}

void comm_allgather(csg_ctx* c, const void* send, void* recv, size_t count,
                    ncclDataType_t t) {
  if (!comm_active(c)) {
    if (send != recv)
      CSG_CUDA(cudaMemcpyAsync(recv, send, count * nccl_type_size(t),
                               cudaMemcpyDeviceToDevice, c->stream));
    return;
  }
  ++c->collectives;
  ProfScope ps_(c->lc, c->comm_group_depth ? "nccl_in_group" : "nccl_allgather", c->stream,
                false);
  check(nccl().AllGather(send, recv, count, t, static_cast<ncclComm_t>(c->comm),
                         c->stream),
        "allgather");
}

size_t nccl_type_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    case ncclInt64: case ncclUint64: case ncclFloat64: return 8;
    default: return 2;
  }
}

}  // namespace csg

using namespace csg;

extern "C" {

csg_status csg_comm_unique_id(unsigned char* out, size_t cap) {
  if (!out || cap < sizeof(ncclUniqueId)) {
    set_error("csg_comm_unique_id: buffer smaller than 128 bytes");
    return CSG_ERR_ARG;
  }
  try {
    ncclUniqueId id;
    check(nccl().GetUniqueId(&id), "get unique id");
    std::memcpy(out, &id, sizeof(id));
    return CSG_OK;
  } catch (const Error& e) {
    set_error(e.what());
    return static_cast<csg_status>(e.status);
  }
}

csg_status csg_ctx_comm_init(csg_ctx* ctx, const unsigned char* id, size_t len,
                             int nranks, int rank) {
  if (!ctx || !id || len < sizeof(ncclUniqueId) || nranks < 1 || rank < 0 ||
      rank >= nranks) {
    set_error("csg_ctx_comm_init: invalid argument");
    return CSG_ERR_ARG;
  }
  try {
    CSG_CUDA(cudaSetDevice(ctx->device));
    ctx->nranks = nranks;
    ctx->rank = rank;
    if (nranks == 1) return CSG_OK;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t comm;
    check(nccl().CommInitRank(&comm, nranks, uid, rank), "comm init");
    ctx->comm = comm;
    return CSG_OK;
  } catch (const Error& e) {
    set_error(e.what());
    return static_cast<csg_status>(e.status);
  }
}

csg_status csg_ctx_comm_info(csg_ctx* ctx, int* nranks, int* rank,
                             uint64_t* collectives) {
  if (!ctx) {
    set_error("null argument");
    return CSG_ERR_ARG;
  }
  if (nranks) *nranks = ctx->nranks;
  if (rank) *rank = ctx->rank;
  if (collectives) *collectives = ctx->collectives;
  return CSG_OK;
}

}  // extern "C"

void csg_comm_release(csg_ctx* ctx) {
  if (ctx && ctx->comm) {
    nccl().CommDestroy(static_cast<ncclComm_t>(ctx->comm));
    ctx->comm = nullptr;
  }
}
