// comm.cuh — NCCL collectives on the engine stream (sharded stores).
#pragma once

#include <nccl.h>

#include "objects.h"

namespace csg {

bool comm_active(const csg_ctx* c);
// In-place all-reduce of count elements on the context stream (no-op alone).
void comm_allreduce(csg_ctx* c, void* ptr, size_t count, ncclDataType_t t,
                    ncclRedOp_t op);
void comm_allgather(csg_ctx* c, const void* send, void* recv, size_t count,
                    ncclDataType_t t);
void comm_group_start(csg_ctx* c);
void comm_group_end(csg_ctx* c);
size_t nccl_type_size(ncclDataType_t t);

}  // namespace csg

void csg_comm_release(csg_ctx* ctx);
