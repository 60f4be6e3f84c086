// NCCL entry points, resolved at run time from the process's libnccl (the one
// torch loads), so libdr has no link-time NCCL dependency.
#pragma once
#include <nccl.h>

#include <string>

#include "dr_internal.h"

namespace dr {

struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*commCount)(const ncclComm_t, int *) = nullptr;
    ncclResult_t (*commUserRank)(const ncclComm_t, int *) = nullptr;
    ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                              ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*reduceScatter)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                                  ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char *(*getErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*commGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
};

NcclApi &nccl();    // throws DR_ERR_NCCL when libnccl or a symbol is missing

#define DR_NCCL(call)                                                                        \
    do {                                                                                     \
        ncclResult_t r_ = (call);                                                            \
        if (r_ != ncclSuccess)                                                               \
            ::dr::fail(DR_ERR_NCCL, std::string(#call) + ": " + ::dr::nccl().getErrorString(r_)); \
    } while (0)

}  // namespace dr
