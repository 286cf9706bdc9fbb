// nccl_dyn.h — the few NCCL entry points the exchange uses, resolved at run
// time (dlopen/dlsym) instead of linked.
//
// A Python host has usually loaded torch's libnccl.so.2 already; linking the
// system copy into libtcse.so would put two NCCL builds with one soname in
// the process.  The loader prefers an NCCL already in the process
// (RTLD_NOLOAD), then TCSE_NCCL_LIBRARY, then the default search path, so the
// library never decides which NCCL the process runs and loads none unless a
// multi-rank exchange is asked for.  Types and values are NCCL's own
// (nccl.h), only the calls go through the table.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

namespace tcse {

struct NcclApi {
    bool ok = false;
    const char* why = "not loaded";
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// process-wide, loaded on first use (thread-safe)
const NcclApi& nccl();

}  // namespace tcse
