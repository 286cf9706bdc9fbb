// nccl_dyn.cpp — run-time binding of NCCL (see nccl_dyn.h).
#include "nccl_dyn.h"

#include <dlfcn.h>

#include <cstdlib>
#include <mutex>

namespace tcse {

namespace {

void* open_nccl() {
    // an NCCL this process already runs (e.g. torch's), else the caller's
    // choice, else the default library path
    if (void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD))
        return h;
    if (const char* p = std::getenv("TCSE_NCCL_LIBRARY"))
        if (void* h = dlopen(p, RTLD_NOW | RTLD_GLOBAL))
            return h;
    if (void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL))
        return h;
    return dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
}

template <typename F>
bool bind(void* h, const char* name, F* f) {
    *f = reinterpret_cast<F>(dlsym(h, name));
    return *f != nullptr;
}

}  // namespace

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = open_nccl();
        if (!h) {
            api.why = "libnccl.so.2 not found (set TCSE_NCCL_LIBRARY)";
            return;
        }
        const bool ok = bind(h, "ncclGetUniqueId", &api.GetUniqueId) &&
                        bind(h, "ncclCommInitRank", &api.CommInitRank) &&
                        bind(h, "ncclCommInitAll", &api.CommInitAll) &&
                        bind(h, "ncclCommDestroy", &api.CommDestroy) &&
                        bind(h, "ncclAllGather", &api.AllGather) && bind(h, "ncclGroupStart", &api.GroupStart) &&
                        bind(h, "ncclGroupEnd", &api.GroupEnd) && bind(h, "ncclGetVersion", &api.GetVersion) &&
                        bind(h, "ncclGetErrorString", &api.GetErrorString);
        api.ok = ok;
        api.why = ok ? "ok" : "libnccl.so.2 lacks an expected symbol";
    });
    return api;
}

}  // namespace tcse
