// host.cpp — C ABI (include/tcse.h) over the sm_100a search kernels.
//
// Host orchestration of the search path, B200-first:
//   * a system is packed once into per-variable occurrence bitsets and its
//     candidate list is computed ON THE DEVICE (search kernel, dump mode);
//   * every optimize_system iteration is one search launch over all
//     processes of all concurrently optimized systems (U, V and W of a scheme
//     share launches) plus one reduce launch that updates the HBM-resident
//     incumbent pool and the next iteration's reinit set;
//   * the host only reads a few bytes of incumbent state per iteration to
//     drive patience and the on_iteration callback;
//   * with a rank partition, the per-iteration costs and each rank's best
//     record are all-gathered and the same reduce runs on every rank, so the
//     result is identical for any world size.
// Semantics follow parallel_search.hpp:117-273 and cse_engine.hpp:29-57.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <utility>
#include <atomic>
#include <condition_variable>
#include <array>
#include <random>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <functional>
#include <map>
#include <unordered_map>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "launch.h"
#include "nccl_dyn.h"

namespace tcse {
cudaError_t launch_search(const LaunchDesc& L, int W, int nt, bool dense, int form, int smem, cudaStream_t st);
struct ReduceLaunch;
}  // namespace tcse

namespace tcse {
struct VerifyDesc {  // verify.cu
    int32_t m, n, p, r;
    int32_t method;
    int32_t trials;
    int64_t off_u, off_v, off_w, off_ab;
    int64_t n_checks;
};
cudaError_t launch_verify(const VerifyDesc* d_descs, const int8_t* d_coef, unsigned long long* d_first, int count,
                          long long max_checks, int max_trials, int max_r, int n_sms, cudaStream_t st);
cudaError_t launch_pack(const XchgLaunch& XL, cudaStream_t st);
cudaError_t launch_reduce(const XchgLaunch& XL, int hist_n, cudaStream_t st);
int barrier_blocks(int n);
}  // namespace tcse

using namespace tcse;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CU(call)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return fail(TCSE_ECUDA, "cuda: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                      \
    } while (0)

inline u32 make_key(int i, int j, int neg) { return (u32(i) << 17) | (u32(j) << 1) | u32(neg); }
inline tcse_pair key_pair(u32 k) {
    tcse_pair p;
    p.i = int(k >> 17);
    p.j = int((k >> 1) & 0xffffu);
    p.rel_sign = (k & 1u) ? -1 : 1;
    return p;
}

int launch_words(int need) {
    static const int ws[] = {1, 2, 3, 4, 8};
    for (int w : ws)
        if (w >= need)
            return w;
    return -1;
}

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}

// Process-wide caching allocator: every C-ABI call is synchronous, so a
// buffer released by a finished call can be reused by the next one without
// the cost (and implicit device synchronisation) of cudaFree/cudaMalloc.
// Power-of-two buckets per device; memory is retained until process exit.
struct DeviceCache {
    std::mutex mu;
    std::multimap<std::pair<int, size_t>, void*> free_blocks;
};

DeviceCache& device_cache() {
    static DeviceCache* c = new DeviceCache;  // never destroyed: outlives static DBufs
    return *c;
}

size_t bucket_bytes(size_t bytes) {
    size_t b = 256;
    while (b < bytes)
        b <<= 1;
    return b;
}

cudaError_t cache_get(size_t bytes, void** p) {
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t b = bucket_bytes(bytes);
    {
        std::lock_guard<std::mutex> lock(device_cache().mu);
        auto it = device_cache().free_blocks.find({dev, b});
        if (it != device_cache().free_blocks.end()) {
            *p = it->second;
            device_cache().free_blocks.erase(it);
            return cudaSuccess;
        }
    }
    return cudaMalloc(p, b);
}

void cache_put(void* p, size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(device_cache().mu);
    device_cache().free_blocks.insert({{dev, bucket_bytes(bytes)}, p});
}

// device buffer that grows, never shrinks (storage from the cache above)
struct DBuf {
    void* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    cudaError_t reserve(size_t bytes) {
        if (bytes <= n)
            return cudaSuccess;
        if (p)
            cache_put(p, n);
        p = nullptr;
        n = 0;
        cudaError_t e = cache_get(bytes, &p);
        if (e == cudaSuccess)
            n = bucket_bytes(bytes);
        return e;
    }
    ~DBuf() {
        if (p)
            cache_put(p, n);
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// A validated system (LinearSystem constructor, linear_system.hpp:84-101)
struct HostSys {
    int n_x = 0, n_e = 0, naive = 0, vcap = 0, mcap = 0, w_need = 1;
    std::vector<std::vector<int>> rows;
};

int validate_system(const tcse_system* s, HostSys* out) {
    if (!s)
        return fail(TCSE_EINVAL, "linear system: null system");
    if (s->n_x < 0)
        return fail(TCSE_EINVAL, "linear system: negative variable count");
    if (s->n_e < 0)
        return fail(TCSE_EINVAL, "linear system: negative expression count");
    out->n_x = s->n_x;
    out->n_e = s->n_e;
    out->rows.assign(size_t(s->n_e), {});
    long long occ = 0;
    int naive = 0;
    std::vector<int> seen(size_t(s->n_x) + 1, -1);
    for (int r = 0; r < s->n_e; ++r) {
        auto& row = out->rows[size_t(r)];
        for (int t = s->row_ptr[r]; t < s->row_ptr[r + 1]; ++t) {
            const int term = s->terms[t];
            if (term == 0 || std::abs(term) > s->n_x)
                return fail(TCSE_EINVAL, "linear system: index %d out of range in expression %d", term, r);
            const int v = std::abs(term);
            if (seen[size_t(v)] == r) {
                for (int x : row)
                    if (x == -term)
                        return fail(TCSE_EINVAL, "linear system: expression %d contains both signs of x%d", r, v);
                return fail(TCSE_EINVAL, "linear system: duplicate term in expression %d", r);
            }
            seen[size_t(v)] = r;
            row.push_back(term);
        }
        const long long t = (long long)row.size();
        occ += t * (t - 1) / 2;
        if (t > 0)
            naive += int(t) - 1;
    }
    out->naive = naive;
    out->vcap = s->n_x + naive;
    out->mcap = int(std::max<long long>(1, occ / 2));
    out->w_need = std::max(1, (s->n_e + 63) / 64);
    if (out->vcap > kMaxVars)
        return fail(TCSE_ECAPACITY, "system too large: %d variables (limit %d)", out->vcap, kMaxVars);
    if (out->mcap >= 65535 || out->mcap > kCoinWords * 32)
        return fail(TCSE_ECAPACITY, "system too large: %d candidate pairs", out->mcap);
    if (launch_words(out->w_need) < 0)
        return fail(TCSE_ECAPACITY, "system too large: %d expressions (limit 512)", s->n_e);
    return TCSE_OK;
}

std::vector<u64> pack_masks(const HostSys& h, int W) {
    std::vector<u64> m(size_t(h.n_x) * 2 * size_t(W), 0ULL);
    for (int r = 0; r < h.n_e; ++r)
        for (int term : h.rows[size_t(r)]) {
            const int v = std::abs(term) - 1;
            const size_t off = size_t(v) * 2 * size_t(W) + (term > 0 ? 0 : size_t(W)) + size_t(r >> 6);
            m[off] |= 1ULL << (r & 63);
        }
    return m;
}

}  // namespace

struct tcse_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t owned_stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int nt = 0;
    int rank = 0, world = 1;
    tcse_allgather_fn allgather = nullptr;
    void* ag_user = nullptr;
    ncclComm_t comm = nullptr;  // payload all-gather on `stream` (tcse_set_nccl / tcse_create_devices)
    bool own_comm = false;
    std::vector<tcse_ctx*> sub;  // multi-device context: rank r runs on sub[r]
    std::shared_ptr<void> local_gather;  // test transport of a shared-device context (below)
    DBuf err;  // int32 err + err_pos
    DBuf slots, rng, perm, hist;  // prep_kernel -> search_kernel hand-off
    // launch groups beyond the first run on their own streams, forked from and
    // joined back into `stream` with events
    cudaStream_t aux[kMaxSys] = {};
    cudaEvent_t fork = nullptr, join[kMaxSys] = {};
};

// one system prepared on the device
struct DevSys {
    HostSys h;
    int W = 1;         // mask words the kernel is instantiated with
    int nt = 64;       // block size (threads per process)
    bool dense = true; // Greedy-Intersections form
    bool bm = false;   // dense layout with per-variable candidate bitmaps
    bool small = false;  // the small-list instantiation (search.cu gi_dense_small)
    bool nt_auto = true; // block size chosen here (not forced by TCSE_NT)
    DBuf masks, keys, cnts;
    int base_m = 0;
    int mcap_full = 0;  // > 0: h.mcap was shrunk to the starting list + slack
};

// the kernel form of a system's launch (search.cu kFormBm / kFormSmall)
inline int kernel_form(const DevSys& d) { return (d.bm ? kFormBm : 0) | (d.small ? kFormSmall : 0); }

namespace {

int coin_words_for(const HostSys& h) {
    // gi coin bits: all coins of a step fit for typical states (sum of
    // degrees), else the kernel evaluates gi densely in chunks
    const long long want = (long long)h.mcap * 24 / 32 + 8;
    static const int floor_words = env_int("TCSE_COIN_MIN", 64);
    // TCSE_COIN_MAX (test hook): a small buffer forces many coin chunks per step
    // (never below one candidate's coins: deg q <= 2 (mcap - 1))
    const int cap_words = std::max((2 * h.mcap + 31) / 32 + 1, std::min(env_int("TCSE_COIN_MAX", 2048), 2048));
    return int(std::min<long long>(std::max<long long>(want, std::min(floor_words, cap_words)), cap_words));
}

// gi evaluation form: the O(deg) walk pays off once candidate lists are long
int gi_dense_for(const HostSys& h) {
    const int forced = env_int("TCSE_GI_DENSE", -1);
    if (forced >= 0)
        return forced ? 1 : 0;
    return h.mcap <= 640 ? 1 : 0;
}

// (W, NT) pairs search_kernel is instantiated for (search.cu launch_search_w)
bool instantiated(int W, int nt) {
    switch (nt) {
        case 32: return W == 1;
        case 64: return W <= 2;
        case 128: return W == 1 || W == 2 || W == 3 || W == 4 || W == 8;
        case 256: return W >= 1 && W <= 4;
        default: return false;
    }
}

// Launch shape of one system: mask words, block size (one warp for small
// candidate lists, wider blocks for long ones) and the gi form.  None of
// these changes results.
void choose_launch(const tcse_ctx* ctx, DevSys* d) {
    d->W = launch_words(d->h.w_need);
    d->dense = gi_dense_for(d->h) != 0;
    int nt = ctx->nt;
    d->nt_auto = nt == 0;
    static const int nt64_max = env_int("TCSE_NT64_MAX", 1024);  // candidate capacity up to which two warps serve
    if (nt == 0) {
        if (d->W == 1 && d->h.mcap <= 96)
            nt = 32;  // one warp per process
        else if (d->W <= 2 && d->h.mcap <= nt64_max)
            nt = 64;
        else if (d->h.mcap <= 1024)
            nt = 128;
        else
            nt = 256;  // long candidate lists: more candidates scored in parallel
    }
    if (!instantiated(d->W, nt))
        nt = 128;
    d->nt = nt;
}

// gi form on the actual starting list (lists only shrink): the dense
// reference loop up to 512 candidates, the O(deg) walk beyond (sweep on every
// fixture)
void pick_bm(DevSys* d, int keep = 3);
std::pair<int, int> bm_residency(DevSys* d);
bool bm_instantiated(int W, int nt);

void pick_form(DevSys* d) {
    static const int dense_max = env_int("TCSE_GI_DENSE_MAX", 512);
    if (env_int("TCSE_GI_DENSE", -1) < 0)
        d->dense = d->base_m <= dense_max;
    pick_bm(d);
    // two-warp systems whose bitmaps cost residency: four warps (half the
    // resident processes by registers, so the bitmaps' shared memory costs
    // relatively less) keep them at no more than a quarter — better than
    // two warps with fewer blocks (5x5x5 W: +19% over two warps without
    // bitmaps, +4% over two warps with them; four warps without them -12%).
    // TCSE_NT128_BM=0 disables.
    static const int bm128 = env_int("TCSE_NT128_BM", 1);
    if (bm128 && !d->bm && d->nt_auto && d->dense && d->nt == 64 && d->base_m > 32 &&
        env_int("TCSE_GI_BM", -1) < 0 && bm_instantiated(d->W, 128)) {
        d->nt = 128;
        pick_bm(d);
        if (!d->bm)
            d->nt = 64;
    }
    // still none: bitmaps worth up to half the resident processes (keep k =
    // TCSE_BM_KEEP of 4) — the popcount scoring they enable outweighs the
    // blocks (6x6x6 U/V at four warps: +3..5%)
    static const int keep = env_int("TCSE_BM_KEEP", 2);
    if (!d->bm && d->base_m > 32)
        pick_bm(d, keep);
}

int smem_one(const DevSys& d) {
    Lay L;
    return int(carve(&L, d.W, d.nt, d.h.vcap, d.h.mcap, d.h.n_e, coin_words_for(d.h), d.dense, d.bm));
}

// processes per SM the register cap allows (search.cu MinBlocks)
int reg_blocks(int nt) { return nt == 32 ? 28 : (nt == 64 ? 14 : (nt == 128 ? 8 : 4)); }

// shapes with a bitmap-pruned instantiation (search.cu launch_search_w)
bool bm_instantiated(int W, int nt) {
    return (W == 1 && (nt == 32 || nt == 64 || nt == 128)) || (W == 2 && (nt == 64 || nt == 128)) ||
           ((W == 3 || W == 4) && nt == 128);
}

// Per-variable candidate bitmaps (O(m/32 + deg) pruned gi scoring) whenever
// the dense layout prunes and the bitmaps ((V+1) * ceil(mcap/32) words more
// shared memory per process) cost at most a quarter of the resident processes.
// TCSE_GI_BM=0/1 forces (results never depend on it).
// resident processes per SM without and with the bitmaps at the system's
// current block size
std::pair<int, int> bm_residency(DevSys* d) {
    const bool bm = d->bm;
    d->bm = false;
    const int s0 = smem_one(*d);
    d->bm = true;
    const int s1 = smem_one(*d);
    d->bm = bm;
    const auto per_sm = [&](int s) { return std::min(reg_blocks(d->nt), (228 * 1024) / (s + kStaticSmem + 1024)); };
    return {per_sm(s0), per_sm(s1)};
}

void pick_bm(DevSys* d, int keep) {
    d->bm = false;
    d->small = false;
    if (!d->dense || !bm_instantiated(d->W, d->nt))
        return;
    // without pruning the bitmaps serve lists of at most 32 candidates (the
    // branch-free reference loop in its own instantiation, search.cu
    // gi_dense_small); TCSE_GI_SMALL=0 keeps the plain loop there
    static const int small = env_int("TCSE_GI_SMALL", 1);
    const bool pruned = env_int("TCSE_GI_PRUNE", d->base_m > 32 ? 1 : 0) != 0;
    const bool small_ok = small && !pruned && d->base_m <= 32 && d->W == 1 && d->nt == 32;
    const int forced = env_int("TCSE_GI_BM", -1);
    if (forced >= 0) {
        d->bm = forced != 0;
    } else {
        if (!pruned && !small_ok)
            return;
        // bitmaps if at least keep / 4 of the resident processes remain
        const auto r = bm_residency(d);
        d->bm = 4 * r.second >= keep * r.first;
    }
    d->small = d->bm && small_ok;
}

// extra_vars: fresh variables a caller-supplied prefix may add beyond the
// search bound.  Every search substitution replaces c >= 2 occurrences and
// the total term count can drop by at most naive (rows never empty), so a
// search creates at most naive/2 fresh variables; an arbitrary replayed
// prefix may use c = 1 pairs, hence the extra allowance.
int prepare(tcse_ctx* ctx, const tcse_system* s, DevSys* d, int extra_vars = 0) {
    int rc = validate_system(s, &d->h);
    if (rc)
        return rc;
    d->h.vcap = d->h.n_x + d->h.naive / 2 + extra_vars + 1;
    choose_launch(ctx, d);
    const int W = d->W;
    const auto masks = pack_masks(d->h, W);
    CU(d->masks.reserve(std::max<size_t>(8, masks.size() * 8)));
    if (!masks.empty())
        CU(cudaMemcpyAsync(d->masks.p, masks.data(), masks.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    CU(d->keys.reserve(size_t(d->h.mcap) * 4));
    CU(d->cnts.reserve(size_t(d->h.mcap) * 2));
    return TCSE_OK;
}

// slot records + seeded mt19937_64 states for `blocks` processes
int reserve_prep(tcse_ctx* ctx, int blocks) {
    const size_t b = size_t(std::max(blocks, 1));
    CU(ctx->slots.reserve(b * sizeof(SlotRec)));
    CU(ctx->rng.reserve(b * kCkpt * 8));
    CU(ctx->perm.reserve(b * 4));
    CU(ctx->hist.reserve(sizeof(int32_t) * kHistStride * kMaxSys * (kMaxSys + 1)));
    return TCSE_OK;
}

int attach_prep(tcse_ctx* ctx, LaunchDesc* L, int block_offset = 0, int group = 0) {
    if (block_offset == 0) {
        const int rc = reserve_prep(ctx, L->total_blocks);
        if (rc)
            return rc;
    }
    L->slots = ctx->slots.as<SlotRec>() + block_offset;
    L->rng = ctx->rng.as<u64>() + size_t(block_offset) * kCkpt;
    // strategy-grouped launch order (search mode; TCSE_ORDER=0 disables)
    static const int order = env_int("TCSE_ORDER", 1);
    if (order && L->sys[0].mode == kModeSearch) {
        L->perm = ctx->perm.as<int32_t>() + block_offset;
        L->hist = ctx->hist.as<int32_t>() + kHistStride * kMaxSys * group;  // one per concurrent launch group
    }
    return TCSE_OK;
}

int check_err(tcse_ctx* ctx) {
    int32_t h[2] = {0, 0};
    CU(cudaMemcpyAsync(h, ctx->err.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (h[0] == TCSE_EREPLAY)
        return fail(TCSE_EREPLAY, "replay_prefix: unreplayable pair at position %d", h[1]);
    if (h[0] == TCSE_ECAPACITY || h[0] == kErrCandOverflow)
        return fail(TCSE_ECAPACITY, "device capacity exceeded (%d)", h[1]);
    if (h[0] != 0)
        return fail(h[0], "device error %d", h[0]);
    return TCSE_OK;
}

SysDesc base_desc(const DevSys& d, int32_t* err) {
    SysDesc sd;
    std::memset(&sd, 0, sizeof sd);
    sd.n_x = d.h.n_x;
    sd.n_e = d.h.n_e;
    sd.naive = d.h.naive;
    sd.words = d.h.w_need;
    sd.coin_words = coin_words_for(d.h);
    sd.gi_dense = d.dense ? 1 : 0;
    sd.gi_bm = d.bm ? 1 : 0;
    // near-best pruning pays once candidate lists are long enough that the
    // O(m^2) scoring outweighs its extra reductions and tie folds: on for
    // systems starting above 32 candidates (laderman-size systems, with
    // frequent exact ties, run the reference loop; sweep
    // scripts/prune_threshold.sh).  TCSE_GI_PRUNE=k forces k (0 = off).
    sd.gi_prune = env_int("TCSE_GI_PRUNE", d.base_m > 32 ? 1 : 0);
    sd.vcap = d.h.vcap;
    sd.mcap = d.h.mcap;
    sd.sub_cap = d.h.naive / 2 + 1;
    sd.base_masks = d.masks.as<u64>();
    sd.forced = -1;
    sd.p_stride = 1;
    sd.stream_comp = -1;
    sd.err = err;
    sd.err_pos = err + 1;
    return sd;
}

// dump the candidate list (or every pair) of replay_prefix(sys, prefix)
int run_dump(tcse_ctx* ctx, DevSys& d, const u32* d_prefix, int n_prefix, int min_count, u32* okeys,
             u16* ocnts, int cap, int* n_out, bool from_base) {
    DBuf dn;
    CU(dn.reserve(4));
    CU(cudaMemsetAsync(ctx->err.p, 0, 8, ctx->stream));
    LaunchDesc L;
    std::memset(&L, 0, sizeof L);
    L.nsys = 1;
    L.total_blocks = 1;
    SysDesc sd = base_desc(d, ctx->err.as<int32_t>());
    sd.mode = kModeDump;
    sd.n_local = 1;
    sd.base_keys = from_base ? d.keys.as<u32>() : nullptr;
    sd.base_cnts = from_base ? d.cnts.as<u16>() : nullptr;
    sd.base_m = from_base ? d.base_m : 0;
    sd.prefix = d_prefix;
    sd.prefix_len = n_prefix;
    sd.dump_min_count = min_count;
    sd.dump_cap = cap;
    sd.dump_keys = okeys;
    sd.dump_cnts = ocnts;
    sd.dump_n = dn.as<int32_t>();
    L.sys[0] = sd;
    std::vector<DevSys*> v{&d};
    int prc = attach_prep(ctx, &L);
    if (prc)
        return prc;
    L.sys[0].gi_dense = d.dense;
    CU(launch_search(L, d.W, d.nt, d.dense, kernel_form(d), smem_one(d), ctx->stream));
    int rc = check_err(ctx);
    if (rc)
        return rc;
    int32_t n = 0;
    CU(cudaMemcpyAsync(&n, dn.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    *n_out = n;
    return TCSE_OK;
}

// base candidate list of a freshly prepared system, computed on the device
int base_candidates(tcse_ctx* ctx, DevSys& d) {
    int n = 0;
    int rc = run_dump(ctx, d, nullptr, 0, 2, d.keys.as<u32>(), d.cnts.as<u16>(), d.h.mcap, &n, false);
    if (rc)
        return rc;
    if (n > d.h.mcap)
        return fail(TCSE_ECAPACITY, "candidate capacity %d < %d", d.h.mcap, n);
    d.base_m = n;
    pick_form(&d);
    return TCSE_OK;
}

// Session layouts are sized for the starting list plus slack instead of the
// worst-case bound (lists rarely grow: a substitution consumes its pair and
// moves the others' occurrences to the fresh variable), e.g. 89 -> 64 KB per
// process on 6x6x6 W (3 processes per SM instead of 2).  A process whose list
// would outgrow the capacity flags kErrCandOverflow before writing; the
// session then re-runs that iteration at full capacity (search_step_begin),
// so results never depend on the slack.  TCSE_MCAP_SLACK=k: capacity m0 + k.
void shrink_capacity(const tcse_ctx* ctx, DevSys* d) {
    const int slack_env = env_int("TCSE_MCAP_SLACK", -1);
    const int slack = slack_env >= 0 ? slack_env : d->base_m / 4 + 64;
    const int eff = std::max(1, d->base_m + slack);
    if (eff >= d->h.mcap)
        return;
    d->mcap_full = d->h.mcap;
    d->h.mcap = eff;
    choose_launch(ctx, d);
    pick_form(d);
}

void restore_capacity(const tcse_ctx* ctx, DevSys* d) {
    if (d->mcap_full == 0)
        return;
    d->h.mcap = d->mcap_full;
    d->mcap_full = 0;
    choose_launch(ctx, d);
    pick_form(d);
}

int upload_pairs(tcse_ctx* ctx, const tcse_pair* pairs, int n, DBuf* buf) {
    std::vector<u32> keys(size_t(std::max(n, 1)), 0u);
    for (int t = 0; t < n; ++t) {
        const tcse_pair& q = pairs[t];
        if (q.i < 1 || q.j <= q.i || q.j > 65535 || q.i > 32767 || (q.rel_sign != 1 && q.rel_sign != -1))
            return fail(TCSE_EREPLAY, "replay_prefix: unreplayable pair at position %d", t);
        keys[size_t(t)] = make_key(q.i, q.j, q.rel_sign < 0);
    }
    CU(buf->reserve(keys.size() * 4));
    CU(cudaMemcpyAsync(buf->p, keys.data(), keys.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
    return TCSE_OK;
}

// validate_config (parallel_search.hpp:117-140), flip mode not supported
int validate_config(const tcse_search_config* c) {
    if (!c)
        return fail(TCSE_EINVAL, "search config: null config");
    if (c->n_processes < 0)
        return fail(TCSE_EINVAL, "search config: n_processes must be >= 0");
    if (c->reinit_fraction < 0.0 || c->reinit_fraction > 1.0)
        return fail(TCSE_EINVAL, "search config: reinit_fraction must be in [0, 1]");
    if (c->patience < 1)
        return fail(TCSE_EINVAL, "search config: patience must be >= 1");
    if (!(c->wall_budget_s >= 0.0))
        return fail(TCSE_EINVAL, "search config: wall_budget_s must be >= 0");
    if (c->forced_strategy < -1 || c->forced_strategy >= TCSE_STRATEGY_COUNT)
        return fail(TCSE_EINVAL, "search config: unknown forced strategy %d", c->forced_strategy);
    if (c->forced_strategy < 0) {
        double total = 0.0;
        for (int k = 0; k < TCSE_STRATEGY_COUNT; ++k) {
            if (c->strategy_weights[k] < 0.0)
                return fail(TCSE_EINVAL, "search config: strategy weights must be >= 0");
            total += c->strategy_weights[k];
        }
        if (total <= 0.0)
            return fail(TCSE_EINVAL, "search config: all strategy weights are zero");
    }
    return TCSE_OK;
}

// pick_mixed_substrategy's weight checks (strategies.hpp:240-250)
int validate_mix(const double* mix) {
    int positive = 0;
    for (int k = 0; k < 4; ++k) {
        if (mix[k] < 0.0)
            return fail(TCSE_EINVAL, "mixed strategy: negative weight");
        positive += mix[k] > 0.0;
    }
    if (positive == 0)
        return fail(TCSE_EINVAL, "mixed strategy: all weights are zero");
    return TCSE_OK;
}



}  // namespace

extern "C" {

const char* tcse_last_error(void) { return g_err.c_str(); }
int32_t tcse_abi_version(void) { return TCSE_ABI_VERSION; }

int32_t tcse_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess)
        return 0;
    return n;
}

void tcse_default_search_config(tcse_search_config* cfg) {
    std::memset(cfg, 0, sizeof *cfg);
    static const double w[7] = {0.0, 4.0, 1.0, 2.0, 8.0, 0.1, 0.01};  // parallel_search.hpp:31-39
    for (int k = 0; k < 7; ++k)
        cfg->strategy_weights[k] = w[k];
    cfg->n_processes = 0;
    cfg->reinit_fraction = 0.40;
    cfg->patience = 10;
    cfg->master_seed = 0;
    cfg->forced_strategy = -1;
    cfg->max_iterations = 0;
    const double mix[4] = {8.0, 4.0, 2.0, 1.0};  // strategies.hpp:52
    for (int k = 0; k < 4; ++k)
        cfg->mix_weights[k] = mix[k];
}

int32_t tcse_naive_cost(const tcse_system* sys) {
    int cost = 0;
    for (int r = 0; r < sys->n_e; ++r) {
        const int t = sys->row_ptr[r + 1] - sys->row_ptr[r];
        if (t > 0)
            cost += t - 1;
    }
    return cost;
}

tcse_ctx* tcse_create(int32_t device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        fail(TCSE_ECUDA, "tcse_create: no CUDA device (%s)", e != cudaSuccess ? cudaGetErrorString(e) : "0 devices");
        return nullptr;
    }
    if (device < 0 || device >= n) {
        fail(TCSE_EINVAL, "tcse_create: device %d out of range (%d devices)", device, n);
        return nullptr;
    }
    e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        fail(TCSE_ECUDA, "tcse_create: %s", cudaGetErrorString(e));
        return nullptr;
    }
    auto* ctx = new tcse_ctx;
    ctx->device = device;
    ctx->nt = env_int("TCSE_NT", 0);  // 0 = by problem size
    if (ctx->nt != 0 && ctx->nt != 32 && ctx->nt != 64 && ctx->nt != 128 && ctx->nt != 256)
        ctx->nt = 0;
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess ||
        ctx->err.reserve(8) != cudaSuccess) {
        fail(TCSE_ECUDA, "tcse_create: stream/event/buffer allocation failed");
        delete ctx;
        return nullptr;
    }
    return ctx;
}

void tcse_destroy(tcse_ctx* ctx) {
    if (!ctx)
        return;
    for (tcse_ctx* c : ctx->sub)
        tcse_destroy(c);
    ctx->sub.clear();
    cudaSetDevice(ctx->device);
    if (ctx->stream)
        cudaStreamSynchronize(ctx->stream);
    if (ctx->comm && ctx->own_comm && nccl().ok)
        nccl().CommDestroy(ctx->comm);
    ctx->comm = nullptr;
    if (ctx->owned_stream)
        cudaStreamDestroy(ctx->owned_stream);
    else if (ctx->stream)
        cudaStreamDestroy(ctx->stream);
    if (ctx->ev0)
        cudaEventDestroy(ctx->ev0);
    if (ctx->ev1)
        cudaEventDestroy(ctx->ev1);
    for (int g = 0; g < kMaxSys; ++g) {
        if (ctx->aux[g])
            cudaStreamDestroy(ctx->aux[g]);
        if (ctx->join[g])
            cudaEventDestroy(ctx->join[g]);
    }
    if (ctx->fork)
        cudaEventDestroy(ctx->fork);
    delete ctx;
}

int tcse_set_stream(tcse_ctx* ctx, void* stream) {
    if (!ctx)
        return fail(TCSE_EINVAL, "tcse_set_stream: null context");
    if (ctx->owned_stream == nullptr)
        ctx->owned_stream = ctx->stream;
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->owned_stream;
    return TCSE_OK;
}

int tcse_set_partition(tcse_ctx* ctx, int32_t rank, int32_t world, tcse_allgather_fn allgather, void* user) {
    if (!ctx || world < 1 || rank < 0 || rank >= world)
        return fail(TCSE_EINVAL, "tcse_set_partition: bad rank %d / world %d", rank, world);
    if (!ctx->sub.empty())
        return fail(TCSE_EINVAL, "tcse_set_partition: a multi-device context owns its partition");
    ctx->rank = rank;
    ctx->world = world;
    ctx->allgather = allgather;
    ctx->ag_user = user;
    return TCSE_OK;
}

int32_t tcse_nccl_available(void) { return nccl().ok ? 1 : 0; }

int tcse_nccl_unique_id(void* id) {
    if (!id)
        return fail(TCSE_EINVAL, "tcse_nccl_unique_id: null buffer");
    const NcclApi& nc = nccl();
    if (!nc.ok)
        return fail(TCSE_ENCCL, "nccl: %s", nc.why);
    ncclUniqueId u;
    const ncclResult_t r = nc.GetUniqueId(&u);
    if (r != ncclSuccess)
        return fail(TCSE_ENCCL, "ncclGetUniqueId: %s", nc.GetErrorString(r));
    std::memcpy(id, &u, sizeof u);
    return TCSE_OK;
}

int tcse_set_nccl(tcse_ctx* ctx, const void* unique_id, int32_t rank, int32_t world) {
    if (!ctx || !unique_id || world < 1 || rank < 0 || rank >= world)
        return fail(TCSE_EINVAL, "tcse_set_nccl: bad rank %d / world %d", rank, world);
    if (!ctx->sub.empty())
        return fail(TCSE_EINVAL, "tcse_set_nccl: a multi-device context owns its communicators");
    const NcclApi& nc = nccl();
    if (!nc.ok)
        return fail(TCSE_ENCCL, "nccl: %s", nc.why);
    CU(cudaSetDevice(ctx->device));
    ncclUniqueId u;
    std::memcpy(&u, unique_id, sizeof u);
    ncclComm_t comm = nullptr;
    const ncclResult_t r = nc.CommInitRank(&comm, world, u, rank);
    if (r != ncclSuccess)
        return fail(TCSE_ENCCL, "ncclCommInitRank: %s", nc.GetErrorString(r));
    if (ctx->comm && ctx->own_comm)
        nc.CommDestroy(ctx->comm);
    ctx->comm = comm;
    ctx->own_comm = true;
    ctx->rank = rank;
    ctx->world = world;
    ctx->allgather = nullptr;
    return TCSE_OK;
}

}  // extern "C"

namespace {

// In-process all-gather between the rank threads of one context: the
// transport of a shared-device context, which NCCL refuses (one rank per
// GPU).  Only for TCSE_SHARED_DEVICES=1 test runs of the multi-device
// orchestration on a single GPU; payloads go through host memory.
struct LocalGather {
    int world;
    std::mutex mu;
    std::condition_variable cv;
    std::vector<std::vector<char>> slot;
    int arrived = 0, phase = 0;
    explicit LocalGather(int w) : world(w), slot(size_t(w)) {}
    void barrier(std::unique_lock<std::mutex>& lk) {
        const int ph = phase;
        if (++arrived == world) {
            arrived = 0;
            ++phase;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return phase != ph; });
        }
    }
};

struct LocalRank {
    LocalGather* g;
    int rank;
};

int local_allgather(const void* send, void* recv, size_t bytes, void* user) {
    auto* R = static_cast<LocalRank*>(user);
    LocalGather& G = *R->g;
    std::unique_lock<std::mutex> lk(G.mu);
    G.slot[size_t(R->rank)].assign(static_cast<const char*>(send), static_cast<const char*>(send) + bytes);
    G.barrier(lk);
    for (int r = 0; r < G.world; ++r)
        std::memcpy(static_cast<char*>(recv) + size_t(r) * bytes, G.slot[size_t(r)].data(), bytes);
    G.barrier(lk);  // every rank has read before the next iteration overwrites
    return 0;
}

struct LocalGroup {
    LocalGather g;
    std::vector<LocalRank> ranks;
    explicit LocalGroup(int w) : g(w), ranks(size_t(w)) {}
};

}  // namespace

extern "C" {

tcse_ctx* tcse_create_devices(const int32_t* devices, int32_t n_devices) {
    if (!devices || n_devices < 1) {
        fail(TCSE_EINVAL, "tcse_create_devices: need at least one device");
        return nullptr;
    }
    if (n_devices == 1)
        return tcse_create(devices[0]);
    bool shared = false;
    for (int a = 0; a < n_devices; ++a)
        for (int b = a + 1; b < n_devices; ++b)
            shared = shared || devices[a] == devices[b];
    if (shared) {
        if (env_int("TCSE_SHARED_DEVICES", 0) != 1) {
            fail(TCSE_EINVAL, "tcse_create_devices: a device is listed twice (one rank per GPU)");
            return nullptr;
        }
        // test transport: rank threads exchange through host memory
        auto* top = tcse_create(devices[0]);
        if (!top)
            return nullptr;
        auto grp = std::make_shared<LocalGroup>(n_devices);
        top->local_gather = grp;
        for (int k = 0; k < n_devices; ++k) {
            tcse_ctx* c = tcse_create(devices[k]);
            if (!c) {
                tcse_destroy(top);
                return nullptr;
            }
            grp->ranks[size_t(k)] = LocalRank{&grp->g, k};
            c->rank = k;
            c->world = n_devices;
            c->allgather = local_allgather;
            c->ag_user = &grp->ranks[size_t(k)];
            top->sub.push_back(c);
        }
        return top;
    }
    const NcclApi& nc = nccl();
    if (!nc.ok) {
        fail(TCSE_ENCCL, "nccl: %s", nc.why);
        return nullptr;
    }
    auto* top = tcse_create(devices[0]);
    if (!top)
        return nullptr;
    std::vector<ncclComm_t> comms(size_t(n_devices), nullptr);
    std::vector<int> devs(devices, devices + n_devices);
    const ncclResult_t r = nc.CommInitAll(comms.data(), n_devices, devs.data());
    if (r != ncclSuccess) {
        fail(TCSE_ENCCL, "ncclCommInitAll: %s", nc.GetErrorString(r));
        tcse_destroy(top);
        return nullptr;
    }
    for (int k = 0; k < n_devices; ++k) {
        tcse_ctx* c = tcse_create(devices[k]);
        if (!c) {
            for (int j = k; j < n_devices; ++j)
                nc.CommDestroy(comms[size_t(j)]);
            tcse_destroy(top);
            return nullptr;
        }
        c->comm = comms[size_t(k)];
        c->own_comm = true;
        c->rank = k;
        c->world = n_devices;
        top->sub.push_back(c);
    }
    // the container itself is a single-device context on devices[0]: calls
    // other than tcse_optimize_system(s) (run_cse, count_pairs, flips, checks)
    // run there
    return top;
}

int32_t tcse_context_devices(const tcse_ctx* ctx) { return ctx ? int32_t(std::max<size_t>(1, ctx->sub.size())) : 0; }

int tcse_count_pairs(tcse_ctx* ctx, const tcse_system* sys, const tcse_pair* prefix, int32_t n_prefix,
                     int32_t min_count, tcse_pair_count* out, int32_t cap, int32_t* n_out) {
    if (!ctx || min_count < 1 || cap < 0 || n_prefix < 0)
        return fail(TCSE_EINVAL, "tcse_count_pairs: bad argument");
    CU(cudaSetDevice(ctx->device));
    DevSys d;
    HostSys probe;
    int rc = validate_system(sys, &probe);
    if (rc)
        return rc;
    rc = prepare(ctx, sys, &d, n_prefix);
    if (rc)
        return rc;
    rc = base_candidates(ctx, d);
    if (rc)
        return rc;
    DBuf dpre;
    rc = upload_pairs(ctx, prefix, n_prefix, &dpre);
    if (rc)
        return rc;
    // every pair of the state fits in (vcap^2) entries; candidates in mcap
    const size_t dcap = min_count >= 2 ? size_t(d.h.mcap)
                                       : std::max<size_t>(1, size_t(d.h.vcap) * size_t(d.h.vcap));
    DBuf dk, dc;
    CU(dk.reserve(dcap * 4));
    CU(dc.reserve(dcap * 2));
    int n = 0;
    rc = run_dump(ctx, d, dpre.as<u32>(), n_prefix, min_count, dk.as<u32>(), dc.as<u16>(), int(dcap), &n, true);
    if (rc)
        return rc;
    const int ncopy = std::min(n, int(dcap));
    std::vector<u32> hk(size_t(std::max(ncopy, 1)));
    std::vector<u16> hc(size_t(std::max(ncopy, 1)));
    if (ncopy > 0) {
        CU(cudaMemcpyAsync(hk.data(), dk.p, size_t(ncopy) * 4, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaMemcpyAsync(hc.data(), dc.p, size_t(ncopy) * 2, cudaMemcpyDeviceToHost, ctx->stream));
    }
    CU(cudaStreamSynchronize(ctx->stream));
    for (int t = 0; t < ncopy && t < cap; ++t) {
        out[t].pair = key_pair(hk[size_t(t)]);
        out[t].count = hc[size_t(t)];
    }
    *n_out = n;
    if (n > cap)
        return fail(TCSE_ECAPACITY, "count_pairs: %d pairs exceed capacity %d", n, cap);
    return TCSE_OK;
}

int tcse_run_cse(tcse_ctx* ctx, const tcse_system* sys, const tcse_pair* prefix, int32_t n_prefix,
                 const tcse_process_config* cfgs, int32_t n, tcse_record* out, uint64_t* trace,
                 int32_t trace_stride, tcse_stats* stats) {
    if (!ctx || n < 0 || n_prefix < 0 || (n > 0 && (!cfgs || !out)))
        return fail(TCSE_EINVAL, "tcse_run_cse: bad argument");
    if (n == 0)
        return TCSE_OK;
    for (int b = 0; b < n; ++b) {
        if (cfgs[b].strategy < 0 || cfgs[b].strategy >= TCSE_STRATEGY_COUNT)
            return fail(TCSE_EINVAL, "select_pair: unknown strategy");
        if (cfgs[b].strategy == TCSE_MIXED) {
            int rc = validate_mix(cfgs[b].mix_weights);
            if (rc)
                return rc;
        }
    }
    const auto t0 = std::chrono::steady_clock::now();
    CU(cudaSetDevice(ctx->device));
    DevSys d;
    HostSys probe;
    int rc = validate_system(sys, &probe);
    if (rc)
        return rc;
    rc = prepare(ctx, sys, &d, n_prefix);
    if (rc)
        return rc;
    rc = base_candidates(ctx, d);
    if (rc)
        return rc;
    DBuf dpre, dcfg, dcost, dlen, down, dstrat, dseed, dwops, dsubs, dtrace;
    rc = upload_pairs(ctx, prefix, n_prefix, &dpre);
    if (rc)
        return rc;
    const int sub_cap = d.h.naive / 2 + 1;
    CU(dcfg.reserve(sizeof(tcse_process_config) * size_t(n)));
    CU(cudaMemcpyAsync(dcfg.p, cfgs, sizeof(tcse_process_config) * size_t(n), cudaMemcpyHostToDevice, ctx->stream));
    CU(dcost.reserve(4 * size_t(n)));
    CU(dlen.reserve(4 * size_t(n)));
    CU(down.reserve(4 * size_t(n)));
    CU(dstrat.reserve(4 * size_t(n)));
    CU(dseed.reserve(8 * size_t(n)));
    CU(dwops.reserve(8 * size_t(n)));
    CU(dsubs.reserve(4 * size_t(n) * size_t(sub_cap)));
    if (trace && trace_stride > 0)
        CU(dtrace.reserve(8 * size_t(n) * size_t(trace_stride)));
    CU(cudaMemsetAsync(ctx->err.p, 0, 8, ctx->stream));

    LaunchDesc L;
    std::memset(&L, 0, sizeof L);
    L.nsys = 1;
    L.total_blocks = n;
    SysDesc sd = base_desc(d, ctx->err.as<int32_t>());
    sd.mode = kModeRun;
    sd.base_keys = d.keys.as<u32>();
    sd.base_cnts = d.cnts.as<u16>();
    sd.base_m = d.base_m;
    sd.n_local = n;
    sd.cfgs = dcfg.as<tcse_process_config>();
    sd.prefix = dpre.as<u32>();
    sd.prefix_len = n_prefix;
    sd.out_cost = dcost.as<int32_t>();
    sd.out_len = dlen.as<int32_t>();
    sd.out_own = down.as<int32_t>();
    sd.out_strategy = dstrat.as<int32_t>();
    sd.out_seed = dseed.as<u64>();
    sd.out_wops = dwops.as<u64>();
    sd.out_subs = dsubs.as<u32>();
    sd.trace = (trace && trace_stride > 0) ? dtrace.as<u64>() : nullptr;
    sd.trace_stride = trace_stride;
    L.sys[0] = sd;
    std::vector<DevSys*> v{&d};
    rc = attach_prep(ctx, &L);
    if (rc)
        return rc;
    CU(cudaEventRecord(ctx->ev0, ctx->stream));
    L.sys[0].gi_dense = d.dense;
    CU(launch_search(L, d.W, d.nt, d.dense, kernel_form(d), smem_one(d), ctx->stream));
    CU(cudaEventRecord(ctx->ev1, ctx->stream));
    rc = check_err(ctx);
    if (rc)
        return rc;
    const size_t nn = size_t(n);
    std::vector<int32_t> hcost(nn), hlen(nn), hown(nn), hstrat(nn);
    std::vector<u64> hseed((size_t)n), hwops((size_t)n);
    std::vector<u32> hsubs(size_t(n) * size_t(sub_cap));
    CU(cudaMemcpyAsync(hcost.data(), dcost.p, 4 * size_t(n), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(hlen.data(), dlen.p, 4 * size_t(n), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(hown.data(), down.p, 4 * size_t(n), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(hstrat.data(), dstrat.p, 4 * size_t(n), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(hseed.data(), dseed.p, 8 * size_t(n), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(hwops.data(), dwops.p, 8 * size_t(n), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(hsubs.data(), dsubs.p, 4 * size_t(n) * size_t(sub_cap), cudaMemcpyDeviceToHost, ctx->stream));
    if (sd.trace)
        CU(cudaMemcpyAsync(trace, dtrace.p, 8 * size_t(n) * size_t(trace_stride), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    uint64_t steps = 0, wops = 0;
    for (int b = 0; b < n; ++b) {
        tcse_record& r = out[b];
        wops += hwops[size_t(b)];
        if (hlen[size_t(b)] > r.cap)
            return fail(TCSE_ECAPACITY, "run_cse: record %d needs %d entries, capacity %d", b, hlen[size_t(b)], r.cap);
        for (int t = 0; t < hlen[size_t(b)]; ++t)
            r.subs[t] = key_pair(hsubs[size_t(b) * size_t(sub_cap) + size_t(t)]);
        r.n_subs = hlen[size_t(b)];
        r.cost = hcost[size_t(b)];
        r.strategy = hstrat[size_t(b)];
        r.seed = hseed[size_t(b)];
        steps += uint64_t(hown[size_t(b)]);
    }
    if (stats) {
        std::memset(stats, 0, sizeof *stats);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        stats->kernel_ms = ms;
        stats->steps = steps;
        stats->wops = wops;
        stats->processes = uint64_t(n);
        stats->launches = 1;
        stats->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    return TCSE_OK;
}

}  // extern "C"

#include "session.inc"

extern "C" {

// replay_prefix + total_cost + expand_and_verify (linear_system.hpp:193-258)
int tcse_verify_record(const tcse_system* sys, const tcse_pair* subs, int32_t n_subs, int32_t* cost_out) {
    HostSys h;
    int rc = validate_system(sys, &h);
    if (rc && rc != TCSE_ECAPACITY)
        return rc;
    const int nx = sys->n_x;
    // rows as dense signed coefficient maps over current variables
    std::vector<std::vector<int>> rows = h.rows;
    std::vector<tcse_pair> defs;
    for (int t = 0; t < n_subs; ++t) {
        const tcse_pair q = subs[t];
        const int k = nx + int(defs.size()) + 1;
        const int first = q.i, second = q.rel_sign * q.j;
        int replaced = 0;
        if (q.i >= 1 && q.j > q.i && q.j < k && (q.rel_sign == 1 || q.rel_sign == -1)) {
            for (auto& row : rows) {
                auto has = [&](int x) { return std::find(row.begin(), row.end(), x) != row.end(); };
                auto erase = [&](int x) { row.erase(std::find(row.begin(), row.end(), x)); };
                if (has(first) && has(second)) {
                    erase(first);
                    erase(second);
                    row.push_back(k);
                    ++replaced;
                } else if (has(-first) && has(-second)) {
                    erase(-first);
                    erase(-second);
                    row.push_back(-k);
                    ++replaced;
                }
            }
        }
        if (replaced == 0)
            return fail(TCSE_EREPLAY, "replay_prefix: unreplayable pair at position %d", t);
        defs.push_back(q);
    }
    int cost = int(defs.size());
    for (const auto& row : rows)
        if (!row.empty())
            cost += int(row.size()) - 1;
    *cost_out = cost;
    // expansion over base variables
    std::vector<std::vector<long long>> ex(size_t(nx) + defs.size() + 1, std::vector<long long>(size_t(nx) + 1, 0));
    for (int v = 1; v <= nx; ++v)
        ex[size_t(v)][size_t(v)] = 1;
    for (size_t t = 0; t < defs.size(); ++t) {
        const size_t id = size_t(nx) + t + 1;
        for (int b = 1; b <= nx; ++b)
            ex[id][size_t(b)] = ex[size_t(defs[t].i)][size_t(b)] + defs[t].rel_sign * ex[size_t(defs[t].j)][size_t(b)];
    }
    for (int r = 0; r < sys->n_e; ++r) {
        std::vector<long long> acc(size_t(nx) + 1, 0);
        for (int term : rows[size_t(r)])
            for (int b = 1; b <= nx; ++b)
                acc[size_t(b)] += (term > 0 ? 1 : -1) * ex[size_t(std::abs(term))][size_t(b)];
        int nonzero = 0;
        for (int b = 1; b <= nx; ++b) {
            if (acc[size_t(b)] == 0)
                continue;
            ++nonzero;
            if (acc[size_t(b)] != 1 && acc[size_t(b)] != -1)
                return 0;
            const int want = acc[size_t(b)] > 0 ? b : -b;
            if (std::find(h.rows[size_t(r)].begin(), h.rows[size_t(r)].end(), want) == h.rows[size_t(r)].end())
                return 0;
        }
        if (nonzero != int(h.rows[size_t(r)].size()))
            return 0;
    }
    return 1;
}

}  // extern "C"

#include "flip_mode.inc"
