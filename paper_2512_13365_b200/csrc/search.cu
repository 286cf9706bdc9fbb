// search.cu — sm_100a kernels of the ternary-CSE search hot path.
//
// K1 search_kernel<W, NT>: ONE CSE PROCESS PER THREAD BLOCK.  A block owns its
// expression set as per-variable occurrence bitsets in shared memory (bit r of
// P[v] / N[v] = expression r holds +x_v / -x_v; W 64-bit words cover up to 64W
// expressions), keeps the substitutable-pair list (frequency >= 2) sorted in
// canonical order, and loops select -> substitute -> incremental recount until
// no pair repeats — run_cse (cse_engine.hpp:29-43).  All seven selection
// strategies (strategies.hpp:61-285) run on the device and consume the
// process's std::mt19937_64 stream exactly like the reference, so records are
// bit-identical to the reference's for every strategy, not only greedy.
//
// K2 reduce_kernel: the iteration barrier of optimize_system
// (parallel_search.hpp:255-266, 149-163) on the device: argmin over
// (cost, process id), incumbent update with a record copy in HBM, the
// substitution-step sum, and the worst-fraction reinit set for the next
// iteration (pick_reinit) by a cost histogram + ordered scan.
//
// Exactness notes:
//  * pair frequency = popc(P_i & P_j) + popc(N_i & N_j) (rel +) or
//    popc(P_i & N_j) + popc(N_i & P_j) (rel -): a pair occurs at most once per
//    expression (linear_system.hpp:129-131), so this equals count_pairs.
//  * after substituting q = (i, j, s) -> k only pairs touching {i, j, k} change
//    (counts touching i or j can only drop; pairs with k are new), so the
//    candidate list is updated incrementally and merged in canonical order.
//  * double arithmetic uses explicit __dadd_rn/__dmul_rn (no FMA contraction),
//    matching the reference built for baseline x86-64.
//  * Greedy-Intersections (score_intersections_from, strategies.hpp:136-153)
//    is a sequential double sum per candidate q over all other candidates.
//    It is evaluated EXACTLY in O(deg q) instead of O(m): the candidates
//    between two consecutive neighbours of q contribute integers c-1, and a
//    run of integer additions to a double is exact except where the running
//    sum crosses a binade, which is located by binary search in a prefix sum
//    and rounded once — the same value the reference's loop produces.
//
// Shared memory is one dynamic buffer (g_smem) carved per system; every
// access goes through g_smem + offset so it compiles to LDS/STS.
#include <cuda_runtime.h>

#include "launch.h"

namespace tcse {

#define FULLMASK 0xffffffffu

extern __shared__ __align__(16) unsigned char g_smem[];

// ------------------------------------------------------------------ keys

__device__ __forceinline__ int key_i(u32 k) { return int(k >> 17); }
__device__ __forceinline__ int key_j(u32 k) { return int((k >> 1) & 0xffffu); }
__device__ __forceinline__ int key_neg(u32 k) { return int(k & 1u); }
__device__ __forceinline__ u32 make_key(int i, int j, int neg) {
    return (u32(i) << 17) | (u32(j) << 1) | u32(neg);
}

// ------------------------------------------------------------------- rng

constexpr u64 kMtUM = 0xffffffff80000000ULL;
constexpr u64 kMtLM = 0x7fffffffULL;
constexpr u64 kMtA = 0xb5026f5aa96619e9ULL;
constexpr u64 kMtF = 6364136223846793005ULL;
// top bit of the tempered output = parity of these raw state bits
#ifndef TCSE_FUSED_TWIST_MIN
#define TCSE_FUSED_TWIST_MIN 128  // block sizes whose coin generations run register-resident (mt_coin_run)
#endif
#ifndef TCSE_COLD_MIN
#define TCSE_COLD_MIN 64  // block sizes keeping cold per-process values in shared memory
#endif
#ifndef TCSE_ONLY_GI
#define TCSE_ONLY_GI 0
#endif
#ifndef TCSE_GI_BALANCE
#define TCSE_GI_BALANCE 0  // 1: work-balanced contiguous candidate ranges in the bitmap gi pass
#endif
#ifndef TCSE_SMALL_TWIST_COINS
#define TCSE_SMALL_TWIST_COINS 0  // 1: smaller blocks extract coins inside the smem twist (-6% on A/B)
#endif
constexpr u64 kCoinMask = 0x8080000004000200ULL;

// coin of raw state word x: parity of x & kCoinMask (one POPC: the two
// halves' masked bits folded by XOR first)
__device__ __forceinline__ u32 coin_bit(u64 x) {
    return u32(__popc((u32(x >> 32) & u32(kCoinMask >> 32)) ^ (u32(x) & u32(kCoinMask)))) & 1u;
}

__device__ __forceinline__ u64 mt_temper(u64 z) {
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71d67fffeda60000ULL;
    z ^= (z << 37) & 0xfff7eee000000000ULL;
    z ^= (z >> 43);
    return z;
}

__device__ __forceinline__ u64 mt_mix(u64 a, u64 b, u64 far) {
    const u64 y = (a & kMtUM) | (b & kMtLM);
    return far ^ (y >> 1) ^ ((y & 1ULL) ? kMtA : 0ULL);
}

// splitmix64 / mix_seed (rng.hpp:8-23)
__device__ __forceinline__ u64 splitmix64(u64 x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

// generate_canonical<double,53>(mt19937_64): double(x) / 2^64, below 1
__device__ __forceinline__ double canonical(u64 x) {
    double r = __dmul_rn(__ull2double_rn(x), 0x1p-64);
    return r >= 1.0 ? 0x1.fffffffffffffp-1 : r;
}

// uniform_real_distribution<double>(a, b): canonical * (b - a) + a
__device__ __forceinline__ double uniform_real(u64 x, double a, double b) {
    return __dadd_rn(__dmul_rn(canonical(x), __dsub_rn(b, a)), a);
}

// ---------------------------------------------------------- smem layout

__shared__ Lay lay;

// fixed-size per-process scratch at link-time addresses (static shared
// memory, sized for the widest block): the process's mt19937_64 state, the
// double-buffered block-reduction slots, the broadcast words.  Constant
// addresses: no layout offset loaded from shared memory at each use.
__shared__ u64 g_mt[312];
__shared__ u32 g_red[2 * (8 + 2)];
__shared__ double g_reds[2 * 8];
__shared__ int g_redi[2 * 8];
__shared__ u32 g_bcast[4];

#if defined(TCSE_GI_STATS) || defined(TCSE_SNAP_STATS)
// debug build only: gi path counters (approx steps, lone picks, folds,
// overflow fallbacks, reference-loop steps, sum of m, multi-survivor steps)
__device__ unsigned long long g_gi_stats[8];
#define DBG_STAT(k, v) do { if (threadIdx.x == 0) atomicAdd(&g_gi_stats[k], (unsigned long long)(v)); } while (0)
#endif
#ifdef TCSE_GI_STATS
#define GI_STAT(k, v) DBG_STAT(k, v)
#else
#define GI_STAT(k, v) do { } while (0)
#endif
#ifdef TCSE_SNAP_STATS  // snapshot use: reinit processes, full hits, misses, sum of prefixes, steps replayed anyway
#define SNAP_STAT(k, v) DBG_STAT(k, v)
#else
#define SNAP_STAT(k, v) do { } while (0)
#endif

__device__ __forceinline__ double __int_as_double_lo(int v) { return __hiloint2double(0, v); }
__device__ __forceinline__ int __double_lo_as_int(double d) { return __double2loint(d); }

__device__ __forceinline__ u64 globaltimer() {
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// the masks open the carve (carve(): offset 0), so their base needs no
// load of the layout from shared memory
__device__ __forceinline__ u64* mask_base() { return reinterpret_cast<u64*>(g_smem); }

template <typename T>
__device__ __forceinline__ T* sp(u32 off) {
    return reinterpret_cast<T*>(g_smem + off);
}

// ------------------------------------------------------ block primitives
//
// Reductions end right after their single read phase; callers alternate
// between two scratch buffers (St::rsel), so a buffer is reused only after
// every thread has passed the next primitive's barrier.

__device__ __forceinline__ u32 warp_incl_scan(u32 v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(FULLMASK, v, o);
        if (lane >= o)
            v += t;
    }
    return v;
}

template <int NT>
__device__ __forceinline__ u32 block_scan(u32 v, u32* red, u32* total) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const u32 inc = warp_incl_scan(v, lane);
    if (NW == 1) {
        *total = __shfl_sync(FULLMASK, inc, 31);
        return inc - v;
    }
    // one barrier: every thread adds the (at most 8) warp totals itself
    if (lane == 31)
        red[warp] = inc;
    __syncthreads();
    u32 pre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const u32 x = red[w];
        tot += x;
        pre += w < warp ? x : 0u;
    }
    *total = tot;
    return pre + inc - v;
}

// out of line (one copy per kernel instead of one per call site): low 32
// bits the exclusive prefix, high 32 bits the block total
template <int NT>
__device__ __noinline__ u64 block_scan_ool(u32 v, u32* red) {
    u32 total;
    const u32 ex = block_scan<NT>(v, red, &total);
    return (u64(total) << 32) | ex;
}

template <int NT>
__device__ __forceinline__ u32 block_max(u32 v, u32* red) {
    constexpr int NW = NT / 32;
    v = __reduce_max_sync(FULLMASK, v);
    if (NW == 1)
        return v;
    if ((threadIdx.x & 31) == 0)
        red[threadIdx.x >> 5] = v;
    __syncthreads();
    u32 r = red[0];
#pragma unroll
    for (int w = 1; w < NW; ++w)
        r = max(r, red[w]);
    return r;
}

template <int NT>
__device__ __forceinline__ u32 block_sum(u32 v, u32* red) {
    constexpr int NW = NT / 32;
    v = __reduce_add_sync(FULLMASK, v);
    if (NW == 1)
        return v;
    if ((threadIdx.x & 31) == 0)
        red[threadIdx.x >> 5] = v;
    __syncthreads();
    u32 r = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w)
        r += red[w];
    return r;
}

// first maximum of (score, index): larger score wins, ties to the smaller
// index (the reference's strict-> scan); threads without a candidate carry
// (-inf, 0x7fffffff), so any real score beats them (scores can be negative
// for user alpha/beta)
template <int NT>
__device__ __forceinline__ int block_argmax_double(double s, int idx, double* reds, int* redi) {
    constexpr int NW = NT / 32;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double s2 = __shfl_down_sync(FULLMASK, s, o);
        const int i2 = __shfl_down_sync(FULLMASK, idx, o);
        if (s2 > s || (s2 == s && i2 < idx)) {
            s = s2;
            idx = i2;
        }
    }
    if (NW == 1)
        return __shfl_sync(FULLMASK, idx, 0);
    if ((threadIdx.x & 31) == 0) {
        reds[threadIdx.x >> 5] = s;
        redi[threadIdx.x >> 5] = idx;
    }
    __syncthreads();
    double bs = reds[0];
    int bi = redi[0];
#pragma unroll
    for (int w = 1; w < NW; ++w)
        if (reds[w] > bs || (reds[w] == bs && redi[w] < bi)) {
            bs = reds[w];
            bi = redi[w];
        }
    return bi;
}

// ------------------------------------------------- cold helpers (no inline)

// mt19937_64 seeding (one thread, any destination)
__device__ __noinline__ void mt_seed(u64* mt, u64 s) {
    u64 x = s;
    mt[0] = x;
#pragma unroll 1
    for (u32 i = 1; i < 312; ++i) {
        x = kMtF * (x ^ (x >> 62)) + i;
        mt[i] = x;
    }
}

// the same seeding straight into the process's shared-memory state (one
// thread; LDS/STS addressing)
__device__ __noinline__ void mt_seed_smem(u64 s) {
    u64* mt = g_mt;
    u64 x = s;
    mt[0] = x;
#pragma unroll 4
    for (u32 i = 1; i < 312; ++i) {
        x = kMtF * (x ^ (x >> 62)) + i;
        mt[i] = x;
    }
}

// first output of mt19937_64(s) without storing the state (registers only)
__device__ __noinline__ u64 mt_first_output(u64 s) {
    u64 x = s;
    const u64 x0 = x;
    x = kMtF * (x ^ (x >> 62)) + 1;
    const u64 x1 = x;
#pragma unroll 4
    for (u32 i = 2; i <= 156; ++i)
        x = kMtF * (x ^ (x >> 62)) + i;
    return mt_temper(mt_mix(x0, x1, x));
}

// the process's stream seed: the slot seed, or mix_seed{slot.seed, comp} in
// flip mode (parallel_search.hpp:441)
__device__ __forceinline__ u64 stream_seed(const SysDesc& sd, u64 seed) {
    if (sd.stream_comp >= 0) {
        seed = splitmix64(0x5851f42d4c957f2dULL ^ seed);
        seed = splitmix64(seed ^ u64(sd.stream_comp));
    }
    return seed;
}

// cooperative twist of the 312-word state (block-uniform call), two
// barriers: thread i owns new[i] = mix(old[i], old[i+1], old[i+156]) and
// new[156+i] = mix(old[156+i], old[157+i], new[i]); the one cross-thread
// input, new[0] for new[311], is recomputed from old words by its owner.
// COINS: also emit the generation's first n outputs as coin bits (tempered
// top bit = parity of raw bits kCoinMask) at coin positions pos0 + e.
template <int NT, bool COINS>
__device__ __noinline__ void mt_twist_impl(u32* coin, u32 pos0, u32 n) {
    constexpr int R = (156 + NT - 1) / NT;
    u64* mt = g_mt;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    u64 lo[R], hi[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = tid + r * NT;
        if (i < 156) {
            const u64 o156 = mt[i + 156];
            lo[r] = mt_mix(mt[i], mt[i + 1], o156);
            const u64 nxt = i < 155 ? mt[i + 157] : mt_mix(mt[0], mt[1], mt[156]);  // old[312] := new[0]
            hi[r] = mt_mix(o156, nxt, lo[r]);
        }
    }
    if (COINS) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int i = tid + r * NT;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const int e = i + half * 156;
                const u32 bit = (i < 156 && u32(e) < n) ? coin_bit(half ? hi[r] : lo[r]) : 0u;
                const u32 ball = __ballot_sync(FULLMASK, bit);
                if (lane == 0 && ball) {
                    const u32 pos = pos0 + u32(e);
                    const u32 w0 = pos >> 5, sh = pos & 31;
                    atomicOr(&coin[w0], ball << sh);
                    if (sh)
                        atomicOr(&coin[w0 + 1], ball >> (32 - sh));
                }
            }
        }
    }
    __syncthreads();  // every old word read
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = tid + r * NT;
        if (i < 156) {
            mt[i] = lo[r];
            mt[i + 156] = hi[r];
        }
    }
    __syncthreads();  // new state visible
}

// small blocks (NT <= 64: R = 3..5 words per thread, one or two warps) keep
// the register-light form: each phase read, barrier, write, barrier
template <int NT>
__device__ __noinline__ void mt_twist_small() {
    constexpr int R = (156 + NT - 1) / NT;
    u64* mt = g_mt;
    const int tid = threadIdx.x;
    u64 v[R];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = tid + r * NT;
        if (i < 156)
            v[r] = mt_mix(mt[i], mt[i + 1], mt[i + 156]);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = tid + r * NT;
        if (i < 156)
            mt[i] = v[r];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = 156 + tid + r * NT;
        if (i < 312)
            v[r] = mt_mix(mt[i], mt[i == 311 ? 0 : i + 1], mt[i - 156]);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = 156 + tid + r * NT;
        if (i < 312)
            mt[i] = v[r];
    }
    __syncthreads();
}

// The same twist that also emits the new generation's first n outputs as
// coin bits at coin positions pos0 + e (each warp's 32 consecutive elements
// by one ballot, straight from the registers the twist computed them in: no
// second pass over the state in shared memory)
__device__ __forceinline__ void coin_ballot(u32* coin, u32 pos0, int e, u32 n, u64 x, int lane) {
    const u32 bit = u32(e) < n ? coin_bit(x) : 0u;
    const u32 ball = __ballot_sync(FULLMASK, bit);
    if (lane == 0 && ball) {
        const u32 pos = pos0 + u32(e - lane);
        const u32 w0 = pos >> 5, sh = pos & 31;
        atomicOr(&coin[w0], ball << sh);
        if (sh)
            atomicOr(&coin[w0 + 1], ball >> (32 - sh));
    }
}

template <int NT>
__device__ __noinline__ void mt_twist_small_coins(u32* coin, u32 pos0, u32 n) {
    constexpr int R = (156 + NT - 1) / NT;
    u64* mt = g_mt;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    u64 v[R];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = tid + r * NT;
        v[r] = i < 156 ? mt_mix(mt[i], mt[i + 1], mt[i + 156]) : 0ULL;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = tid + r * NT;
        if (i < 156)
            mt[i] = v[r];
        if (r * NT < 156)  // warp-uniform: the warp's 32 elements exist in part
            coin_ballot(coin, pos0, i, i < 156 ? n : 0u, v[r], lane);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = 156 + tid + r * NT;
        v[r] = i < 312 ? mt_mix(mt[i], mt[i == 311 ? 0 : i + 1], mt[i - 156]) : 0ULL;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = 156 + tid + r * NT;
        if (i < 312)
            mt[i] = v[r];
        if (r * NT < 156)
            coin_ballot(coin, pos0, i, i < 312 ? n : 0u, v[r], lane);
    }
    __syncthreads();
}

// Coins from consecutive fresh mt19937_64 generations with the state held in
// registers (precondition: every output of the current generation consumed).
// Element i < 156 of the state is the pair (lo = mt[i], hi = mt[i + 156]),
// in lane i % 32 of group i / 32 (groups round-robin over the warps).  One
// twist: new lo[i] = mix(lo[i], lo[i+1], hi[i]), new hi[i] = mix(hi[i],
// hi[i+1], new lo[i]), with old[312] := new[0] for i = 155 — neighbours come
// by shuffle within a group and from the previous twist's published group
// boundaries (double-buffered) across groups, so a generation costs one
// barrier (none for one-warp blocks) instead of the smem twist's two to five.
// Output e of generation t is coin pos0 + 312 t + e (tempered top bit =
// parity of raw bits {63, 55, 26, 9}).  Writes the last generation back to
// smem and returns how many of its outputs were taken.
template <int NT>
__device__ __noinline__ u32 mt_coin_run(u32* coin, u32 pos0, u32 nbits) {
    constexpr int NW = NT / 32;
    constexpr int RG = (5 + NW - 1) / NW;  // groups per warp
    __shared__ u64 bnd[2][12];             // per group (lo, hi) of lane 0, + lo of element 1
    u64* mt = g_mt;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    u64 lo[RG], hi[RG];
#pragma unroll
    for (int r = 0; r < RG; ++r) {
        const int g = warp + r * NW;
        const int i = 32 * g + lane;
        lo[r] = 0ULL;
        hi[r] = 0ULL;
        if (g < 5 && i < 156) {
            lo[r] = mt[i];
            hi[r] = mt[i + 156];
            if (lane == 0) {
                bnd[0][2 * g] = lo[r];
                bnd[0][2 * g + 1] = hi[r];
            }
            if (i == 1)
                bnd[0][10] = lo[r];
        }
    }
    if (NW > 1)
        __syncthreads();
    else
        __syncwarp();
    const u32 T = (nbits + 311) / 312;
    u32 n_t = 0;
#pragma unroll 1
    for (u32 t = 0; t < T; ++t) {
        const int b = int(t & 1u);
        n_t = min(312u, nbits - 312u * t);
        const u32 base = pos0 + 312u * t;
#pragma unroll
        for (int r = 0; r < RG; ++r) {
            const int g = warp + r * NW;
            if (g >= 5)  // warp-uniform
                continue;
            const int i = 32 * g + lane;
            u64 nlo = __shfl_down_sync(FULLMASK, lo[r], 1);
            u64 nhi = __shfl_down_sync(FULLMASK, hi[r], 1);
            if (lane == 31 && g < 4) {
                nlo = bnd[b][2 * g + 2];
                nhi = bnd[b][2 * g + 3];
            }
            if (i == 155) {
                nlo = bnd[b][1];                                     // old[156]
                nhi = mt_mix(bnd[b][0], bnd[b][10], bnd[b][1]);      // old[312] := new[0]
            }
            const u64 l2 = mt_mix(lo[r], nlo, hi[r]);
            const u64 h2 = mt_mix(hi[r], nhi, l2);
            lo[r] = l2;
            hi[r] = h2;
            const bool ok = i < 156;
            const u32 blo = (ok && u32(i) < n_t) ? coin_bit(l2) : 0u;
            const u32 bhi = (ok && u32(i) + 156u < n_t) ? coin_bit(h2) : 0u;
            const u32 balo = __ballot_sync(FULLMASK, blo);
            const u32 bahi = __ballot_sync(FULLMASK, bhi);
            if (lane == 0) {
                if (balo) {
                    const u32 pos = base + 32u * u32(g);
                    const u32 w0 = pos >> 5, sh = pos & 31;
                    atomicOr(&coin[w0], balo << sh);
                    if (sh)
                        atomicOr(&coin[w0 + 1], balo >> (32 - sh));
                }
                if (bahi) {
                    const u32 pos = base + 156u + 32u * u32(g);
                    const u32 w0 = pos >> 5, sh = pos & 31;
                    atomicOr(&coin[w0], bahi << sh);
                    if (sh)
                        atomicOr(&coin[w0 + 1], bahi >> (32 - sh));
                }
                bnd[b ^ 1][2 * g] = l2;
                bnd[b ^ 1][2 * g + 1] = h2;
            }
            if (i == 1)
                bnd[b ^ 1][10] = l2;
        }
        if (NW > 1)
            __syncthreads();
        else
            __syncwarp();
    }
#pragma unroll
    for (int r = 0; r < RG; ++r) {
        const int g = warp + r * NW;
        const int i = 32 * g + lane;
        if (g < 5 && i < 156) {
            mt[i] = lo[r];
            mt[i + 156] = hi[r];
        }
    }
    __syncthreads();
    return n_t;
}

#ifndef TCSE_TWIST_REG_MIN
#define TCSE_TWIST_REG_MIN TCSE_FUSED_TWIST_MIN  // block sizes twisting in registers (2 barriers)
#endif
template <int NT>
__device__ __forceinline__ void mt_twist() {
    if constexpr (NT >= TCSE_TWIST_REG_MIN)
        mt_twist_impl<NT, false>(nullptr, 0u, 0u);
    else
        mt_twist_small<NT>();
}

struct Slot {
    int strategy;
    double alpha, beta, p_greedy;
    u64 seed;
};

// assign_strategies (parallel_search.hpp:183-205) for global process p: the
// first five outputs of mt19937_64(mix_seed{master, salt, iteration, p})
__device__ __noinline__ void derive_slot(const SysDesc& sd, int iteration, u64 p, Slot* out) {
    u64 h = 0x5851f42d4c957f2dULL;
    h = splitmix64(h ^ sd.master_seed);
    h = splitmix64(h ^ sd.salt);
    h = splitmix64(h ^ u64(int64_t(iteration)));
    h = splitmix64(h ^ p);
    u64 x = h;
    const u64 l0 = x;
    x = kMtF * (x ^ (x >> 62)) + 1;
    const u64 l1 = x;
    x = kMtF * (x ^ (x >> 62)) + 2;
    const u64 l2 = x;
    x = kMtF * (x ^ (x >> 62)) + 3;
    const u64 l3 = x;
    x = kMtF * (x ^ (x >> 62)) + 4;
    const u64 l4 = x;
    x = kMtF * (x ^ (x >> 62)) + 5;
    const u64 l5 = x;
#pragma unroll 10
    for (u32 i = 6; i <= 156; ++i)
        x = kMtF * (x ^ (x >> 62)) + i;
    const u64 h0 = x;
    x = kMtF * (x ^ (x >> 62)) + 157;
    const u64 h1 = x;
    x = kMtF * (x ^ (x >> 62)) + 158;
    const u64 h2 = x;
    x = kMtF * (x ^ (x >> 62)) + 159;
    const u64 h3 = x;
    x = kMtF * (x ^ (x >> 62)) + 160;
    const u64 h4 = x;
    const u64 o0 = mt_temper(mt_mix(l0, l1, h0));
    const u64 o1 = mt_temper(mt_mix(l1, l2, h1));
    const u64 o2 = mt_temper(mt_mix(l2, l3, h2));
    const u64 o3 = mt_temper(mt_mix(l3, l4, h3));
    const u64 o4 = mt_temper(mt_mix(l4, l5, h4));
    out->alpha = uniform_real(o0, 0.0, 0.5);
    out->beta = uniform_real(o1, 0.5, 1.0);
    out->p_greedy = uniform_real(o2, 0.5, 1.0);
    if (sd.forced >= 0) {
        out->strategy = sd.forced;
        out->seed = o3;
    } else if (iteration == 1 && p == 0) {
        out->strategy = TCSE_GREEDY;
        out->seed = o3;
    } else {
        double target = __dmul_rn(uniform_real(o3, 0.0, 1.0), sd.weight_total);
        int st = TCSE_GREEDY;
        for (int k = 0; k < 7; ++k) {
            target = __dsub_rn(target, sd.weights[k]);
            if (target < 0.0) {
                st = k;
                break;
            }
        }
        out->strategy = st;
        out->seed = o4;
    }
}

// frequency of (a, b, neg), 1-based ids (count_pairs, linear_system.hpp:151-161)
template <int W>
__device__ __forceinline__ int count_pair(int a, int b, int neg) {
    const u64* pa = mask_base() + size_t(a - 1) * 2 * W;
    const u64* pb = mask_base() + size_t(b - 1) * 2 * W;
    int c = 0;
#pragma unroll
    for (int w = 0; w < W; ++w)
        c += neg ? (__popcll(pa[w] & pb[W + w]) + __popcll(pa[W + w] & pb[w]))
                 : (__popcll(pa[w] & pb[w]) + __popcll(pa[W + w] & pb[W + w]));
    return c;
}

// every pair of the state with count >= minc, canonical order (dump mode,
// base candidate lists)
template <int W, int NT>
__device__ __noinline__ int all_pairs(int V, int minc, u32* okeys, u16* ocnts, int cap, int rsel0) {
    const int tid = threadIdx.x;
    int n_total = 0, rsel = rsel0;
    for (int a = 1; a < V; ++a) {
        const int L = 2 * (V - a);
        const int E = (L + NT - 1) / NT;
        const int e0 = min(L, tid * E), e1 = min(L, e0 + E);
        u32 local = 0;
        for (int e = e0; e < e1; ++e)
            local += count_pair<W>(a, a + 1 + (e >> 1), e & 1) >= minc ? 1u : 0u;
        u32 total;
        rsel ^= 1;
        u32 ex = block_scan<NT>(local, g_red + rsel * (NT / 32 + 2), &total);
        for (int e = e0; e < e1; ++e) {
            const int b = a + 1 + (e >> 1);
            const int cc = count_pair<W>(a, b, e & 1);
            if (cc >= minc) {
                const int pos = n_total + int(ex);
                if (pos < cap) {
                    okeys[pos] = make_key(a, b, e & 1);
                    ocnts[pos] = u16(cc);
                }
                ++ex;
            }
        }
        n_total += int(total);
    }
    __syncthreads();
    return n_total;
}

// FNV-1a over (i, j, sign, count) of the candidate list (trace, one thread)
__device__ __noinline__ u64 cand_hash(const u32* keys, const u16* cnts, int m) {
    u64 h = 0xcbf29ce484222325ULL;
    for (int t = 0; t < m; ++t) {
        const u32 kk = keys[t];
        const int f[4] = {key_i(kk), key_j(kk), key_neg(kk) ? -1 : 1, int(cnts[t])};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const u32 u = u32(f[q]);
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                h ^= (u >> (8 * b)) & 0xffu;
                h *= 0x100000001b3ULL;
            }
        }
    }
    return h;
}

// ------------------------------------------------------------- process

template <int W, int NT>
struct St {
    static constexpr int NW = NT / 32;
    int tid, lane;
    int V;      // variables alive (n_x + n_f)
    int m;      // candidates
    int cost;   // total_cost (linear_system.hpp:202-204)
    int mti;    // mt19937_64 position (312 = twist pending)
    int rsel;   // reduction buffer selector
    u32 last_coins;

    __device__ __forceinline__ u32* keys() { return sp<u32>(lay.keys0); }
    __device__ __forceinline__ u16* cnts() { return sp<u16>(lay.cnts0); }
    __device__ __forceinline__ u64* P(int v) { return mask_base() + size_t(v) * 2 * W; }
    __device__ __forceinline__ u64* N(int v) { return mask_base() + size_t(v) * 2 * W + W; }
    __device__ __forceinline__ u32* red() {
        rsel ^= 1;
        return g_red + rsel * (NW + 2);
    }
    __device__ __forceinline__ int argmax(double s, int idx) {
        rsel ^= 1;
        const int q = block_argmax_double<NT>(s, idx, g_reds + rsel * NW, g_redi + rsel * NW);
        return q == 0x7fffffff ? 0 : q;  // only for NaN scores: stay inside the list
    }

    // ---- mt19937_64, block-uniform: every thread walks the same stream
    __device__ __forceinline__ u64 draw() {
        if (mti >= 312) {
            mt_twist<NT>();
            mti = 0;
        }
        return mt_temper(g_mt[mti++]);
    }

    // uniform_int_distribution downscaling: _S_nd<unsigned __int128>
    // (bits/uniform_int_dist.h:257-281); value in [0, range)
    __device__ u64 nd(u64 range) {
        u64 x = draw();
        u64 lo = x * range;
        u64 hi = __umul64hi(x, range);
        if (lo < range) {
            const u64 th = (0ULL - range) % range;
            while (lo < th) {
                x = draw();
                lo = x * range;
                hi = __umul64hi(x, range);
            }
        }
        return hi;
    }

    // n coin flips (uniform_int_distribution<int>(0,1) == top tempered bit)
    // precleared: the caller zeroed the buffer's first words behind a barrier
    // (only the register-resident generations of 128-/256-thread blocks OR
    // bits into the buffer; smaller blocks store whole words)
    __device__ void draw_coins(u32 nbits, bool precleared = false) {
        u32* coin = sp<u32>(lay.coin);
        if (!precleared && (NT >= TCSE_FUSED_TWIST_MIN || TCSE_SMALL_TWIST_COINS)) {
            const u32 words = (nbits + 31) >> 5;
#pragma unroll 1
            for (u32 w = tid; w < words; w += NT)
                coin[w] = 0u;
            __syncthreads();
        }
        u32 done = 0;
        while (done < nbits) {
            if (mti >= 312) {
                if constexpr (NT >= TCSE_FUSED_TWIST_MIN) {
                    // every remaining coin from fresh generations, state in registers
                    mti = int(mt_coin_run<NT>(coin, done, nbits - done));
                    done = nbits;
                    break;
                } else {
#if TCSE_SMALL_TWIST_COINS
                    // twist and extract this generation's coins in one pass
                    const u32 n = min(312u, nbits - done);
                    mt_twist_small_coins<NT>(coin, done, n);
                    mti = int(n);
                    done += n;
                    continue;
#else
                    mt_twist<NT>();
                    mti = 0;
#endif
                }
            }
            // this segment's coins as whole buffer words: lane l of word k
            // holds position 32 (done / 32 + k) + l, element l + 32 k - sh of
            // the generation's remaining outputs; a plain store per word,
            // except the first word's OR onto the previous segment's bits
            // (written before the twist's barriers).  Bits past the segment
            // stay zero until the next segment ORs them.
            const u32 n = min(u32(312 - mti), nbits - done);
            const u32 sh = done & 31u;
            const u32 nw32 = (sh + n + 31) & ~31u;
            // (branch-free body: a clamped load from a 32-bit shared address
            // computed once — a generic pointer makes the compiler rebuild
            // the shared window base inside the loop —, one store path for
            // lane 0; the loop bound is per warp)
            const u32 mt_s = u32(__cvta_generic_to_shared(g_mt)) + 8u * u32(mti);
            u32* cw = coin + (done >> 5);
            const u32 prev = sh ? cw[0] : 0u;  // the previous segment's bits of the first word
            for (u32 t0 = u32(tid & ~31); t0 < nw32; t0 += NT) {
                const u32 e = t0 + u32(lane) - sh;  // wraps for t < sh: out of range
                const bool ok = e < n;
                u32 lo, hi;
                asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(mt_s + 8u * (ok ? e : 0u)));
                const u32 bit = u32(__popc((hi & u32(kCoinMask >> 32)) ^ (lo & u32(kCoinMask)))) & 1u;
                const u32 ball = __ballot_sync(FULLMASK, ok && bit);
                if (lane == 0)
                    cw[t0 >> 5] = t0 == 0u ? (prev | ball) : ball;
            }
            mti += int(n);
            done += n;
        }
        __syncthreads();
    }

    // ---- substitution (apply_substitution, linear_system.hpp:167-189):
    // returns the replaced occurrences; 0 leaves the state untouched
    __device__ int apply(u32 q) {
        u32* bc = g_bcast;
        if (tid == 0) {
            const int i = key_i(q) - 1, j = key_j(q) - 1, neg = key_neg(q);
            u64* pi = P(i);
            u64* pj = P(j);
            u64* pk = P(V);
            u64 rp[W], rn[W];
            int c = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                rp[w] = pi[w] & (neg ? pj[W + w] : pj[w]);
                rn[w] = pi[W + w] & (neg ? pj[w] : pj[W + w]);
                c += __popcll(rp[w]) + __popcll(rn[w]);
            }
            if (c > 0) {
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    pi[w] &= ~rp[w];
                    pi[W + w] &= ~rn[w];
                    if (!neg) {
                        pj[w] &= ~rp[w];
                        pj[W + w] &= ~rn[w];
                    } else {
                        pj[W + w] &= ~rp[w];
                        pj[w] &= ~rn[w];
                    }
                    pk[w] = rp[w];
                    pk[W + w] = rn[w];
                }
            }
            bc[0] = u32(c);
        }
        __syncthreads();
        const int c = int(bc[0]);
        if (c > 0) {
            ++V;
            cost -= c - 1;
        }
        return c;
    }

    // incremental candidate maintenance after q -> k (= V, 1-based); false if
    // the new list would not fit the capacity (nothing written, block-uniform)
    __device__ bool update(u32 q) {
        const int i = key_i(q), j = key_j(q);
        const int k = V;
        const u32* ok = keys();
        const u16* oc = cnts();
        u32* kc = sp<u32>(lay.kcopy);  // the old keys: the list is rewritten in place below
        u16* tcnt = sp<u16>(lay.tcnt);
        u16* ncp = sp<u16>(lay.ncp);
        u16* ncn = sp<u16>(lay.ncn);
        u32* aux = sp<u32>(lay.aux);
        u32* newexcl = sp<u32>(lay.newexcl);
        // (a) recount old candidates touching i or j (their counts only drop);
        // blocked ranges, survivors counted on the way
        const int Em = (m + NT - 1) / NT;
        const int a0 = min(m, tid * Em), a1 = min(m, a0 + Em);
        u32 keep = 0;
#pragma unroll 1
        for (int t = a0; t < a1; ++t) {
            const u32 kk = ok[t];
            const int a = key_i(kk), b = key_j(kk);
            const u16 ct = (a == i || a == j || b == i || b == j) ? u16(count_pair<W>(a, b, key_neg(kk))) : oc[t];
            tcnt[t] = ct;
            kc[t] = kk;
            keep += ct >= 2 ? 1u : 0u;
        }
        // (b) the new variable's pairs (x, k, +/-)
        const u64* pk = P(k - 1);
        bool anynew = false;
        u64 kp[W], kn[W];
#pragma unroll
        for (int w = 0; w < W; ++w) {
            kp[w] = pk[w];
            kn[w] = pk[W + w];
        }
#pragma unroll 1
        for (int x = tid + 1; x < k; x += NT) {
            const u64* px = P(x - 1);
            int cp = 0, cn = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                cp += __popcll(px[w] & kp[w]) + __popcll(px[W + w] & kn[w]);
                cn += __popcll(px[w] & kn[w]) + __popcll(px[W + w] & kp[w]);
            }
            ncp[x] = u16(cp);
            ncn[x] = u16(cn);
            anynew |= (cp >= 2) | (cn >= 2);
        }
        // survivors' scan, high half: threads that found a repeating (x, k, .)
        const u64 sc = block_scan_ool<NT>(keep | (anynew ? 0x10000u : 0u), red());
        // (every read of the old list is done: the scan's barrier separates
        // them from the in-place rewrite, which reads kc / tcnt only)
        u32* dk = sp<u32>(lay.keys0);
        u16* dc = sp<u16>(lay.cnts0);
        if ((sc >> 48) == 0) {
            // common case: no pair with k repeats, the list only loses entries
            u32 o = u32(sc) & 0xffffu;
#pragma unroll 1
            for (int t = a0; t < a1; ++t)
                if (tcnt[t] >= 2) {
                    dk[o] = kc[t];
                    dc[o] = tcnt[t];
                    ++o;
                }
            __syncthreads();
            m = int((sc >> 32) & 0xffffu);
            return true;
        }
        // (c) general case: old survivors of this thread's candidate range
        // [a0, a1) (counted in (a)) and new pairs (x, k, +/-) of its variable
        // range [x0, x1) within [1, k); one packed scan, low 16 bits old
        const int Ex = (k - 1 + NT - 1) / NT;
        const int x0 = min(k, 1 + tid * Ex), x1 = min(k, x0 + Ex);
        u32 nn = 0;
#pragma unroll 1
        for (int x = x0; x < x1; ++x)
            nn += (ncp[x] >= 2 ? 1u : 0u) + (ncn[x] >= 2 ? 1u : 0u);
        const u64 sc_excl = block_scan_ool<NT>(keep | (nn << 16), red());
        const u32 excl = u32(sc_excl), total = u32(sc_excl >> 32);
        const u32 n_old = total & 0xffffu, n_new = total >> 16;
        if (int(n_old + n_new) > mcap)
            return false;
        u32 o = excl & 0xffffu, n = excl >> 16;
#pragma unroll 1
        for (int t = a0; t < a1; ++t) {
            aux[t] = o;
            o += tcnt[t] >= 2 ? 1u : 0u;
        }
#pragma unroll 1
        for (int x = x0; x < x1; ++x) {
            newexcl[x] = n;
            n += (ncp[x] >= 2 ? 1u : 0u) + (ncn[x] >= 2 ? 1u : 0u);
        }
        __syncthreads();
        o = excl & 0xffffu;
#pragma unroll 1
        for (int t = a0; t < a1; ++t)
            if (tcnt[t] >= 2) {
                const u32 kk = kc[t];
                const u32 dest = o + newexcl[key_i(kk)];
                dk[dest] = kk;
                dc[dest] = tcnt[t];
                ++o;
            }
        n = excl >> 16;
#pragma unroll 1
        for (int x = x0; x < x1; ++x) {
#pragma unroll 1
            for (int sg = 0; sg < 2; ++sg) {
                const u16 c = sg ? ncn[x] : ncp[x];
                if (c >= 2) {
                    // old survivors before (x, k, .) are those with i <= x
                    const u32 bound = u32(x + 1) << 17;
                    int lo = 0, hi = m;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (kc[mid] < bound)
                            lo = mid + 1;
                        else
                            hi = mid;
                    }
                    const u32 before = lo < m ? aux[lo] : n_old;
                    const u32 dest = n + before;
                    dk[dest] = make_key(x, k, sg);
                    dc[dest] = c;
                    ++n;
                }
            }
        }
        __syncthreads();
        m = int(n_old + n_new);
        return true;
    }

    // ---- selection strategies (strategies.hpp); return a candidate index

    // greedy_from (61-69): first maximum in canonical order
    __device__ int sel_greedy() {
        const u16* c = cnts();
        u32 best = 0;
#pragma unroll 1
        for (int t = tid; t < m; t += NT)
            best = max(best, (u32(c[t]) << 16) | (0xffffu - u32(t)));
        best = block_max<NT>(best, red());
        return int(0xffffu - (best & 0xffffu));
    }

    // greedy_alternative_from (71-83): uniform over the argmax set
    __device__ int sel_ga() {
        const u16* c = cnts();
        u32 mx = 0;
#pragma unroll 1
        for (int t = tid; t < m; t += NT)
            mx = max(mx, u32(c[t]));
        mx = block_max<NT>(mx, red());
        // the argmax set's size is the scan's total (one pass, one barrier less)
        const int E = (m + NT - 1) / NT;
        const int e0 = min(m, tid * E), e1 = min(m, e0 + E);
        u32 local = 0;
#pragma unroll 1
        for (int e = e0; e < e1; ++e)
            local += c[e] == mx ? 1u : 0u;
        const u64 sc_ex = block_scan_ool<NT>(local, red());
        u32 ex = u32(sc_ex);
        const u32 r = u32(nd(u32(sc_ex >> 32)));
        u32* bc = g_bcast;
#pragma unroll 1
        for (int e = e0; e < e1; ++e)
            if (c[e] == mx) {
                if (ex == r)
                    bc[1] = u32(e);
                ++ex;
            }
        __syncthreads();
        return int(bc[1]);
    }

    // weighted_random_from (85-98): first q with prefix(c - 1) > u * total
    __device__ int sel_wr() {
        const u16* c = cnts();
        u32* bc = g_bcast;
        // the total weight is the scan's total (one pass, two barriers less);
        // bc[1] was last read before the previous substitution's barriers
        if (tid == 0)
            bc[1] = u32(m - 1);
        const int E = (m + NT - 1) / NT;
        const int e0 = min(m, tid * E), e1 = min(m, e0 + E);
        u32 local = 0;
#pragma unroll 1
        for (int e = e0; e < e1; ++e)
            local += u32(c[e]) - 1u;
        const u64 sc_s = block_scan_ool<NT>(local, red());
        u32 s = u32(sc_s);
        const double target = __dmul_rn(uniform_real(draw(), 0.0, 1.0), double(u32(sc_s >> 32)));
#pragma unroll 1
        for (int e = e0; e < e1; ++e) {
            const u32 s1 = s + u32(c[e]) - 1u;
            if (double(s1) > target && double(s) <= target)
                bc[1] = u32(e);
            s = s1;
        }
        __syncthreads();
        return int(bc[1]);
    }

    // select_greedy_intersections (162-176), alpha != 0.  Coins are drawn in
    // (q, s) order; q's score is the reference's sequential double sum,
    // evaluated in O(deg q) (see the header comment).
    template <bool dense, int F = 0>
    __device__ int sel_gi(double alpha, double beta) {
        constexpr bool SM = (F & kFormSmall) != 0;
        constexpr bool BM = (F & kFormBm) != 0;  // the system's gi_bm, known at compile time
#ifndef TCSE_GI_HYBRID
#define TCSE_GI_HYBRID 1
#endif
        // one-warp pruned systems (the 4x4x4 U, V lists start at 40
        // candidates): once the list is down to 32 the exact small-list loop
        // replaces the approximate pass
        // (also the 2-word two-warp kernel — 5x5x5 U, V lists start at ~40 —
        // not the 1-word one: -2% on the 4x4x4 W group, +3.5% on 5x5x5:110)
        constexpr bool HYB = TCSE_GI_HYBRID && BM && !SM && (NT == 32 || (NT == 64 && W == 2));
        // the walk needs a non-decreasing running sum (beta >= 0, always true
        // for assign_strategies' slots); any other beta runs the reference loop
        const bool walk = !dense && beta >= 0.0;
        // dense form with near-best pruning: integer score sums in the
        // candidate loop, exact folds only for near-ties (same bound as the walk)
        // (never in the small-list instantiation: its systems do not prune,
        // so the pruning code is compiled out of it)
        const bool approx = !SM && dense && gi_prune > 0 && m >= gi_prune && beta >= 0.0 && !(HYB && m <= 32);
        // lists of at most 32 candidates without pruning: the reference loop
        // branch-free over bitmap neighbour masks (gi_dense_small)
        // (its own instantiation, SM: the code costs the others spills)
        const bool small = (SM || HYB) && dense && !approx && m <= 32;
        // max c - 1 over the list (crossing bound) and max coins per candidate
        // in wbt's spare slot
        u32* s_wmax = reinterpret_cast<u32*>(sp<double>(lay.wbt) + sd_ne + 1);
        u32* s_dmax = s_wmax + 1;
        const u32* ks = keys();
        const u16* c = cnts();
        const int V1 = V + 1;
        u32* nA = sp<u32>(lay.nA);
        u32* nB = sp<u32>(lay.nB);
        u32* qbase = sp<u32>(lay.qbase);
        double* wbt = sp<double>(lay.wbt);
        const u32* coin = sp<u32>(lay.coin);
        // @region gi_zero
        const int nwl = int(bm_stride(mcap));  // bitmap row stride (words)
        const int nwm = (m + 31) >> 5;     // words in use this step
        u32* bm = sp<u32>(lay.bm);
#pragma unroll 1
        for (int v = tid; v < V1; v += NT) {
            nA[v] = 0u;
            if (walk)
                nB[v] = 0u;
        }
        if (BM && (approx || small)) {
#pragma unroll 1
            for (int v = tid; v < V1; v += NT)
#pragma unroll 1
                for (int w = 0; w < nwm; ++w)
                    bm[v * nwl + w] = 0u;
        }
#pragma unroll 1
        for (int cc = tid; cc <= sd_ne; cc += NT)
            wbt[cc] = __dmul_rn(beta, double(cc - 1));
        if (tid == 0) {
            *s_wmax = 0u;
            *s_dmax = 0u;
        }
        __syncthreads();
        // @region gi_counts
        // per-variable candidate counts (reference loop: total in nA; walk: A = as
        // second element, B = as first element)
        if (!walk) {
            u32 lmax = 0u;
            // bitmap layout: row 0 (no variable has id 0) marks the heavy
            // candidates (c >= 3, weight > 1), one ballot per 32 of them
            const bool hb = BM && (approx || small);
            const int mr = hb ? (m + 31) & ~31 : m;
#pragma unroll 1
            for (int t = tid; t < mr; t += NT) {
                const bool on = t < m;
                if (on) {
                    const u32 kk = ks[t];
                    atomicAdd(&nA[key_i(kk)], 1u);
                    atomicAdd(&nA[key_j(kk)], 1u);
                    lmax = max(lmax, u32(c[t]) - 1u);
                    if (hb) {
                        atomicOr(&bm[key_i(kk) * nwl + (t >> 5)], 1u << (t & 31));
                        atomicOr(&bm[key_j(kk) * nwl + (t >> 5)], 1u << (t & 31));
                    }
                }
                if (hb) {  // warp-uniform: mr and NT are multiples of 32
                    const u32 heavy = __ballot_sync(FULLMASK, on && c[t] >= 3);
                    if (lane == 0)
                        bm[t >> 5] = heavy;
                }
            }
            if (approx) {
                lmax = __reduce_max_sync(FULLMASK, lmax);
                if (lane == 0)
                    atomicMax(s_wmax, lmax);
            }
        } else {
            u32* bs = sp<u32>(lay.bs);
            u32 lmax = 0u;
#pragma unroll 1
            for (int t = tid; t < m; t += NT) {
                const u32 kk = ks[t];
                const int a = key_i(kk), b = key_j(kk);
                atomicAdd(&nA[b], 1u);
                atomicAdd(&nB[a], 1u);
                if (t == 0 || key_i(ks[t - 1]) != a)
                    bs[a] = u32(t);
                lmax = max(lmax, u32(c[t]) - 1u);
            }
            lmax = __reduce_max_sync(FULLMASK, lmax);
            if (lane == 0)
                atomicMax(s_wmax, lmax);
        }
        __syncthreads();
        if (walk) {
            // @region gi_aoff
            // A-list offsets: scan over variables
            u32* aoff = sp<u32>(lay.aoff);
            u32* cursor = sp<u32>(lay.cursor);
            const int E = (V1 + NT - 1) / NT;
            const int e0 = min(V1, tid * E), e1 = min(V1, e0 + E);
            u32 local = 0;
#pragma unroll 1
            for (int e = e0; e < e1; ++e)
                local += nA[e];
            u32 total;
            const u64 sc_ex = block_scan_ool<NT>(local, red());
            u32 ex = u32(sc_ex);
            total = u32(sc_ex >> 32);
#pragma unroll 1
            for (int e = e0; e < e1; ++e) {
                aoff[e] = ex;
                cursor[e] = ex;
                ex += nA[e];
            }
        }
        // @region gi_deg_scan
        // coins per q = candidates sharing a variable, minus q itself (and its
        // opposite-sign twin, counted under both variables); w prefix sums
        const int E = (m + NT - 1) / NT;
        const int e0 = min(m, tid * E), e1 = min(m, e0 + E);
        u32 D;
        {
            u32 ld = 0, lw = 0, dmax = 0;
#pragma unroll 1
            for (int e = e0; e < e1; ++e) {
                const u32 kk = ks[e];
                const u32 twin = (e + 1 < m && ks[e + 1] == (kk | 1u) && !(kk & 1u)) ||
                                         (e > 0 && (kk & 1u) && ks[e - 1] == (kk & ~1u))
                                     ? 1u
                                     : 0u;
                const int a = key_i(kk), b = key_j(kk);
                const u32 dq = !walk ? nA[a] + nA[b] - 2u - twin : nA[a] + nB[a] + nA[b] + nB[b] - 2u - twin;
                qbase[e] = dq;  // this thread's range only; prefix below
                ld += dq;
                dmax = max(dmax, dq);
                lw += u32(c[e]) - 1u;
            }
            if (approx) {
                dmax = __reduce_max_sync(FULLMASK, dmax);
                if (lane == 0)
                    atomicMax(s_dmax, dmax);
            }
            u32 exd, W_ = 0, exw = 0;
            if ((walk || approx) && m <= 180 && u32(m) * (*s_wmax + 1u) < 65536u) {
                // degrees (sum <= 2 m^2) and weights in one packed 16/16 scan
                const u64 sc = block_scan_ool<NT>(ld | (lw << 16), red());
                exd = u32(sc) & 0xffffu;
                exw = u32(sc) >> 16;
                D = u32(sc >> 32) & 0xffffu;
                W_ = u32(sc >> 32) >> 16;
            } else {
                const u64 sc_exd = block_scan_ool<NT>(ld, red());
                exd = u32(sc_exd);
                D = u32(sc_exd >> 32);
                if (walk || approx) {
                    const u64 sc_w = block_scan_ool<NT>(lw, red());
                    exw = u32(sc_w);
                    W_ = u32(sc_w >> 32);
                }
            }
            u32* wp = sp<u32>(lay.wp);
#pragma unroll 1
            for (int e = e0; e < e1; ++e) {
                const u32 dq = qbase[e];
                qbase[e] = exd;
                exd += dq;
                if (walk || approx) {
                    wp[e] = exw;
                    exw += u32(c[e]) - 1u;
                }
            }
            if (tid == 0) {
                qbase[m] = D;
                if (walk || approx)
                    wp[m] = W_;
            }
            // the first coin chunk's words, behind the barrier below (only
            // where coin bits are OR-ed in: draw_coins)
            if (dense && (NT >= TCSE_FUSED_TWIST_MIN || TCSE_SMALL_TWIST_COINS)) {
                u32* coin = sp<u32>(lay.coin);
                const u32 words = (min(D, lay.coin_cap) + 31) >> 5;
#pragma unroll 1
                for (u32 w = tid; w < words; w += NT)
                    coin[w] = 0u;
            }
        }
        __syncthreads();
        last_coins = D;
        double best_s = -INFINITY;
        int best_q = 0x7fffffff;
        const double topmin = double(*s_wmax) + 1.0;
        if (walk) {
            u32* aoff = sp<u32>(lay.aoff);
            u32* cursor = sp<u32>(lay.cursor);
            u32* bs = sp<u32>(lay.bs);
            u16* alist = sp<u16>(lay.alist);
            const u32* wp = sp<u32>(lay.wp);
            // @region gi_alist
            // A lists: candidate indices by second element, index order
#pragma unroll 1
            for (int t = tid; t < m; t += NT)
                alist[atomicAdd(&cursor[key_j(ks[t])], 1u)] = u16(t);
            __syncthreads();
#pragma unroll 1
            for (int v = tid; v < V1; v += NT) {
                const int b0 = int(aoff[v]), n = int(nA[v]);
#pragma unroll 1
                for (int x = 1; x < n; ++x) {
                    const u16 t = alist[b0 + x];
                    int y = x - 1;
                    while (y >= 0 && alist[b0 + y] > t) {
                        alist[b0 + y + 1] = alist[b0 + y];
                        --y;
                    }
                    alist[b0 + y + 1] = t;
                }
            }
            // Scores in chunks of candidates whose coins fit the buffer.
            // prune: every candidate first gets an approximate score from
            // exact integer sums (disjoint weight D_q, coin-weighted
            // intersecting weight C_q): H~ = w_q + a (D_q + b C_q).  The
            // reference's sequential double H differs from H~ by at most
            // eps (recursive-summation bound, 4x margin: DESIGN.md section 3),
            // so only candidates with H~ >= max H~ - 2 eps can be the
            // reference's pick; those alone are folded exactly (the walk
            // below, bit-identical to score_intersections_from) while their
            // coins are still in the buffer, and the exact scores decide.
            const u32 cap = lay.coin_cap;
            const u32 T = wp[m];
            const double eps =
                double(m + 16) * (double(*s_wmax) + fabs(alpha) * double(T) * fmax(1.0, beta)) * 0x1p-51;
            const double eps2 = __dmul_rn(2.0, eps);
            double B = -INFINITY;  // running max of the approximate scores
            int q_lo = 0;
            while (q_lo < m) {
                const u32 c0 = qbase[q_lo];
                // (every remaining coin fits: the common case, no search)
                int lo = qbase[m] - c0 <= cap ? m : q_lo + 1, hi = m;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (qbase[mid] - c0 <= cap)
                        lo = mid;
                    else
                        hi = mid - 1;
                }
                const int q_hi = lo;
                // @region gi_coins
                draw_coins(qbase[q_hi] - c0);  // barrier-separated clear, ends with a barrier
                // @region gi_approx_pass
                if (!gi_prune) {
                    for (int q = q_lo + tid; q < q_hi; q += NT) {
                        const double h = gi_fold(ks, c, m, q, c0, alpha, topmin);
                        if (h > best_s || best_q == 0x7fffffff) {
                            best_s = h;
                            best_q = q;
                        }
                    }
                } else {
                    double lb = -INFINITY, h1 = 0.0, h2 = 0.0;
                    int q1 = -1, q2 = -1;
                    bool ovf = false;
                    for (int q = q_lo + tid; q < q_hi; q += NT) {
                        const double h = gi_approx(ks, c, q, c0, T, alpha, beta);
                        lb = fmax(lb, h);
                        const double lim = __dsub_rn(lb, eps2);
                        if (q1 >= 0 && h1 < lim)
                            q1 = -1;
                        if (q2 >= 0 && h2 < lim)
                            q2 = -1;
                        if (h >= lim) {
                            if (q1 < 0) {
                                q1 = q;
                                h1 = h;
                            } else if (q2 < 0) {
                                q2 = q;
                                h2 = h;
                            } else {
                                ovf = true;
                            }
                        }
                    }
                    // @region gi_folds
                    int lone = 0;
                    const u32 info = near_best(lb, eps2, q1, h1, q2, h2, ovf, B, lone);
                    if (info == 1u && q_lo == 0 && q_hi == m)
                        return lone;  // a lone near-best candidate is the pick: no fold, no argmax
                    const double thr = __dsub_rn(B, eps2);
                    if (ovf) {  // more than two near-ties in one thread: rescan
                        const double2 r = gi_rescan(ks, c, m, q_lo, q_hi, c0, T, alpha, beta, topmin, thr, best_s,
                                                    best_q);
                        best_s = r.x;
                        best_q = __double_lo_as_int(r.y);
                    } else {
                        if (q1 >= 0 && h1 >= thr)
                            gi_keep(gi_fold(ks, c, m, q1, c0, alpha, topmin), q1, best_s, best_q);
                        if (q2 >= 0 && h2 >= thr)
                            gi_keep(gi_fold(ks, c, m, q2, c0, alpha, topmin), q2, best_s, best_q);
                    }
                }
                __syncthreads();
                q_lo = q_hi;
            }
        } else {
            // @region gi_dense
            // Dense layout.  With near-best pruning (approx; needs T < 2^16 and
            // at most 64 coins per candidate) one pass per coin chunk computes
            // every candidate's exact integer sums (intersecting weight I_q and
            // its coin-selected part C_q, packed I << 16 | C) and the
            // approximate score w_q + a (T - w_q - I_q + b C_q) — within eps of
            // the reference's sequential double (the walk's bound).  Only
            // candidates within 2 eps of the best approximate score can be the
            // reference's pick: a lone one is the pick; several are folded
            // exactly (gi_fold_dense, one warp per candidate) and the exact
            // scores decide.  A thread with more than two near-best candidates,
            // or the layout without pruning, runs the reference loop itself
            // (gi_dense_chunk).
            const u32 cap = lay.coin_cap;
            const bool use_approx = approx && wp_total() < 65536u && *s_dmax <= 64u;
            const u32 T = use_approx ? wp_total() : 0u;
            const double eps = use_approx ? double(m + 16) * (double(*s_wmax) +
                                                              fabs(alpha) * double(T) * fmax(1.0, beta)) * 0x1p-51
                                          : 0.0;
            const double eps2 = __dmul_rn(2.0, eps);
            double B = -INFINITY;
            int q_lo = 0;
            while (q_lo < m) {
                const u32 c0 = qbase[q_lo];
                // (every remaining coin fits: the common case, no search)
                int lo = qbase[m] - c0 <= cap ? m : q_lo + 1, hi = m;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (qbase[mid] - c0 <= cap)
                        lo = mid;
                    else
                        hi = mid - 1;
                }
                const int q_hi = lo;
                draw_coins(qbase[q_hi] - c0, dense && q_lo == 0);  // walk layout (beta < 0) clears here
                if (!use_approx) {
                    GI_STAT(4, 1);
                    double2 r;
                    if constexpr (SM || HYB)
                        r = small ? gi_dense_small(ks, c, m, q_lo, q_hi, c0, alpha, best_s, best_q, int(bm_stride(mcap)))
                                  : gi_dense_chunk(ks, c, m, q_lo, q_hi, c0, alpha, best_s, best_q);
                    else
                        r = gi_dense_chunk(ks, c, m, q_lo, q_hi, c0, alpha, best_s, best_q);
                    best_s = r.x;
                    best_q = __double_lo_as_int(r.y);
                } else {
                    double lb = -INFINITY, h1 = 0.0, h2 = 0.0;
                    int q1 = -1, q2 = -1;
                    bool ovf = false;
                    if constexpr (BM) {
#if TCSE_GI_BALANCE
                        // contiguous candidate ranges of equal work (coins + a
                        // per-candidate share) per thread: lanes finish together
                        const u32 per = 6u;
                        const u32 total = qbase[q_hi] - c0 + per * u32(q_hi - q_lo);
                        auto split = [&](u32 target) {
                            int lo2 = q_lo, hi2 = q_hi;  // first q with work(q) >= target
                            while (lo2 < hi2) {
                                const int mid = (lo2 + hi2) >> 1;
                                if (qbase[mid] - c0 + per * u32(mid - q_lo) < target)
                                    lo2 = mid + 1;
                                else
                                    hi2 = mid;
                            }
                            return lo2;
                        };
                        const int qa = split(u32((u64(total) * u32(tid)) / NT));
                        const int qb = tid == NT - 1 ? q_hi : split(u32((u64(total) * u32(tid + 1)) / NT));
#pragma unroll 1
                        for (int q = qa; q < qb; ++q)
                            gi_score_bm(q, c0, T, alpha, beta, eps2, lb, q1, h1, q2, h2, ovf);
#else
#pragma unroll 1
                        for (int q = q_lo + tid; q < q_hi; q += NT)
                            gi_score_bm(q, c0, T, alpha, beta, eps2, lb, q1, h1, q2, h2, ovf);
#endif
                    } else {
                        for (int qb = q_lo; qb < q_hi;) {
                            if (q_hi - qb > NT) {
                                gi_pass<2>(qb + tid, q_hi, c0, T, alpha, beta, eps2, lb, q1, h1, q2, h2, ovf);
                                qb += 2 * NT;
                            } else {
                                gi_pass<1>(qb + tid, q_hi, c0, T, alpha, beta, eps2, lb, q1, h1, q2, h2, ovf);
                                qb += NT;
                            }
                        }
                    }
                    int lone = 0;
                    const u32 info = near_best(lb, eps2, q1, h1, q2, h2, ovf, B, lone);
                    const double thr = __dsub_rn(B, eps2);
                    const bool k1 = q1 >= 0 && h1 >= thr, k2 = q2 >= 0 && h2 >= thr;
                    GI_STAT(0, 1);
                    GI_STAT(5, m);
                    if (info >> 16) {
                        GI_STAT(3, 1);
                        const double2 r = gi_dense_chunk(ks, c, m, q_lo, q_hi, c0, alpha, best_s, best_q);
                        best_s = r.x;
                        best_q = __double_lo_as_int(r.y);
                    } else if ((info & 0xffffu) == 1u && q_lo == 0 && q_hi == m) {
                        // a lone near-best candidate is the reference's pick
                        // (single chunk: no argmax pass, every thread knows it)
                        GI_STAT(1, 1);
                        return lone;
                    } else {
                        // fold every near-best candidate exactly, one warp each
                        GI_STAT(6, 1);
                        GI_STAT(2, info & 0xffffu);
#pragma unroll 1
                        for (int r = 0; r < 2; ++r) {
                            const bool mine = r == 0 ? k1 : k2;
                            const int qm = r == 0 ? q1 : q2;
                            u32 pend = __ballot_sync(FULLMASK, mine);
                            while (pend) {
                                const int src = __ffs(pend) - 1;
                                pend &= pend - 1;
                                const int qf = __shfl_sync(FULLMASK, qm, src);
                                gi_keep(gi_fold_dense(ks, c, m, qf, c0, alpha, topmin), qf, best_s, best_q);
                            }
                        }
                    }
                }
                if (q_hi < m)  // the coin buffer is refilled; after the last chunk argmax's barrier suffices
                    __syncthreads();
                q_lo = q_hi;
            }
        }
        // @region gi_argmax
        return argmax(best_s, best_q);
    }

    __device__ __forceinline__ u32 wp_total() { return sp<u32>(lay.wp)[m]; }

    // score_intersections_from's loop for candidates [q_lo, q_hi) of the
    // current coin chunk; each thread carries up to K candidates through one
    // pass (K independent double chains); first maximum kept per thread.
    // Static and out of line: a cold path (prune off, negative beta, chunk
    // overflow) that must not pull the process state into local memory.
    template <int K>
    static __device__ __forceinline__ double2 gi_dense_chunk_k(const u32* ks, const u16* c, int m_, int q_lo, int q_hi,
                                                               u32 c0, double alpha, double best_s, int best_q) {
        const u32* qbase = sp<u32>(lay.qbase);
        const double* wbt = sp<double>(lay.wbt);
        const u32* coin = sp<u32>(lay.coin);
        for (int q0 = q_lo + int(threadIdx.x); q0 < q_hi; q0 += K * NT) {
            int qv[K], qi[K], qj[K];
            u32 ptr[K];
            double fut[K];
#pragma unroll
            for (int t = 0; t < K; ++t) {
                qv[t] = q0 + t * NT;
                const bool on = qv[t] < q_hi;
                const u32 kq = on ? ks[qv[t]] : 0u;
                qi[t] = on ? key_i(kq) : -1;  // -1 never matches a variable
                qj[t] = on ? key_j(kq) : -1;
                ptr[t] = on ? qbase[qv[t]] - c0 : 0u;
                fut[t] = 0.0;
            }
            for (int s = 0; s < m_; ++s) {
                const u32 kk = ks[s];
                const int si = key_i(kk), sj = key_j(kk);
                const u16 cs = c[s];
                const double wd = double(int(cs) - 1);
                const double wb = wbt[cs];
#pragma unroll
                for (int t = 0; t < K; ++t) {
                    const bool self = s == qv[t];
                    const bool inter = !self && ((si == qi[t]) | (si == qj[t]) | (sj == qi[t]) | (sj == qj[t]));
                    double add = self ? 0.0 : wd;  // q itself is skipped (fut + 0.0 == fut)
                    if (inter) {
                        add = ((coin[ptr[t] >> 5] >> (ptr[t] & 31u)) & 1u) ? wb : 0.0;
                        ++ptr[t];
                    }
                    fut[t] = __dadd_rn(fut[t], add);
                }
            }
#pragma unroll
            for (int t = 0; t < K; ++t)
                if (qv[t] < q_hi)
                    gi_keep(__dadd_rn(double(int(c[qv[t]]) - 1), __dmul_rn(alpha, fut[t])), qv[t], best_s, best_q);
        }
        return make_double2(best_s, __int_as_double_lo(best_q));
    }

    // The same loop for lists of at most 32 candidates (m <= NT: one
    // candidate per lane), branch-free: q's intersecting candidates as a
    // 32-bit mask from the per-variable bitmaps, its coins as a 32-bit window
    // in a register (deg q <= m - 1 <= 31).  The +0.0 additions of the reference (q
    // itself, a coin that did not select) are skipped: exact, the running
    // sum starts at +0.0 and never becomes -0.0.
    static __device__ __noinline__ double2 gi_dense_small(const u32* ks, const u16* c, int m_, int q_lo, int q_hi,
                                                          u32 c0, double alpha, double best_s, int best_q, int nwl) {
        const int q = q_lo + int(threadIdx.x);
        if (q < q_hi) {
            const u32* bm = sp<u32>(lay.bm);
            const double* wbt = sp<double>(lay.wbt);
            const u32* coin = sp<u32>(lay.coin);
            const u32 kq = ks[q];
            const u32 nb = (bm[key_i(kq) * nwl] | bm[key_j(kq) * nwl]) & ~(1u << q);
            const u32 p = sp<u32>(lay.qbase)[q] - c0;
            u32 win = __funnelshift_r(coin[p >> 5], coin[(p >> 5) + 1], p & 31u);
            double fut = 0.0;
#pragma unroll 4
            for (int s = 0; s < m_; ++s) {
                const u16 cs = c[s];
                const u32 in = (nb >> s) & 1u;
                // one addend and one predicated add (the compiler would add
                // and select the result instead)
                const u32 take = in ? (win & 1u) : u32(s != q);
                const double a = in ? wbt[cs] : double(int(cs) - 1);
                asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p add.rn.f64 %0, %0, %1;\n\t}"
                    : "+d"(fut)
                    : "d"(a), "r"(take));
                win >>= in;
            }
            gi_keep(__dadd_rn(double(int(c[q]) - 1), __dmul_rn(alpha, fut)), q, best_s, best_q);
        }
        return make_double2(best_s, __int_as_double_lo(best_q));
    }

    // K = 1 when the chunk fits one candidate per thread (no idle chains)
    static __device__ __noinline__ double2 gi_dense_chunk(const u32* ks, const u16* c, int m_, int q_lo, int q_hi,
                                                          u32 c0, double alpha, double best_s, int best_q) {
        if (q_hi - q_lo <= NT)
            return gi_dense_chunk_k<1>(ks, c, m_, q_lo, q_hi, c0, alpha, best_s, best_q);
        return gi_dense_chunk_k<3>(ks, c, m_, q_lo, q_hi, c0, alpha, best_s, best_q);
    }

    // Approximate gi score of candidate q from the per-variable candidate
    // bitmaps: q's intersecting candidates in canonical order are the set bits
    // of bm[qi] | bm[qj] minus q itself, so the pass is O(m/32 + deg q) instead
    // of O(m); the k-th of them takes coin k (64-bit window: at most 64 coins
    // per candidate on this path).  Exact integer sums packed I << 16 | C, as
    // in gi_pass; near-best bookkeeping as in the walk's approximate pass.
    __device__ __forceinline__ void gi_score_bm(int q, u32 c0, u32 T, double alpha, double beta, double eps2,
                                                double& lb, int& q1, double& h1, int& q2, double& h2, bool& ovf) {
        const u32* ks = keys();
        const u16* c = cnts();
        const u32* coin = sp<u32>(lay.coin);
        const u32 kq = ks[q];
        const int nwl = int(bm_stride(mcap));
        const u32* bi = sp<u32>(lay.bm) + key_i(kq) * nwl;
        const u32* bj = sp<u32>(lay.bm) + key_j(kq) * nwl;
        const u32* hv0 = sp<u32>(lay.bm);  // row 0: heavy candidates (c >= 3)
        const u32 p = sp<u32>(lay.qbase)[q] - c0;
        const u32 w0 = coin[p >> 5], w1 = coin[(p >> 5) + 1], w2 = coin[(p >> 5) + 2];
        // q's coins: bit k decides its k-th intersecting candidate
        u64 win = (u64(__funnelshift_r(w1, w2, p & 31u)) << 32) | __funnelshift_r(w0, w1, p & 31u);
        // per word of the list: the n intersecting candidates there take the
        // window's next n coins; weight-1 candidates (c = 2, the common
        // case) count by popcount, only heavy ones are visited one by one
        u32 I = 0u, C = 0u;
        const int nwm = (m + 31) >> 5;
#pragma unroll 1
        for (int wd = 0; wd < nwm; ++wd) {
            u32 msk = bi[wd] | bj[wd];
            if (wd == (q >> 5))
                msk &= ~(1u << (q & 31));
            if (msk == 0u)
                continue;
            const int n = __popc(msk);
            const u32 sel = u32(win) & (0xffffffffu >> (32 - n));  // coins of these n, in order
            I += u32(n);
            C += u32(__popc(sel));
            u32 hv = msk & hv0[wd];
            while (hv) {
                const int b = __ffs(hv) - 1;
                hv &= hv - 1;
                const u32 x = u32(c[(wd << 5) + b]) - 2u;  // weight beyond 1
                I += x;
                C += ((sel >> __popc(msk & ((1u << b) - 1u))) & 1u) ? x : 0u;
            }
            win >>= n;
        }
        const u32 wq = u32(c[q]) - 1u;
        const double F = __dadd_rn(double(T - wq - I), __dmul_rn(beta, double(C)));
        const double h = __dadd_rn(double(wq), __dmul_rn(alpha, F));
        lb = fmax(lb, h);
        const double lim = __dsub_rn(lb, eps2);
        if (q1 >= 0 && h1 < lim)
            q1 = -1;
        if (q2 >= 0 && h2 < lim)
            q2 = -1;
        if (h >= lim) {
            if (q1 < 0) {
                q1 = q;
                h1 = h;
            } else if (q2 < 0) {
                q2 = q;
                h2 = h;
            } else {
                ovf = true;
            }
        }
    }

    // Approximate gi scores of candidates q0, q0 + NT, ..., q0 + (K-1) NT
    // (< q_hi): exact integer sums over the list, packed A = I << 16 | C with
    // I = intersecting weight, C = its coin-selected part (T < 2^16 on this
    // path).  A candidate's coins (at most 64 on this path) sit in a 64-bit
    // window consumed one bit per intersecting candidate.  Near-best
    // bookkeeping as in the walk's approximate pass.
    template <int K>
    __device__ __forceinline__ void gi_pass(int q0, int q_hi, u32 c0, u32 T, double alpha, double beta, double eps2,
                                            double& lb, int& q1, double& h1, int& q2, double& h2, bool& ovf) {
        const u32* ks = keys();
        const u16* c = cnts();
        const u32* qbase = sp<u32>(lay.qbase);
        const u32* coin = sp<u32>(lay.coin);
        int qv[K], qi[K], qj[K];
        u32 lo[K], hi[K], A[K];
#pragma unroll
        for (int t = 0; t < K; ++t) {
            qv[t] = q0 + t * NT;
            const bool on = qv[t] < q_hi;
            const u32 kq = on ? ks[qv[t]] : 0u;
            qi[t] = on ? key_i(kq) : -1;  // -1 never matches a variable
            qj[t] = on ? key_j(kq) : -1;
            const u32 p = on ? qbase[qv[t]] - c0 : 0u;
            const u32 w0 = coin[p >> 5], w1 = coin[(p >> 5) + 1], w2 = coin[(p >> 5) + 2];
            lo[t] = __funnelshift_r(w0, w1, p & 31u);
            hi[t] = __funnelshift_r(w1, w2, p & 31u);
            A[t] = 0u;
        }
        const int m_ = m;
#pragma unroll 2
        for (int s = 0; s < m_; ++s) {
            const u32 kk = ks[s];
            const int si = key_i(kk), sj = key_j(kk);
            const u32 w = u32(c[s]) - 1u;
            const u32 wI = w << 16, wC = wI | w;
#pragma unroll
            for (int t = 0; t < K; ++t) {
                const bool inter = (s != qv[t]) & ((si == qi[t]) | (si == qj[t]) | (sj == qi[t]) | (sj == qj[t]));
                if (inter) {
                    A[t] += (lo[t] & 1u) ? wC : wI;
                    lo[t] = __funnelshift_r(lo[t], hi[t], 1);
                    hi[t] >>= 1;
                }
            }
        }
#pragma unroll
        for (int t = 0; t < K; ++t) {
            if (qv[t] >= q_hi)
                continue;
            const u32 wq = u32(c[qv[t]]) - 1u;
            const double F = __dadd_rn(double(T - wq - (A[t] >> 16)), __dmul_rn(beta, double(A[t] & 0xffffu)));
            const double h = __dadd_rn(double(wq), __dmul_rn(alpha, F));
            lb = fmax(lb, h);
            const double lim = __dsub_rn(lb, eps2);
            if (q1 >= 0 && h1 < lim)
                q1 = -1;
            if (q2 >= 0 && h2 < lim)
                q2 = -1;
            if (h >= lim) {
                if (q1 < 0) {
                    q1 = qv[t];
                    h1 = h;
                } else if (q2 < 0) {
                    q2 = qv[t];
                    h2 = h;
                } else {
                    ovf = true;
                }
            }
        }
    }

    // exact gi score of q (score_intersections_from's sequential sum) on the
    // dense layout, by one whole warp: q's intersecting candidates come from
    // ballots over the list in canonical order, runs of disjoint candidates
    // are added in O(1) by add_run.  Warp-uniform q, result on every lane.
    static __device__ __noinline__ double gi_fold_dense(const u32* ks, const u16* c, int m_, int q, u32 c0,
                                                       double alpha, double topmin) {
        const u32* coin = sp<u32>(lay.coin);
        const u32* wp = sp<u32>(lay.wp);
        const double* wbt = sp<double>(lay.wbt);
        const int lane = int(threadIdx.x & 31);
        const u32 kq = ks[q];
        const int qi = key_i(kq), qj = key_j(kq);
        u32 ptr = sp<u32>(lay.qbase)[q] - c0;
        double f = 0.0;
        int prev = 0;
        for (int base = 0; base < m_; base += 32) {
            const int s = base + lane;
            bool hit = false;
            if (s < m_) {
                const u32 kk = ks[s];
                const int si = key_i(kk), sj = key_j(kk);
                hit = (si == qi) | (si == qj) | (sj == qi) | (sj == qj);  // q itself included
            }
            u32 msk = __ballot_sync(FULLMASK, hit);
            while (msk) {
                const int s2 = base + __ffs(msk) - 1;
                msk &= msk - 1;
                f = add_run(f, prev, s2, wp, topmin);
                prev = s2 + 1;
                if (s2 != q) {
                    if ((coin[ptr >> 5] >> (ptr & 31u)) & 1u)
                        f = __dadd_rn(f, wbt[c[s2]]);
                    ++ptr;
                }
            }
        }
        f = add_run(f, prev, m_, wp, topmin);
        return __dadd_rn(double(int(c[q]) - 1), __dmul_rn(alpha, f));
    }

    __device__ __forceinline__ static void gi_keep(double h, int q, double& best_s, int& best_q) {
        if (h > best_s || (h == best_s && q < best_q) || best_q == 0x7fffffff) {
            best_s = h;
            best_q = q;
        }
    }

    // gi pruning (dense and walk) in one barrier: B = max(B, block max of lb) and the
    // near-best count (ovf flags << 16 | candidates >= B - eps2).  Each warp
    // publishes its max, its count relative to its own max and the index of
    // its max; a warp whose max is B counts exactly, another warp within the
    // window counts as 1 (a lower bound: it holds at least its max).  So the
    // count is exact whenever it is <= 1 on a single chunk, the only case that
    // decides anything: then `lone` is the pick (the candidate scoring B).
    __device__ __forceinline__ u32 near_best(double lb, double eps2, int q1, double h1, int q2, double h2, bool ovf,
                                             double& B, int& lone) {
        double wm = lb;
        wm = fmax(wm, __shfl_xor_sync(FULLMASK, wm, 16));
        wm = fmax(wm, __shfl_xor_sync(FULLMASK, wm, 8));
        wm = fmax(wm, __shfl_xor_sync(FULLMASK, wm, 4));
        wm = fmax(wm, __shfl_xor_sync(FULLMASK, wm, 2));
        wm = fmax(wm, __shfl_xor_sync(FULLMASK, wm, 1));
        const double wthr = __dsub_rn(wm, eps2);
        u32 wi = (ovf ? 0x1000000u : 0u) + (u32(q1 >= 0 && h1 >= wthr) + u32(q2 >= 0 && h2 >= wthr)) * 0x10000u;
        wi = __reduce_add_sync(FULLMASK, wi);
        const u32 qm = lb != wm ? 0xffffu : (q1 >= 0 && h1 == lb ? u32(q1) : (q2 >= 0 && h2 == lb ? u32(q2) : 0xffffu));
        wi |= __reduce_min_sync(FULLMASK, qm);
        if (NW == 1) {
            B = fmax(B, wm);
            lone = int(wi & 0xffffu);
            return ((wi >> 24) << 16) | ((wi >> 16) & 0xffu);
        }
        rsel ^= 1;
        double* r = g_reds + rsel * NW;
        u32* ri = reinterpret_cast<u32*>(g_redi + rsel * NW);
        if (lane == 0) {
            r[tid >> 5] = wm;
            ri[tid >> 5] = wi;
        }
        __syncthreads();
        double cm = r[0];
#pragma unroll
        for (int w = 1; w < NW; ++w)
            cm = fmax(cm, r[w]);
        B = fmax(B, cm);
        const double thr = __dsub_rn(B, eps2);
        u32 info = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const double x = r[w];
            const u32 y = ri[w];
            info += ((y >> 24) << 16) + (x >= thr ? (x == B ? ((y >> 16) & 0xffu) : 1u) : 0u);
            if (x == B)
                lone = int(y & 0xffffu);
        }
        return info;
    }

    // Candidate q's intersecting candidates in canonical order: the merge of
    // variable qi's and qj's lists (A list = candidates holding the variable
    // second, by index; then the contiguous run holding it first).  q itself
    // and its opposite-sign twin appear in both and are visited once.
    template <typename F>
    static __device__ __forceinline__ void gi_neighbours(const u32* ks, int q, F&& visit) {
        const u32 kq = ks[q];
        const int qi = key_i(kq), qj = key_j(kq);
        const u32* aoff = sp<u32>(lay.aoff);
        const u32* nA = sp<u32>(lay.nA);
        const u32* nB = sp<u32>(lay.nB);
        const u32* bs = sp<u32>(lay.bs);
        const u16* alist = sp<u16>(lay.alist);
        const int ai = int(aoff[qi]), nai = int(nA[qi]), bi = int(bs[qi]), li = nai + int(nB[qi]);
        const int aj = int(aoff[qj]), naj = int(nA[qj]), bj = int(bs[qj]), lj = naj + int(nB[qj]);
        int pi = 0, pj = 0;
        for (;;) {
            const int xi = pi < li ? (pi < nai ? int(alist[ai + pi]) : bi + (pi - nai)) : 0x7fffffff;
            const int xj = pj < lj ? (pj < naj ? int(alist[aj + pj]) : bj + (pj - naj)) : 0x7fffffff;
            const int s = min(xi, xj);
            pi += xi == s;
            pj += xj == s;
            if (!visit(s))
                break;
        }
    }

    // approximate gi score of q: exact integer sums, three roundings
    static __device__ __forceinline__ double gi_approx(const u32* ks, const u16* c, int q, u32 c0, u32 T,
                                                       double alpha, double beta) {
        const u32* coin = sp<u32>(lay.coin);
        u32 ptr = sp<u32>(lay.qbase)[q] - c0;
        u32 I = 0, C = 0;
        gi_neighbours(ks, q, [&](int s) {
            if (s == 0x7fffffff)
                return false;
            if (s != q) {
                const u32 w = u32(c[s]) - 1u;
                I += w;
                C += ((coin[ptr >> 5] >> (ptr & 31u)) & 1u) ? w : 0u;
                ++ptr;
            }
            return true;
        });
        const u32 wq = u32(c[q]) - 1u;
        const double F = __dadd_rn(double(T - wq - I), __dmul_rn(beta, double(C)));
        return __dadd_rn(double(wq), __dmul_rn(alpha, F));
    }

    static __device__ __noinline__ double2 gi_rescan(const u32* ks, const u16* c, int m_, int q_lo, int q_hi, u32 c0,
                                                     u32 T, double alpha, double beta, double topmin, double thr,
                                                     double best_s, int best_q) {
        for (int q = q_lo + int(threadIdx.x); q < q_hi; q += NT)
            if (gi_approx(ks, c, q, c0, T, alpha, beta) >= thr)
                gi_keep(gi_fold(ks, c, m_, q, c0, alpha, topmin), q, best_s, best_q);
        return make_double2(best_s, __int_as_double_lo(best_q));
    }

    // exact gi score of q: score_intersections_from's sequential sum, runs of
    // disjoint candidates added in O(1) by add_run
    static __device__ __noinline__ double gi_fold(const u32* ks, const u16* c, int m_, int q, u32 c0, double alpha,
                                                  double topmin) {
        const u32* coin = sp<u32>(lay.coin);
        const u32* wp = sp<u32>(lay.wp);
        const double* wbt = sp<double>(lay.wbt);
        u32 ptr = sp<u32>(lay.qbase)[q] - c0;
        double f = 0.0;
        int prev = 0;
        gi_neighbours(ks, q, [&](int s) {
            f = add_run(f, prev, s == 0x7fffffff ? m_ : s, wp, topmin);
            if (s == 0x7fffffff)
                return false;
            prev = s + 1;
            if (s != q) {
                if ((coin[ptr >> 5] >> (ptr & 31u)) & 1u)
                    f = __dadd_rn(f, wbt[c[s]]);
                ++ptr;
            }
            return true;
        });
        return __dadd_rn(double(int(c[q]) - 1), __dmul_rn(alpha, f));
    }

    // Sequential double sum f + w_L + ... + w_{R-1} (w_t = c_t - 1 >= 1,
    // wp = exclusive prefix sums, f >= 0), bit-identical to adding one at a
    // time: integer additions are exact until the running sum crosses a
    // binade, where exactly one rounding happens.  Integers never change the
    // fraction of f and below 2^52 the tie bit is fractional, so the rounding
    // at a crossing depends only on the fraction and the new binade — not on
    // which element crosses — as long as no single element can skip a binade
    // (top >= topmin = max w + 1): then the crossing is done in O(1).  Below
    // that the crossing element is located by binary search in wp.
    static __device__ __forceinline__ double add_run(double f, int L, int R, const u32* wp, double topmin) {
        u32 tot = wp[R] - wp[L];
        while (tot != 0u) {
            if (f == trunc(f))
                return __dadd_rn(f, double(tot));  // integer + integer: exact
            const long long bits = __double_as_longlong(f);
            const double top = __longlong_as_double((long long)((((bits >> 52) & 0x7ff) + 1)) << 52);
            const double gap = __dsub_rn(top, f);  // exact (Sterbenz)
            if (double(tot) < gap)
                return __dadd_rn(f, double(tot));  // stays in the binade: exact
            u32 step;
            if (top >= topmin) {
                step = u32(ceil(gap));  // any crossing partial sum rounds alike
            } else {
                // first element whose partial sum reaches the binade top
                const u32 need = wp[L] + u32(ceil(gap));
                int lo = L + 1, hi = R;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (wp[mid] >= need)
                        hi = mid;
                    else
                        lo = mid + 1;
                }
                step = wp[lo] - wp[L];
                L = lo;
            }
            f = __dadd_rn(f, double(step));  // the one rounding
            tot -= step;
        }
        return f;
    }

    // select_greedy_potential (196-220), alpha != 0: (c-1) + alpha * created,
    // created = pairs with the trial variable k reaching frequency >= 2
    __device__ int sel_gp(double alpha) {
        const u32* ks = keys();
        const u16* c = cnts();
        double best_s = -INFINITY;
        int best_q = 0x7fffffff;
        for (int q = tid; q < m; q += NT) {
            const u32 kq = ks[q];
            const int qi = key_i(kq), qj = key_j(kq), neg = key_neg(kq);
            const u64* a = P(qi - 1);
            const u64* b = P(qj - 1);
            u64 rp[W], rn[W];
#pragma unroll
            for (int w = 0; w < W; ++w) {
                rp[w] = a[w] & (neg ? b[W + w] : b[w]);
                rn[w] = a[W + w] & (neg ? b[w] : b[W + w]);
            }
            int created = 0;
            for (int x = 1; x <= V; ++x) {
                if (x == qi || x == qj)
                    continue;
                const u64* px = P(x - 1);
                int cp = 0, cn = 0;
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    cp += __popcll(px[w] & rp[w]) + __popcll(px[W + w] & rn[w]);
                    cn += __popcll(px[w] & rn[w]) + __popcll(px[W + w] & rp[w]);
                }
                created += (cp >= 2) + (cn >= 2);
            }
            const double h = __dadd_rn(double(int(c[q]) - 1), __dmul_rn(alpha, double(created)));
            if (h > best_s || best_q == 0x7fffffff) {
                best_s = h;
                best_q = q;
            }
        }
        return argmax(best_s, best_q);
    }

    // pick_mixed_substrategy (236-258); weights validated on the host
    __device__ int mixed_sub(const double* mix) {
        double total = 0.0;
        int positive = 0, only = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (mix[k] > 0.0) {
                ++positive;
                only = k;
            }
            total = __dadd_rn(total, mix[k]);
        }
        int pick = 3;
        if (positive == 1) {
            pick = only;
        } else {
            double target = __dmul_rn(uniform_real(draw(), 0.0, 1.0), total);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                target = __dsub_rn(target, mix[k]);
                if (target < 0.0) {
                    pick = k;
                    break;
                }
            }
        }
        return pick == 0 ? TCSE_GREEDY_INTERSECTIONS
                         : (pick == 1 ? TCSE_GREEDY_ALTERNATIVE : (pick == 2 ? TCSE_GREEDY_RANDOM : TCSE_WEIGHTED_RANDOM));
    }

    int sd_ne;
    int gi_bm;     // dense layout carries per-variable candidate bitmaps
    int gi_prune;  // 0: no pruning (test hook); dense layout: prune from this many candidates on
    int mcap;  // candidate capacity of the layout
};

// the system block `blk` belongs to (blocks are contiguous per system)
__device__ __forceinline__ const SysDesc& find_sys(const LaunchDesc& L, int blk) {
    if (L.table) {
        int lo = 0, hi = L.table_n - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (L.table[mid].block_begin <= blk)
                lo = mid;
            else
                hi = mid - 1;
        }
        return L.table[lo];
    }
    int s = 0;
#pragma unroll
    for (int t = 1; t < kMaxSys; ++t)
        if (t < L.nsys && blk >= L.sys[t].block_begin)
            s = t;
    return L.sys[s];
}

__device__ __forceinline__ void set_error(const SysDesc& sd, int code, int pos) {
    if (atomicCAS(sd.err, 0, code) == 0 && sd.err_pos)
        *sd.err_pos = pos;
}

// Register cap: resident processes per SM are bounded by registers before
// shared memory unless the kernel is held to ~64 registers at 128 threads.
#ifndef TCSE_MINB32
#define TCSE_MINB32 28
#endif
#ifndef TCSE_MINB64
#define TCSE_MINB64 14
#endif
#ifndef TCSE_MINB_SMALL
#define TCSE_MINB_SMALL TCSE_MINB32
#endif
template <int NT, bool SM>
struct MinBlocks {
    static constexpr int value =
        SM ? TCSE_MINB_SMALL : (NT == 32 ? TCSE_MINB32 : (NT == 64 ? TCSE_MINB64 : (NT == 128 ? 8 : 4)));
};

// ------------------------------------------------------ prefix snapshots
//
// A reinit process (parallel_search.hpp:242-248) replays the first k
// substitutions of the incumbent, k ~ U[1, 3 len / 4]; every such process of
// an iteration replays a prefix of the SAME record.  The launch's builder
// block (one per system, scheduled first) replays it once with the same
// apply / update code and publishes the state after each substitution; a
// reinit process copies the newest published state at or below its k from
// L2 and replays only the rest — the same state either way, so results do
// not depend on how far the builder got (nobody waits for it).

__device__ __forceinline__ u32 ld_acquire(const u32* p) {
    u32 v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(u32* p, u32 v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// the system's base state (masks of the n_x input variables, starting
// candidate list) into shared memory
template <int W, int NT>
__device__ __forceinline__ void load_base_impl(const SysDesc& sd, int tid) {
    // (descriptor fields in registers first: read through the descriptor
    // reference, every iteration would reload them behind the shared
    // stores, serialising the copy on the load latency)
    u64* mask = mask_base();
    const int nw = sd.n_x * 2 * W;
    const u64* __restrict__ gmask = sd.base_masks;
#pragma unroll 4
    for (int t = tid; t < nw; t += NT)
        mask[t] = __ldg(gmask + t);
    const u32* __restrict__ gkeys = sd.base_keys;
    const u16* __restrict__ gcnts = sd.base_cnts;
    const int bm = sd.base_m;
    if (gkeys) {
        u32* k0 = sp<u32>(lay.keys0);
        u16* c0 = sp<u16>(lay.cnts0);
#pragma unroll 4
        for (int t = tid; t < bm; t += NT) {
            k0[t] = __ldg(gkeys + t);
            c0[t] = __ldg(gcnts + t);
        }
    }
}

// one out-of-line copy for two-warp and wider blocks (fewer spills in the
// main loop: +1% on 4x4x4); one-warp blocks inline it (-1% out of line)
template <int W, int NT>
__device__ __noinline__ void load_base_ool(const SysDesc& sd, int tid) {
    load_base_impl<W, NT>(sd, tid);
}

template <int W, int NT>
__device__ __forceinline__ void load_base(const SysDesc& sd, int tid) {
    if constexpr (NT >= 64)
        load_base_ool<W, NT>(sd, tid);
    else
        load_base_impl<W, NT>(sd, tid);
}

// snapshot k (1-based) of the state in shared memory: (V, m, cost) header,
// V mask rows, the list
template <int W, int NT>
__device__ __noinline__ void snap_store(const SysDesc& sd, int k, int V, int m, int cost) {
    const int tid = threadIdx.x;
    unsigned char* base = sd.snap + size_t(k - 1) * size_t(sd.snap_stride);
    if (tid == 0)
        *reinterpret_cast<int4*>(base) = make_int4(V, m, cost, 0);
    const u64* mask = mask_base();
    u64* gm = reinterpret_cast<u64*>(base + 16);
    for (int t = tid; t < V * 2 * W; t += NT)
        gm[t] = mask[t];
    const u32* ks = sp<u32>(lay.keys0);
    const u16* cs = sp<u16>(lay.cnts0);
    u32* gk = reinterpret_cast<u32*>(base + sd.snap_koff);
    u16* gc = reinterpret_cast<u16*>(base + sd.snap_coff);
    for (int t = tid; t < m; t += NT) {
        gk[t] = ks[t];
        gc[t] = cs[t];
    }
}

// snapshot k into shared memory (L2 reads: the lines may be stale in L1
// from an earlier iteration); returns (V, m, cost)
template <int W, int NT>
__device__ __noinline__ int4 snap_load(const SysDesc& sd, int k) {
    const int tid = threadIdx.x;
    const unsigned char* base = sd.snap + size_t(k - 1) * size_t(sd.snap_stride);
    const int4 h = __ldcg(reinterpret_cast<const int4*>(base));
    u64* mask = mask_base();
    const u64* gm = reinterpret_cast<const u64*>(base + 16);
    for (int t = tid; t < h.x * 2 * W; t += NT)
        mask[t] = __ldcg(gm + t);
    u32* ks = sp<u32>(lay.keys0);
    u16* cs = sp<u16>(lay.cnts0);
    const u32* gk = reinterpret_cast<const u32*>(base + sd.snap_koff);
    const u16* gc = reinterpret_cast<const u16*>(base + sd.snap_coff);
    for (int t = tid; t < h.y; t += NT) {
        ks[t] = __ldcg(gk + t);
        cs[t] = __ldcg(gc + t);
    }
    return h;
}

template <int W, int NT>
struct St;

// the builder block of sys: replays the incumbent's first 3 len / 4
// substitutions (the longest prefix a reinit process draws) and publishes
// each state.  Same conditions as prep_slot's reinit flag; a prefix the
// processes could not replay (capacity, bad pair) is simply not published —
// the processes replay it themselves and report exactly as without snapshots.
template <int W, int NT>
__device__ __noinline__ void build_snapshots(const SysDesc& sd) {
    const int tid = threadIdx.x;
    const IncState* I = sd.loop;
    if (!sd.snap || !I || !sd.reinit || !I->active || *sd.err != 0)
        return;
    const int len = I->len;
    const int K = min(3 * len / 4, sd.snap_k);
    if (len < 2 || K < 1)
        return;
    if (tid == 0)
        carve(&lay, W, NT, sd.vcap, sd.mcap, sd.n_e, sd.coin_words, sd.gi_dense, sd.gi_bm);
    __syncthreads();
    load_base<W, NT>(sd, tid);
    __syncthreads();
    St<W, NT> pr;
    pr.tid = tid;
    pr.lane = tid & 31;
    pr.V = sd.n_x;
    pr.cost = sd.naive;
    pr.m = sd.base_m;
    pr.mti = 312;
    pr.rsel = 0;
    pr.last_coins = 0;
    pr.sd_ne = sd.n_e;
    pr.gi_prune = sd.gi_prune;
    pr.gi_bm = sd.gi_bm;
    pr.mcap = sd.mcap;
    for (int k = 1; k <= K; ++k) {
        const u32 q = sd.inc_keys[k - 1];
        const int qi = key_i(q), qj = key_j(q);
        if (qi < 1 || qj <= qi || qj > pr.V || pr.apply(q) == 0 || !pr.update(q))
            return;
        snap_store<W, NT>(sd, k, pr.V, pr.m, pr.cost);
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            st_release(sd.snap_ready, u32(k));
        }
    }
}

template <int W, int NT, bool GID, int F>
__global__ void __launch_bounds__(NT, (MinBlocks<NT, (F & kFormSmall) != 0>::value))
    search_kernel(const __grid_constant__ LaunchDesc L) {
    if (int(blockIdx.x) < L.n_builders) {
        build_snapshots<W, NT>(L.sys[blockIdx.x]);
        return;
    }
    // launch order -> process block: blocks of one strategy run together, most
    // expensive strategies first (instruction-cache locality, shorter tail)
    const int bx = int(blockIdx.x) - L.n_builders;
    const int blk = L.perm ? L.perm[bx] : bx;
    const SysDesc& sd = find_sys(L, blk);
    const int lp = blk - sd.block_begin;
    if (lp >= sd.n_local)
        return;
    const int tid = threadIdx.x;

    // ---- process configuration (prep_kernel) + base state (all threads)
    __shared__ SlotRec s_slot;
    if (tid == 0) {
        carve(&lay, W, NT, sd.vcap, sd.mcap, sd.n_e, sd.coin_words, sd.gi_dense, sd.gi_bm);
        s_slot = L.slots[blk];
    }
    __syncthreads();
    // a reinit process with snapshots loads its state once it knows its
    // prefix length (below)
    const bool snap = sd.snap && sd.base_keys && s_slot.reinit;
    {
        if (!snap)
            load_base<W, NT>(sd, tid);
        if (s_slot.rng && !L.rng) {
            // seed the process's mt19937_64 in shared memory (one thread, while
            // the others load the base state): no HBM hand-off
            if (tid == 0)
                mt_seed_smem(stream_seed(sd, s_slot.seed));
        } else if (s_slot.rng && tid < kCkpt) {
            // 32 checkpoints of the seeding chain (256 B from HBM per process):
            // lane c restarts the chain at word 10c and fills words 10c..10c+9
            u64* mt = g_mt;
            u64 x = __ldg(L.rng + size_t(blk) * kCkpt + size_t(tid));
            const int i0 = tid * kCkptStride;
            mt[i0] = x;
#pragma unroll
            for (int j = 1; j < kCkptStride; ++j) {
                if (i0 + j >= 312)
                    break;
                x = kMtF * (x ^ (x >> 62)) + u64(i0 + j);
                mt[i0 + j] = x;
            }
        }
    }
    __syncthreads();
    const int strategy = s_slot.strategy;
    if (strategy < 0)  // converged system or failed launch (prep_kernel)
        return;
    if (tid == 0 && L.clock)
        atomicMin(&L.clock->gstart[L.group], globaltimer());
    const int reinit = s_slot.reinit;
    const double alpha = s_slot.alpha, beta = s_slot.beta, p_greedy = s_slot.p_greedy;
    const double* s_mix = s_slot.mix;

    St<W, NT> pr;
    pr.tid = tid;
    pr.lane = tid & 31;
    pr.V = sd.n_x;
    pr.cost = sd.naive;
    pr.mti = 312;
    pr.rsel = 0;
    pr.last_coins = 0;
    pr.sd_ne = sd.n_e;
    pr.gi_prune = sd.gi_prune;
    pr.gi_bm = sd.gi_bm;
    pr.mcap = sd.mcap;
    if (sd.base_keys) {
        pr.m = sd.base_m;
    } else {
        pr.m = all_pairs<W, NT>(pr.V, 2, sp<u32>(lay.keys0), sp<u16>(lay.cnts0), sd.mcap, 0);
        if (pr.m > sd.mcap) {
            set_error(sd, TCSE_ECAPACITY, pr.m);
            return;
        }
    }

    // ---- prefix: reinit from the incumbent (parallel_search.hpp:242-248) or a
    // fixed replay (cse_engine.hpp:47-57); replayed through the same
    // apply/update path as the selected substitutions
    const u32* pre = nullptr;
    int n_pre = 0;
    if (reinit) {
        const u64 k_max = u64(3 * reinit / 4);  // reinit = incumbent length
        n_pre = int(1 + pr.nd(k_max));
        pre = sd.inc_keys;
    } else if (sd.mode != kModeSearch && sd.prefix_len > 0) {
        n_pre = sd.prefix_len;
        pre = sd.prefix;
    }
    const bool rec_prefix = reinit != 0;  // records carry the prefix in search mode
    // cold per-process values (two-warp and wider blocks) live in shared
    // memory, not in the main loop's registers: the record row and the trace
    // hook (thread 0 only; round 2 also took the word-op counter there: +3% on 4x4x4, +3% on
    // 5x5x5; one-warp blocks keep them in registers: -2% there, and so do
    // 256-thread blocks: -0.5% on 6x6x6).  The slot's alpha / beta / p_greedy
    // read from shared memory at each use instead: -3% (more spills).
    constexpr bool kCold = NT >= TCSE_COLD_MIN && NT <= 128;
    __shared__ u32* s_rec;
    __shared__ u64* s_trace;
    __shared__ int s_step;
    u32* rec = nullptr;
    int step = 0;
    u64 wops = 0;
    if (kCold) {
        if (tid == 0) {
            s_rec = sd.out_subs ? sd.out_subs + size_t(lp) * size_t(sd.sub_cap) : nullptr;
            s_trace = sd.trace ? sd.trace + size_t(lp) * size_t(sd.trace_stride) : nullptr;
            s_step = 0;
        }
        __syncthreads();
    } else {
        rec = sd.out_subs ? sd.out_subs + size_t(lp) * size_t(sd.sub_cap) : nullptr;
    }
#define TCSE_REC (kCold ? s_rec : rec)
    const bool dump = sd.mode == kModeDump;
    int n_rec = 0;
    int t_pre0 = 0;
    if (snap) {
        // the newest published snapshot at or below n_pre (or the base state)
        __shared__ int s_k;
        if (tid == 0)
            s_k = min(n_pre, int(ld_acquire(sd.snap_ready)));
        __syncthreads();
        t_pre0 = s_k;
        SNAP_STAT(0, 1);
        SNAP_STAT(1, t_pre0 == n_pre);
        SNAP_STAT(2, t_pre0 == 0);
        SNAP_STAT(3, n_pre);
        SNAP_STAT(4, n_pre - t_pre0);
        if (t_pre0 > 0) {
            const int4 h = snap_load<W, NT>(sd, t_pre0);
            pr.V = h.x;
            pr.m = h.y;
            pr.cost = h.z;
            if (sd.out_subs)  // the record carries the prefix
                for (int t = tid; t < t_pre0; t += NT)
                    TCSE_REC[t] = pre[t];
            n_rec = t_pre0;
        } else {
            load_base<W, NT>(sd, tid);
        }
        __syncthreads();
    }
    // prefix replay (reinit from the incumbent, or a fixed replay): apply +
    // update only, its own loop so the search loop carries no prefix state
    for (int t_pre = t_pre0; t_pre < n_pre; ++t_pre) {
        const u32 q = pre[t_pre];
        const int qi = key_i(q), qj = key_j(q);
        if (qi < 1 || qj <= qi || qj > pr.V || pr.apply(q) == 0) {
            set_error(sd, TCSE_EREPLAY, t_pre);
            if (tid == 0 && sd.out_cost)
                sd.out_cost[lp] = -1;
            return;
        }
        if (!pr.update(q)) {
            set_error(sd, kErrCandOverflow, pr.m);
            return;
        }
        if (rec_prefix) {
            if (tid == 0 && n_rec < sd.sub_cap)
                TCSE_REC[n_rec] = q;
            ++n_rec;
            if (n_rec > sd.sub_cap) {
                set_error(sd, TCSE_ECAPACITY, n_rec);
                return;
            }
        }
    }
    const int n_rec0 = n_rec;  // steps selected by this process = n_rec - n_rec0
    const int sub_cap = sd.sub_cap;
    const int V0 = pr.V;  // V grows by one per selected step
    // word-ops per step: recount 12 (V - 1) W_E +
    // substitution 8 W_E + selection (m, + coins for gi, + m (V - 2) 4 W_E
    // for gp); the V terms are summed in closed form after the loop, the
    // list sizes and coins here, gp's rare term in shared memory
    u32 msum = 0;
    __shared__ u64 s_gpw;
    if (tid == 0)
        s_gpw = 0;
    while (!dump) {
        if (kCold) {
            if (sd.trace) {  // parity hook only
                if (tid == 0) {
                    if (s_step < sd.trace_stride)
                        s_trace[s_step] = cand_hash(pr.keys(), pr.cnts(), pr.m);
                    ++s_step;
                }
            }
        } else if (sd.trace) {  // parity hook only
            if (tid == 0 && step < sd.trace_stride)
                sd.trace[size_t(lp) * size_t(sd.trace_stride) + size_t(step)] = cand_hash(pr.keys(), pr.cnts(), pr.m);
            ++step;
        }
        if (pr.m == 0)
            break;
        int strat = strategy;
        if (strat == TCSE_MIXED)
            strat = pr.mixed_sub(s_mix);  // select_mixed (strategies.hpp:260-269)
        if (strat == TCSE_GREEDY_RANDOM)  // select_greedy_random (119-124)
            strat = uniform_real(pr.draw(), 0.0, 1.0) < p_greedy ? TCSE_GREEDY_ALTERNATIVE : TCSE_WEIGHTED_RANDOM;
        if ((strat == TCSE_GREEDY_INTERSECTIONS || strat == TCSE_GREEDY_POTENTIAL) && alpha == 0.0)
            strat = TCSE_GREEDY;  // gain only (strategies.hpp:140-141, 205-206)
        msum += u32(pr.m);
        int pick;
#if TCSE_ONLY_GI  // experiment: a Greedy-Intersections-only kernel (code size / registers)
        if (true) {
            pick = pr.template sel_gi<GID, F>(alpha, beta);
            msum += pr.last_coins;
        } else
#endif
        if (strat == TCSE_GREEDY) {
            pick = pr.sel_greedy();
        } else if (strat == TCSE_GREEDY_ALTERNATIVE) {
            pick = pr.sel_ga();
        } else if (strat == TCSE_WEIGHTED_RANDOM) {
            pick = pr.sel_wr();
        } else if (strat == TCSE_GREEDY_INTERSECTIONS) {
            pick = pr.template sel_gi<GID, F>(alpha, beta);
            msum += pr.last_coins;
        } else {
            if (tid == 0)
                s_gpw += u64(pr.m) * u64(pr.V - 2) * 4 * u64(sd.words);
            pick = pr.sel_gp(alpha);
        }
        const u32 q = pr.keys()[pick];
        pr.apply(q);  // a selected candidate always occurs (c >= 2)
        if (!pr.update(q)) {
            set_error(sd, kErrCandOverflow, pr.m);
            return;
        }
        if (n_rec >= sub_cap) {  // the record would outgrow its row
            set_error(sd, TCSE_ECAPACITY, n_rec + 1);
            return;
        }
        if (tid == 0)
            TCSE_REC[n_rec] = q;
        ++n_rec;
    }
    {
        const u64 S = u64(n_rec - n_rec0), we = u64(sd.words);
        wops = we * (12 * (S * u64(V0 - 1) + S * (S - 1) / 2) + 8 * S) + msum + s_gpw;
    }
#undef TCSE_REC

    if (dump) {
        if (sd.dump_min_count >= 2) {
            const u32* ks = pr.keys();
            const u16* cs = pr.cnts();
            for (int t = tid; t < pr.m && t < sd.dump_cap; t += NT) {
                sd.dump_keys[t] = ks[t];
                sd.dump_cnts[t] = cs[t];
            }
            if (tid == 0)
                *sd.dump_n = pr.m;
        } else {
            const int n = all_pairs<W, NT>(pr.V, sd.dump_min_count, sd.dump_keys, sd.dump_cnts, sd.dump_cap,
                                           pr.rsel);
            if (tid == 0)
                *sd.dump_n = n;
        }
        return;
    }
    if (tid == 0) {
        sd.out_cost[lp] = pr.cost;
        sd.out_len[lp] = n_rec;
        sd.out_own[lp] = n_rec - n_rec0;
        sd.out_strategy[lp] = strategy;
        sd.out_seed[lp] = s_slot.seed;
        if (sd.out_wops)
            sd.out_wops[lp] = wops;
        if (L.clock)
            atomicMax(&L.clock->gend[L.group], globaltimer());
    }
}

// ------------------------------------------------------------------ K0

// One thread per process: assign_strategies' slot (parallel_search.hpp:
// 183-205) or the explicit ProcessConfig, the reinit flag, and — when the
// process will draw — its seeded mt19937_64 state (the 311-step sequential
// seeding runs here with full-GPU parallelism instead of serially at the
// start of every search block).
struct PrepOut {
    int sys;      // system index in the launch (placement histogram)
    int st;       // strategy, -1 = nothing to place (no process / skipped)
    int reinit;   // incumbent length when the process restarts from a prefix
    bool seed;    // the process draws: seed its stream
    u64 ps;       // stream seed
};

__device__ __forceinline__ PrepOut prep_slot(const LaunchDesc& L, int b) {
    PrepOut o;
    o.sys = 0;
    o.st = -1;
    o.reinit = 0;
    o.seed = false;
    o.ps = 0;
    if (b >= L.total_blocks)
        return o;
#pragma unroll
    for (int t = 1; t < kMaxSys; ++t)
        if (t < L.nsys && b >= L.sys[t].block_begin)
            o.sys = t;
    const SysDesc& sd = find_sys(L, b);
    const int lp = b - sd.block_begin;
    if (lp >= sd.n_local)
        return o;
    // the iteration and the incumbent length: from the device loop state in a
    // session (graph replays need no host parameters), else from the descriptor
    int iteration = sd.iteration, inc_len = sd.inc_len;
    if (sd.loop) {
        if (!sd.loop->active || *sd.err != 0) {  // converged system, or the launch already failed
            L.slots[b].strategy = -1;
            o.st = 7;  // placed last (strategy slot 7 is unused)
            return o;
        }
        iteration = sd.loop->iteration + 1;
        inc_len = sd.loop->len;
    }
    SlotRec r;
    Slot sl;
    if (sd.mode == kModeSearch) {
        derive_slot(sd, iteration, u64(sd.p0) + u64(lp) * u64(max(sd.p_stride, 1)), &sl);
        for (int k = 0; k < 4; ++k)
            r.mix[k] = sd.mix[k];
    } else if (sd.mode == kModeRun) {
        const tcse_process_config& c = sd.cfgs[lp];
        sl.strategy = c.strategy;
        sl.alpha = c.alpha;
        sl.beta = c.beta;
        sl.p_greedy = c.p_greedy;
        sl.seed = c.seed;
        for (int k = 0; k < 4; ++k)
            r.mix[k] = c.mix_weights[k];
    } else {
        sl.strategy = TCSE_GREEDY;
        sl.alpha = sl.beta = sl.p_greedy = 0.0;
        sl.seed = 0;
        for (int k = 0; k < 4; ++k)
            r.mix[k] = 0.0;
    }
    const int reinit = (sd.mode == kModeSearch && sd.reinit && sd.reinit[lp] && inc_len >= 2) ? 1 : 0;
    const int st = sl.strategy;
    const bool rng = reinit || st == TCSE_GREEDY_ALTERNATIVE || st == TCSE_WEIGHTED_RANDOM ||
                     st == TCSE_GREEDY_RANDOM || st == TCSE_MIXED ||
                     (st == TCSE_GREEDY_INTERSECTIONS && sl.alpha != 0.0);
    r.strategy = st;
    r.reinit = reinit ? inc_len : 0;
    r.rng = rng ? 1 : 0;
    r.pad = 0;
    r.alpha = sl.alpha;
    r.beta = sl.beta;
    r.p_greedy = sl.p_greedy;
    r.seed = sl.seed;
    L.slots[b] = r;
    o.st = st;
    o.reinit = r.reinit;
    o.seed = rng;
    o.ps = stream_seed(sd, sl.seed);
    return o;
}

// One thread per process: assign_strategies' slot (parallel_search.hpp:
// 183-205) or the explicit ProcessConfig, the reinit flag, and — when the
// process will draw and the launch hands states off through HBM — 32
// checkpoints of its mt19937_64 seeding chain (words 0, 10, ..., 310).  The
// 311-step sequential chain runs here with full-GPU parallelism; the search
// block rebuilds the 312-word state from the checkpoints with 32 lanes of
// 9 steps each, so neither side has the whole chain on its critical path and
// the hand-off is 256 B per process instead of 2.5 KB.  The checkpoints
// leave through a shared-memory tile, 8 per process per round, so each warp
// store covers whole 64-byte runs.
constexpr int kPrepNT = 128;
constexpr int kSeedChunk = 8;  // 312 = 39 x 8

__global__ void __launch_bounds__(kPrepNT) prep_kernel(const __grid_constant__ LaunchDesc L) {
    const int b = int(blockIdx.x * blockDim.x + threadIdx.x);
    const int tid = threadIdx.x;
    if (b == 0 && L.clock && L.group == 0 && L.clock->t_begin == 0)
        L.clock->t_begin = globaltimer();  // the search's first launch
    if (b < L.nsys && L.sys[b].snap_ready)
        *L.sys[b].snap_ready = 0u;  // no snapshot of this iteration yet (search launch follows on the stream)
    const PrepOut o = prep_slot(L, b);
    u64 x0 = 0, x1 = 0, x156 = 0;  // for the first output (work class below)
    if (L.rng) {
        __shared__ u64 tile[kPrepNT][kSeedChunk + 1];
        __shared__ unsigned char s_seed[kPrepNT];
        const int b0 = int(blockIdx.x * blockDim.x);
        s_seed[tid] = o.seed ? 1 : 0;
        if (__syncthreads_or(o.seed)) {
            u64 x = o.ps;
            x0 = x;
            u64 x150 = 0;
            // (the chain in unrolled 10-step segments between checkpoints:
            // one thread per process at one warp per SM sub-partition, so
            // the kernel's time is this chain's instruction count)
#pragma unroll 1
            for (int r0 = 0; r0 < kCkpt; r0 += kSeedChunk) {
#pragma unroll 1
                for (int k = 0; k < kSeedChunk; ++k) {
                    const int c = r0 + k;  // checkpoint c = state word c * kCkptStride
                    if (c > 0) {
                        const u64 i0 = u64((c - 1) * kCkptStride);
#pragma unroll
                        for (int j = 1; j <= kCkptStride; ++j)
                            x = kMtF * (x ^ (x >> 62)) + (i0 + u64(j));
                    }
                    if (c == 15)
                        x150 = x;
                    tile[tid][k] = x;
                }
                __syncthreads();
                // thread tid writes checkpoint (tid % 8) of process rr * 16 + tid / 8
#pragma unroll
                for (int rr = 0; rr < kSeedChunk; ++rr) {
                    const int p = rr * (kPrepNT / kSeedChunk) + tid / kSeedChunk, k = tid % kSeedChunk;
                    if (s_seed[p])
                        L.rng[size_t(b0 + p) * kCkpt + size_t(r0 + k)] = tile[p][k];
                }
                __syncthreads();
            }
            // state words 1 and 156 (the first output, work class below)
            x1 = kMtF * (x0 ^ (x0 >> 62)) + 1ULL;
            x156 = x150;
#pragma unroll
            for (int j = 151; j <= 156; ++j)
                x156 = kMtF * (x156 ^ (x156 >> 62)) + u64(j);
        }
    }
    if (L.hist) {
        // placement bucket (strategy, work class): fresh processes, then reinit
        // ones by the length of their replayed prefix (estimated from the
        // first output of their stream, ignoring the rare rejection: the
        // order never changes results).  Counted per block in shared memory
        // first: one global atomic per non-empty bucket and block instead of
        // one per process on a handful of addresses
        constexpr int kBuckets = 8 * kWorkClasses;
        __shared__ int s_h[kMaxSys * kBuckets];
        for (int t = tid; t < kMaxSys * kBuckets; t += kPrepNT)
            s_h[t] = 0;
        __syncthreads();
        if (o.st >= 0) {
            int cls = 0;
            if (o.reinit) {
                const u64 x = L.rng ? mt_temper(mt_mix(x0, x1, x156)) : mt_first_output(o.ps);
                const u64 n_pre = 1 + __umul64hi(x, u64(3 * o.reinit / 4));
                cls = 1 + min(3, int(4 * n_pre / u64(o.reinit + 1)));
            }
            if (o.st < 7)
                L.slots[b].pad = cls;
            atomicAdd(&s_h[o.sys * kBuckets + o.st + 8 * cls], 1);
        }
        __syncthreads();
        for (int t = tid; t < kMaxSys * kBuckets; t += kPrepNT)
            if (s_h[t])
                atomicAdd(&L.hist[(t / kBuckets) * kHistStride + (t % kBuckets)], s_h[t]);
    }
}

// launch position of every block: per system, strategies in the order
// gp, gi, mix, gr, ga, wr, g (roughly decreasing cost), any order within one
__global__ void __launch_bounds__(128) place_kernel(const __grid_constant__ LaunchDesc L) {
    constexpr int kBuckets = 8 * kWorkClasses;
    __shared__ int s_cnt[kMaxSys * kBuckets];
    __shared__ int s_base[kMaxSys * kBuckets];
    const int tid = threadIdx.x;
    const int b = int(blockIdx.x * blockDim.x + tid);
    for (int t = tid; t < kMaxSys * kBuckets; t += 128)
        s_cnt[t] = 0;
    __syncthreads();
    int s = 0, bucket = -1, rank = 0, base = 0;
    if (b < L.total_blocks) {
#pragma unroll
        for (int t = 1; t < kMaxSys; ++t)
            if (t < L.nsys && b >= L.sys[t].block_begin)
                s = t;
        const SysDesc& sd = L.sys[s];
        if (b - sd.block_begin < sd.n_local) {
            const int order[8] = {TCSE_GREEDY_POTENTIAL, TCSE_GREEDY_INTERSECTIONS, TCSE_MIXED, TCSE_GREEDY_RANDOM,
                                  TCSE_GREEDY_ALTERNATIVE, TCSE_WEIGHTED_RANDOM, TCSE_GREEDY, 7};
            // within a strategy, fresh processes before reinit ones (which
            // replay part of the incumbent instead of selecting: shorter);
            // skipped blocks (slot 7) last
            const int st0 = L.slots[b].strategy;
            const int st = st0 < 0 ? 7 : st0, cls = st0 < 0 ? 0 : L.slots[b].pad;
            const int* h = L.hist + s * kHistStride;
            base = sd.block_begin;
            for (int k = 0; k < 8 && order[k] != st; ++k)
#pragma unroll
                for (int c = 0; c < kWorkClasses; ++c)
                    base += h[order[k] + 8 * c];
            for (int c = 0; c < cls; ++c)
                base += h[st + 8 * c];
            bucket = s * kBuckets + st + 8 * cls;
            rank = atomicAdd(&s_cnt[bucket], 1);  // any order within a bucket
        }
    }
    __syncthreads();
    for (int t = tid; t < kMaxSys * kBuckets; t += 128)
        if (s_cnt[t])
            s_base[t] = atomicAdd(&L.hist[(t / kBuckets) * kHistStride + 8 * kWorkClasses + (t % kBuckets)], s_cnt[t]);
    __syncthreads();
    if (bucket >= 0)
        L.perm[base + s_base[bucket] + rank] = b;
}

// ----------------------------------------------------------------- K2
//
// The iteration barrier (parallel_search.hpp:237-270) as two short kernels
// on the launch stream, all reading only device state so a whole iteration
// can be replayed from a CUDA graph:
//   pack    — this rank's payload: its slice of costs, its best record, its
//             launch error;
//   (the payloads are all-gathered here when world > 1: NCCL on the stream)
//   barrier — nblk blocks per system tally the n gathered costs (partial
//             argmin, cost histograms, this rank's step / word-op sums); the
//             last block to arrive merges them: global argmin by (cost, id),
//             strict improvement, incumbent record copy, patience and
//             max_iterations (the loop variables of optimize_system), and the
//             next reinit flags (pick_reinit, 149-163).
// A launch error on any rank (device capacity, replay) skips the barrier on
// every rank, so the host re-runs or reports the same iteration everywhere.

__device__ __forceinline__ int part_of(int n, int world, int r) { return int((long long)n * r / world); }

constexpr int kRedNT = 1024;  // pack / barrier block
constexpr int kTallyNT = 256;  // barrier block
constexpr int kTallyPer = 2048;  // gathered costs per tally block

// owner rank of global process p (contiguous partition)
__device__ __forceinline__ int owner_of(int n, int world, int p) {
    int r = int((long long)p * world / n);
    while (r + 1 < world && part_of(n, world, r + 1) <= p)
        ++r;
    while (r > 0 && part_of(n, world, r) > p)
        --r;
    return r;
}

// direct mode (X.recv == null: one rank, no exchange): the barrier reads the
// per-process outputs themselves and pack is not launched
__device__ __forceinline__ int gathered_cost(const XchgDesc& X, int p) {
    if (!X.recv)
        return X.cost[p];
    const int r = owner_of(X.n, X.world, p);
    return X.recv[size_t(r) * size_t(X.words_total) + size_t(X.sys_off) + size_t(p - part_of(X.n, X.world, r))];
}

// first launch error among the gathered payloads (0 = none)
__device__ __forceinline__ int gathered_error(const XchgDesc& X) {
    if (!X.recv)
        return 0;  // the local error word is checked by the caller
    int e = 0;
    for (int r = 0; r < X.world && e == 0; ++r)
        e = X.recv[size_t(r) * size_t(X.words_total) + size_t(X.sys_off) + size_t(X.n_max) + 6];
    return e;
}

// K2a: this rank's payload (local argmin + record copy), one block per system
__global__ void __launch_bounds__(kRedNT) pack_kernel(const __grid_constant__ XchgLaunch XL) {
    const XchgDesc& X = XL.x[blockIdx.x];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (blockIdx.x == 0 && tid == 0 && XL.clock)
        XL.clock->xstart = globaltimer();
    if (!X.inc->active)
        return;  // every rank agrees (identical barriers)
    __shared__ u64 s_min[32];
    __shared__ int s_bp;
    int32_t* out = X.send + X.sys_off;
    const int err = *XL.err;
    if (err != 0) {  // only the error travels
        if (tid == 0)
            out[X.n_max + 6] = err;
        return;
    }
    u64 best = ~0ULL;
    for (int t = tid; t < X.n_local; t += kRedNT) {
        const int32_t c = X.cost[t];
        out[t] = c;
        best = min(best, (u64(u32(c)) << 32) | u64(u32(t)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        best = min(best, __shfl_down_sync(FULLMASK, best, o));
    if (lane == 0)
        s_min[warp] = best;
    __syncthreads();
    if (tid == 0) {
        u64 b = s_min[0];
        for (int w = 1; w < kRedNT / 32; ++w)
            b = min(b, s_min[w]);
        int32_t* h = out + X.n_max;
        const int t = X.n_local > 0 ? int(b & 0xffffffffu) : -1;
        h[0] = t >= 0 ? 1 : 0;
        h[1] = t >= 0 ? X.p0 + t : -1;
        h[2] = t >= 0 ? X.len[t] : 0;
        h[3] = t >= 0 ? X.strat[t] : 0;
        const u64 sd = t >= 0 ? X.seed[t] : 0;
        h[4] = int32_t(u32(sd));
        h[5] = int32_t(u32(sd >> 32));
        h[6] = 0;
        h[7] = (XL.budget_ns && XL.clock && globaltimer() - XL.clock->t_begin >= XL.budget_ns) ? 1 : 0;
        s_bp = t;
    }
    __syncthreads();
    const int t = s_bp;
    if (t >= 0) {
        const int L = X.len[t];
        int32_t* rec = out + X.n_max + kHdr;
        for (int e = tid; e < L; e += kRedNT)
            rec[e] = int32_t(X.subs[size_t(t) * size_t(X.sub_cap) + size_t(e)]);
    }
}

// the iteration's device clock (once per iteration, by the last barrier
// block's first warp: lane g < kMaxSys handles launch group g)
__device__ void clock_tick(LoopClock* k, int lane) {
    u64 lo = ~0ULL, hi = 0;
    if (lane < kMaxSys) {
        const u64 g0 = __ldcg(k->gstart + lane), g1 = __ldcg(k->gend + lane);
        if (g0 != ~0ULL && g1 > g0) {
            k->group_ns[lane] += g1 - g0;
            lo = g0;
            hi = g1;
        }
        k->gstart[lane] = ~0ULL;
        k->gend[lane] = 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(FULLMASK, lo, o));
        hi = max(hi, __shfl_xor_sync(FULLMASK, hi, o));
    }
    if (lane == 0) {
        if (hi > lo) {
            k->search_ns += hi - lo;
            k->iterations += 1;
        }
        const u64 now = globaltimer(), x0 = __ldcg(&k->xstart);
        if (x0 != 0 && now > x0)
            k->exchange_ns += now - x0;
        k->xstart = 0;
    }
}

// K2b: the barrier in one launch (grid: nblk x nsys).  Every block tallies
// kTallyPer gathered costs (partial argmin, cost histogram) and its share of
// this rank's step / word-op sums; the last block of a system to arrive runs
// the barrier: global argmin by (cost, id), strict improvement, incumbent
// record copy, patience / max_iterations, and the next reinit flags
// (threshold cost from the merged histogram + ordered tie scan).
__global__ void __launch_bounds__(kTallyNT) barrier_kernel(const __grid_constant__ XchgLaunch XL) {
    extern __shared__ int hist[];
    const XchgDesc& X = XL.x[blockIdx.y];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kTallyNT / 32;
    constexpr int kS = 3 + 8;
    __shared__ u64 s_red[NW][kS + 1];
    __shared__ int s_flag[6];
    const int nb = X.nblk, n = X.n, world = X.world;
    if (!X.recv && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0 && XL.clock && XL.clock->xstart == 0)
        XL.clock->xstart = globaltimer();  // direct mode: no pack launch stamped it
    bool work = X.inc->active && *XL.err == 0;
    if (work) {
        const int ge = gathered_error(X);
        if (ge != 0) {  // another rank failed: skip the barrier everywhere
            if (blockIdx.x == 0 && tid == 0)
                atomicCAS(XL.err, 0, ge);
            work = false;
        }
    }
    bool last = false;
    if (work) {
        // ---- tally
        const int blk = blockIdx.x;
        for (int v = tid; v < X.hist_n; v += kTallyNT)
            hist[v] = 0;
        __syncthreads();
        const int p0 = blk * kTallyPer, p1 = min(n, p0 + kTallyPer);
        u64 best = ~0ULL;
        for (int p = p0 + tid; p < p1; p += kTallyNT) {
            const int c = gathered_cost(X, p);
            best = min(best, (u64(u32(c)) << 32) | u64(u32(p)));
            atomicAdd(&hist[min(max(c, 0), X.hist_n - 1)], 1);
        }
        u64 sums[kS];
#pragma unroll
        for (int k = 0; k < kS; ++k)
            sums[k] = 0;
        const int lper = (X.n_local + nb - 1) / nb;
        const int l0 = min(X.n_local, blk * lper), l1 = min(X.n_local, l0 + lper);
        for (int t = l0 + tid; t < l1; t += kTallyNT) {
            const u64 own = u64(X.own[t]);
            sums[0] += own;
            sums[1] += u64(X.len[t] - X.own[t]);
            sums[2] += X.wops[t];
            const int st = X.strat[t];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                sums[3 + k] += st == k ? own : 0;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            best = min(best, __shfl_down_sync(FULLMASK, best, o));
#pragma unroll
            for (int k = 0; k < kS; ++k)
                sums[k] += __shfl_down_sync(FULLMASK, sums[k], o);
        }
        if (lane == 0) {
            s_red[warp][0] = best;
#pragma unroll
            for (int k = 0; k < kS; ++k)
                s_red[warp][1 + k] = sums[k];
        }
        __syncthreads();
        if (tid < kS + 1) {
            u64 v = tid == 0 ? ~0ULL : 0;
            for (int w = 0; w < NW; ++w)
                v = tid == 0 ? min(v, s_red[w][0]) : v + s_red[w][tid];
            if (tid == 0)
                X.part_min[blk] = v;
            else
                X.part_sums[size_t(blk) * kS + size_t(tid - 1)] = v;
        }
        for (int v = tid; v < X.hist_n; v += kTallyNT)
            X.part_hist[size_t(blk) * size_t(X.hist_n) + size_t(v)] = hist[v];
        // ---- arrival: the last block of this system runs the barrier
        __threadfence();
        __syncthreads();
        if (tid == 0)
            s_flag[0] = atomicAdd(X.done, 1) == nb - 1 ? 1 : 0;
        __syncthreads();
        last = s_flag[0] != 0;
    }
    if (last) {
        __threadfence();  // the other blocks' partials are visible
        if (tid == 0)
            *X.done = 0;  // for the next iteration
        // ---- combine the partials
        u64 b = ~0ULL;
        u64 sums[kS];
#pragma unroll
        for (int k = 0; k < kS; ++k)
            sums[k] = 0;
        // other blocks' partials: read through L2 (ld.cg), never a stale L1 line
        for (int k = tid; k < nb; k += kTallyNT) {
            b = min(b, __ldcg(X.part_min + k));
#pragma unroll
            for (int j = 0; j < kS; ++j)
                sums[j] += __ldcg(X.part_sums + size_t(k) * kS + size_t(j));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            b = min(b, __shfl_down_sync(FULLMASK, b, o));
#pragma unroll
            for (int k = 0; k < kS; ++k)
                sums[k] += __shfl_down_sync(FULLMASK, sums[k], o);
        }
        __syncthreads();  // s_red reuse
        if (lane == 0) {
            s_red[warp][0] = b;
#pragma unroll
            for (int k = 0; k < kS; ++k)
                s_red[warp][1 + k] = sums[k];
        }
        // merged histogram (every block's counts)
        for (int v = tid; v < X.hist_n; v += kTallyNT) {
            int acc = 0;
            for (int k = 0; k < nb; ++k)
                acc += __ldcg(X.part_hist + size_t(k) * size_t(X.hist_n) + size_t(v));
            hist[v] = acc;
        }
        __syncthreads();
        if (tid == 0) {
            u64 bb = ~0ULL, ss[kS];
            for (int k = 0; k < kS; ++k)
                ss[k] = 0;
            for (int w = 0; w < NW; ++w) {
                bb = min(bb, s_red[w][0]);
                for (int k = 0; k < kS; ++k)
                    ss[k] += s_red[w][1 + k];
            }
            // argmin over (cost, global process id): lowest index wins ties (255-260)
            const int bp = int(bb & 0xffffffffu);
            const int bc = int(bb >> 32);
            const int rb = owner_of(n, world, bp);  // the rank that owns bp carries its record
            IncState* inc = X.inc;
            inc->best_p = bp;
            inc->best_cost = bc;
            inc->steps += ss[0];
            inc->replayed += ss[1];
            inc->wops += ss[2];
            for (int k = 0; k < 8; ++k)
                inc->steps_by_strategy[k] += ss[3 + k];
            if (!inc->have || bc < inc->cost) {  // strictly better (261-266)
                inc->have = 1;
                inc->cost = bc;
                if (X.recv) {
                    const int32_t* h =
                        X.recv + size_t(rb) * size_t(X.words_total) + size_t(X.sys_off) + size_t(X.n_max);
                    inc->len = h[2];
                    inc->strategy = h[3];
                    inc->seed = u64(u32(h[4])) | (u64(u32(h[5])) << 32);
                } else {
                    inc->len = X.len[bp];
                    inc->strategy = X.strat[bp];
                    inc->seed = X.seed[bp];
                }
                inc->improved = 1;
                inc->unchanged = 0;
            } else {
                inc->improved = 0;
                inc->unchanged += 1;
            }
            // the loop condition of optimize_system (268-270) + the stop knob
            inc->iteration += 1;
            if (inc->unchanged >= X.patience || (X.max_iterations > 0 && inc->iteration >= X.max_iterations))
                inc->active = 0;
            s_flag[0] = inc->improved ? rb : -1;
            s_flag[1] = inc->len;
            s_flag[4] = bp;  // (direct mode: the best process's record row)
        }
        __syncthreads();
        const int rb = s_flag[0];
        const int inc_len = s_flag[1];
        if (rb >= 0) {
            if (X.recv) {
                const int32_t* rec =
                    X.recv + size_t(rb) * size_t(X.words_total) + size_t(X.sys_off) + size_t(X.n_max) + kHdr;
                for (int t = tid; t < inc_len; t += kTallyNT)
                    X.inc_keys[t] = u32(rec[t]);
            } else {
                const u32* rec = X.subs + size_t(s_flag[4]) * size_t(X.sub_cap);
                for (int t = tid; t < inc_len; t += kTallyNT)
                    X.inc_keys[t] = rec[t];
            }
        }
        // ---- pick_reinit (149-163) for the next iteration, only if the
        // incumbent can share a prefix (235-237)
        const long long want = llround(__dmul_rn(X.fraction, double(n)));
        const int count = inc_len >= 2 ? int(min(want, (long long)n)) : 0;
        if (count > 0) {
            if (warp == 0) {
                // threshold c*: all costs > c* are chosen, plus the first
                // `need` processes (by index) with cost == c* (stable order,
                // 158-160); one warp scans the histogram from the top
                int acc = 0, cstar = 0, need = 0;
                for (int top = X.hist_n - 1; top >= 0; top -= 32) {
                    const int c = top - lane;
                    const int hc = c >= 0 ? hist[c] : 0;
                    int incl = hc;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(FULLMASK, incl, o);
                        if (lane >= o)
                            incl += y;
                    }
                    const unsigned hit = __ballot_sync(FULLMASK, c >= 0 && acc + incl >= count);
                    if (hit) {
                        const int l = __ffs(hit) - 1;
                        const int il = __shfl_sync(FULLMASK, incl, l), hl = __shfl_sync(FULLMASK, hc, l);
                        cstar = top - l;
                        need = count - (acc + il - hl);
                        break;
                    }
                    acc += __shfl_sync(FULLMASK, incl, 31);
                }
                if (lane == 0) {
                    s_flag[2] = cstar;
                    s_flag[3] = need;
                }
            }
            __syncthreads();
            // publish the threshold and every tally block's tie offset (ties
            // at c* before the block, index order) for the flags kernel
            if (warp == 0) {
                const int cstar = s_flag[2];
                int acc = 0;  // ties at c* before block k (part_min reused for it)
                for (int k0 = 0; k0 < nb; k0 += 32) {
                    const int k = k0 + lane;
                    const int v =
                        k < nb ? __ldcg(X.part_hist + size_t(k) * size_t(X.hist_n) + size_t(min(cstar, X.hist_n - 1)))
                               : 0;
                    int incl = v;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(FULLMASK, incl, o);
                        if (lane >= o)
                            incl += y;
                    }
                    if (k < nb)
                        X.part_min[k] = u64(u32(acc + incl - v));
                    acc += __shfl_sync(FULLMASK, incl, 31);
                }
                if (lane == 0) {
                    X.sel[0] = cstar;
                    X.sel[1] = s_flag[3];
                }
            }
        }
        if (tid == 0)
            X.sel[2] = count;
    }
    // ---- the launch's last block (all systems) advances the device clock
    if (XL.clock) {
        __threadfence();
        __syncthreads();
        if (tid == 0)
            s_flag[5] = atomicAdd(XL.all_done, 1) == int(gridDim.x * gridDim.y) - 1 ? 1 : 0;
        __syncthreads();
        if (s_flag[5] && warp == 0) {
            __threadfence();
            if (lane == 0)
                *XL.all_done = 0;
            clock_tick(XL.clock, lane);
        }
    }
}

// K2c: the next iteration's reinit flags (grid: nblk x nsys), every block
// its kTallyPer processes: all costs above the threshold c*, and the first
// `need` ties at c* in index order (offsets from the barrier's last block)
__global__ void __launch_bounds__(kTallyNT) flags_kernel(const __grid_constant__ XchgLaunch XL) {
    const XchgDesc& X = XL.x[blockIdx.y];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kTallyNT / 32;
    if (XL.budget_ns && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0 && *XL.err == 0) {
        // the fixed-wall-time stop (at the first barrier after the budget):
        // every system of the session at once; with an exchange, rank 0's
        // clock as it travelled in its payload, so every rank agrees
        bool stop = false;
        if (!X.recv) {
            stop = globaltimer() - XL.clock->t_begin >= XL.budget_ns;
        } else {
            for (int s = 0; s < XL.nsys; ++s)
                stop = stop || XL.x[s].recv[size_t(XL.x[s].sys_off) + size_t(XL.x[s].n_max) + 7] != 0;
        }
        if (stop)
            for (int s = 0; s < XL.nsys; ++s)
                XL.x[s].inc->active = 0;
    }
    // a converged system (before or at this barrier) never reads its flags
    if (!X.inc->active || *XL.err != 0)
        return;
    const int n = X.n;
    const int p0 = blockIdx.x * kTallyPer, p1 = min(n, p0 + kTallyPer);
    if (X.sel[2] <= 0) {
        for (int p = p0 + tid; p < p1; p += kTallyNT)
            X.reinit_next[p] = 0;
        return;
    }
    const int cstar = X.sel[0], need = X.sel[1];
    constexpr int kPer = kTallyPer / kTallyNT;
    // coalesced loads: element p0 + r * kTallyNT + tid, r = 0..kPer-1; tie
    // ranks by ballots per row of kTallyNT processes
    int cs[kPer];
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
        const int e = p0 + r * kTallyNT + tid;
        cs[r] = e < p1 ? gathered_cost(X, e) : -1;
    }
    __shared__ int s_w[kPer][NW];
    unsigned bal[kPer];
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
        bal[r] = __ballot_sync(FULLMASK, cs[r] == cstar);
        if (lane == 0)
            s_w[r][warp] = __popc(bal[r]);
    }
    __syncthreads();
    int base = int(X.part_min[blockIdx.x]);
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
        int ex = base + __popc(bal[r] & ((1u << lane) - 1u));
        int tot = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            ex += w < warp ? s_w[r][w] : 0;
            tot += s_w[r][w];
        }
        const int e = p0 + r * kTallyNT + tid;
        if (e < p1)
            X.reinit_next[e] = u8(cs[r] > cstar || (cs[r] == cstar && ex < need));
        base += tot;
    }
}

// ------------------------------------------------------------ dispatch

template <int W, int NT, bool GID, int F = 0>
static cudaError_t launch_w(const LaunchDesc& L, int smem, cudaStream_t st) {
    auto k = search_kernel<W, NT, GID, F>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess)
        return e;
    e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess)
        return e;
    k<<<L.total_blocks + L.n_builders, NT, smem, st>>>(L);
    return cudaGetLastError();
}

// instantiated (W words, block size, gi form) combinations; the host picks
// the block size with pick_nt() and the gi form by problem size
cudaError_t launch_search_w(const LaunchDesc& L, int W, int nt, bool dense, int form, int smem, cudaStream_t st) {
    // lists of at most 32 candidates (Laderman-size systems): their own
    // one-warp instantiation with the branch-free gi loop (gi_dense_small)
    if (dense && (form & kFormSmall) && W == 1 && nt == 32)
        return launch_w<1, 32, true, kFormBm | kFormSmall>(L, smem, st);
    // bitmap-pruned gi: the shapes host.cpp bm_instantiated() lists
    if (dense && (form & kFormBm)) {
        if (W == 1 && nt == 32)
            return launch_w<1, 32, true, kFormBm>(L, smem, st);
        if (W == 1 && nt == 64)
            return launch_w<1, 64, true, kFormBm>(L, smem, st);
        if (W == 2 && nt == 64)
            return launch_w<2, 64, true, kFormBm>(L, smem, st);
        if (W == 1 && nt == 128)
            return launch_w<1, 128, true, kFormBm>(L, smem, st);
        if (W == 2 && nt == 128)
            return launch_w<2, 128, true, kFormBm>(L, smem, st);
        if (W == 3 && nt == 128)
            return launch_w<3, 128, true, kFormBm>(L, smem, st);
        if (W == 4 && nt == 128)
            return launch_w<4, 128, true, kFormBm>(L, smem, st);
    }
#define TCSE_CASE(w_, nt_)                                                                      \
    if (W == w_ && nt == nt_)                                                                   \
        return dense ? launch_w<w_, nt_, true>(L, smem, st) : launch_w<w_, nt_, false>(L, smem, st);
    TCSE_CASE(1, 32)
    TCSE_CASE(1, 64)
    TCSE_CASE(2, 64)
    TCSE_CASE(1, 128)
    TCSE_CASE(2, 128)
    TCSE_CASE(3, 128)
    TCSE_CASE(4, 128)
    TCSE_CASE(8, 128)
    TCSE_CASE(1, 256)
    TCSE_CASE(2, 256)
    TCSE_CASE(3, 256)
    TCSE_CASE(4, 256)
#undef TCSE_CASE
    return cudaErrorInvalidValue;
}

cudaError_t launch_search(const LaunchDesc& L, int W, int nt, bool dense, int form, int smem, cudaStream_t st) {
    const int g = (L.total_blocks + 127) / 128;
    if (L.hist) {
        cudaError_t e = cudaMemsetAsync(L.hist, 0, sizeof(int32_t) * kHistStride * kMaxSys, st);
        if (e != cudaSuccess)
            return e;
    }
    prep_kernel<<<g, kPrepNT, 0, st>>>(L);
    if (L.perm)
        place_kernel<<<g, 128, 0, st>>>(L);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return e;
    return launch_search_w(L, W, nt, dense, form, smem, st);
}

cudaError_t launch_pack(const XchgLaunch& XL, cudaStream_t st) {
    pack_kernel<<<XL.nsys, kRedNT, 0, st>>>(XL);
    return cudaGetLastError();
}

int barrier_blocks(int n) { return (n + kTallyPer - 1) / kTallyPer; }

// the barrier (the exchange, if any, ran before on the stream)
cudaError_t launch_reduce(const XchgLaunch& XL, int hist_n, cudaStream_t st) {
    const int smem = hist_n * int(sizeof(int));
    const int nb = XL.x[0].nblk;
    cudaError_t e = cudaFuncSetAttribute(barrier_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess)
        return e;
    barrier_kernel<<<dim3(nb, XL.nsys), kTallyNT, smem, st>>>(XL);
    flags_kernel<<<dim3(nb, XL.nsys), kTallyNT, 0, st>>>(XL);
    return cudaGetLastError();
}

int search_smem_attr_max() { return 227 * 1024; }

}  // namespace tcse

#if defined(TCSE_GI_STATS) || defined(TCSE_SNAP_STATS)
extern "C" int tcse_debug_gi_stats(unsigned long long* out, int reset) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, tcse::g_gi_stats, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(tcse::g_gi_stats, z, sizeof z);
    }
    return 0;
}
#endif
