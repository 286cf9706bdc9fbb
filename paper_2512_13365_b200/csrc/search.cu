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
#include <cuda_runtime.h>

#include "launch.h"

namespace tcse {

#define FULLMASK 0xffffffffu

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

__device__ __forceinline__ u64 mix_seed4(u64 a, u64 b, u64 c, u64 d) {
    u64 h = 0x5851f42d4c957f2dULL;
    h = splitmix64(h ^ a);
    h = splitmix64(h ^ b);
    h = splitmix64(h ^ c);
    h = splitmix64(h ^ d);
    return h;
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

// ------------------------------------------------------ block primitives

template <int NT>
struct Red {
    static constexpr int NW = NT / 32;
};

__device__ __forceinline__ u32 warp_incl_scan(u32 v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(FULLMASK, v, o);
        if (lane >= o)
            v += t;
    }
    return v;
}

// exclusive block scan of one u32 per thread; total in *total
template <int NT>
__device__ __forceinline__ u32 block_scan(u32 v, u32* red, u32* total) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const u32 inc = warp_incl_scan(v, lane);
    if (lane == 31)
        red[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const u32 w = lane < NW ? red[lane] : 0u;
        const u32 wi = warp_incl_scan(w, lane);
        if (lane < NW)
            red[lane] = wi - w;
        if (lane == NW - 1)
            red[NW] = wi;
    }
    __syncthreads();
    const u32 res = red[warp] + inc - v;
    *total = red[NW];
    __syncthreads();
    return res;
}

template <int NT>
__device__ __forceinline__ u32 block_max(u32 v, u32* red) {
    constexpr int NW = NT / 32;
    v = __reduce_max_sync(FULLMASK, v);
    if ((threadIdx.x & 31) == 0)
        red[threadIdx.x >> 5] = v;
    __syncthreads();
    u32 r = red[0];
#pragma unroll
    for (int w = 1; w < NW; ++w)
        r = max(r, red[w]);
    __syncthreads();
    return r;
}

template <int NT>
__device__ __forceinline__ u32 block_sum(u32 v, u32* red) {
    constexpr int NW = NT / 32;
    v = __reduce_add_sync(FULLMASK, v);
    if ((threadIdx.x & 31) == 0)
        red[threadIdx.x >> 5] = v;
    __syncthreads();
    u32 r = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w)
        r += red[w];
    __syncthreads();
    return r;
}

// first maximum of (score, index): larger score wins, ties to smaller index
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
    __syncthreads();
    return bi;
}

// ------------------------------------------------------------- process

template <int W, int NT>
struct Proc {
    static constexpr int NW = NT / 32;
    const SysDesc& sd;
    int lp;  // local process index
    int tid, lane, warp;

    // shared-memory carve
    u64* mask;  // [vcap][2W]
    u32* keys[2];
    u16* cnts[2];
    u16* tcnt;
    u16* ncp;
    u16* ncn;
    u32* aux;
    u32* newexcl;
    u32* coin;
    u32* qbase;
    u32* nvar;
    double* wd;
    double* wb;
    u64* mt;
    u32* red;
    double* reds;
    int* redi;

    // block-uniform state
    int V;      // variables alive (n_x + n_f)
    int m;      // candidates
    int cur;    // candidate buffer
    int cost;   // total_cost (linear_system.hpp:202-204)
    int n_rec;  // record entries written (prefix included in search mode)
    int n_own;  // substitutions selected by this process
    int mti;    // mt19937_64 position (312 = twist pending)
    u64 wops;   // algorithmic word-intersections (SURVEY.md 8(d) model), thread 0
    u32 last_coins;  // coins drawn by the last gi selection (sum of deg)

    __device__ Proc(const SysDesc& s, int lp_, unsigned char* smem) : sd(s), lp(lp_) {
        tid = threadIdx.x;
        lane = tid & 31;
        warp = tid >> 5;
        auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
        size_t off = 0;
        mask = reinterpret_cast<u64*>(smem + off);
        off += al(size_t(sd.vcap) * 2 * W * 8);
        keys[0] = reinterpret_cast<u32*>(smem + off);
        off += al(size_t(sd.mcap) * 4);
        keys[1] = reinterpret_cast<u32*>(smem + off);
        off += al(size_t(sd.mcap) * 4);
        cnts[0] = reinterpret_cast<u16*>(smem + off);
        off += al(size_t(sd.mcap) * 2);
        cnts[1] = reinterpret_cast<u16*>(smem + off);
        off += al(size_t(sd.mcap) * 2);
        const size_t uni = off;
        tcnt = reinterpret_cast<u16*>(smem + off);
        off += al(size_t(sd.mcap) * 2);
        ncp = reinterpret_cast<u16*>(smem + off);
        off += al(size_t(sd.vcap + 1) * 2);
        ncn = reinterpret_cast<u16*>(smem + off);
        off += al(size_t(sd.vcap + 1) * 2);
        aux = reinterpret_cast<u32*>(smem + off);
        off += al(size_t(sd.mcap) * 4);
        newexcl = reinterpret_cast<u32*>(smem + off);
        off += al(size_t(sd.vcap + 2) * 4);
        const size_t end_upd = off;
        off = uni;
        coin = reinterpret_cast<u32*>(smem + off);
        off += al(size_t(kCoinWords) * 4);
        qbase = reinterpret_cast<u32*>(smem + off);
        off += al(size_t(sd.mcap + 1) * 4);
        nvar = reinterpret_cast<u32*>(smem + off);
        off += al(size_t(sd.vcap + 1) * 4);
        wd = reinterpret_cast<double*>(smem + off);
        off += al(size_t(sd.mcap) * 8);
        wb = reinterpret_cast<double*>(smem + off);
        off += al(size_t(sd.mcap) * 8);
        off = off > end_upd ? off : end_upd;
        mt = reinterpret_cast<u64*>(smem + off);
        off += 312 * 8;
        red = reinterpret_cast<u32*>(smem + off);
        off += al(size_t(NW + 2) * 8);
        reds = reinterpret_cast<double*>(smem + off);
        off += al(size_t(NW + 2) * 8);
        redi = reinterpret_cast<int*>(smem + off);
    }

    // ---- masks
    __device__ __forceinline__ u64* P(int v) { return mask + size_t(v) * 2 * W; }
    __device__ __forceinline__ u64* N(int v) { return mask + size_t(v) * 2 * W + W; }

    // frequency of (a, b, neg) with 1-based ids (count_pairs, linear_system.hpp:151-161)
    __device__ __forceinline__ int count_pair(int a, int b, int neg) {
        const u64* pa = P(a - 1);
        const u64* na = N(a - 1);
        const u64* pb = P(b - 1);
        const u64* nb = N(b - 1);
        int c = 0;
#pragma unroll
        for (int w = 0; w < W; ++w)
            c += neg ? (__popcll(pa[w] & nb[w]) + __popcll(na[w] & pb[w]))
                     : (__popcll(pa[w] & pb[w]) + __popcll(na[w] & nb[w]));
        return c;
    }

    // ---- mt19937_64 (block-uniform: every thread walks the same stream)
    __device__ void seed_rng(u64 s) {  // one thread
        u64 x = s;
        mt[0] = x;
        for (u32 i = 1; i < 312; ++i) {
            x = kMtF * (x ^ (x >> 62)) + i;
            mt[i] = x;
        }
    }

    __device__ void twist() {
        constexpr int R = (156 + NT - 1) / NT;
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
        mti = 0;
    }

    __device__ __forceinline__ u64 draw() {
        if (mti >= 312)
            twist();
        return mt_temper(mt[mti++]);
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

    // n coin flips (uniform_int_distribution<int>(0,1) == top bit) into coin[]
    __device__ void draw_coins(u32 nbits) {
        const u32 words = (nbits + 31) >> 5;
        for (u32 w = tid; w < words; w += NT)
            coin[w] = 0u;
        __syncthreads();
        u32 done = 0;
        while (done < nbits) {
            if (mti >= 312)
                twist();
            const u32 n = min(u32(312 - mti), nbits - done);
            const u32 n32 = (n + 31) & ~31u;
            for (u32 e = tid; e < n32; e += NT) {
                const bool valid = e < n;
                const u32 bit = valid ? u32(mt_temper(mt[mti + e]) >> 63) : 0u;
                const u32 ball = __ballot_sync(FULLMASK, bit);
                if (lane == 0 && ball) {
                    const u32 pos = done + (e - lane);
                    const u32 wd_ = pos >> 5, sh = pos & 31;
                    atomicOr(&coin[wd_], ball << sh);
                    if (sh)
                        atomicOr(&coin[wd_ + 1], ball >> (32 - sh));
                }
            }
            mti += int(n);
            done += n;
        }
        __syncthreads();
    }

    // ---- substitution (apply_substitution, linear_system.hpp:167-189)
    // returns the number of replaced occurrences; 0 leaves the state untouched
    __device__ int apply(u32 q) {
        if (tid == 0) {
            const int i = key_i(q) - 1, j = key_j(q) - 1, neg = key_neg(q);
            const int k = V;
            u64* pi = P(i);
            u64* ni = N(i);
            u64* pj = P(j);
            u64* nj = N(j);
            u64 rp[W], rn[W];
            int c = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                rp[w] = pi[w] & (neg ? nj[w] : pj[w]);
                rn[w] = ni[w] & (neg ? pj[w] : nj[w]);
                c += __popcll(rp[w]) + __popcll(rn[w]);
            }
            if (c > 0) {
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    pi[w] &= ~rp[w];
                    ni[w] &= ~rn[w];
                    if (!neg) {
                        pj[w] &= ~rp[w];
                        nj[w] &= ~rn[w];
                    } else {
                        nj[w] &= ~rp[w];
                        pj[w] &= ~rn[w];
                    }
                    P(k)[w] = rp[w];
                    N(k)[w] = rn[w];
                }
            }
            red[NW + 1] = u32(c);
        }
        __syncthreads();
        const int c = int(red[NW + 1]);
        if (c > 0) {
            ++V;
            cost -= c - 1;
        }
        return c;
    }

    // incremental candidate maintenance after q -> k (= V, 1-based)
    __device__ void update(u32 q) {
        const int i = key_i(q), j = key_j(q);
        const int k = V;
        const u32* ok = keys[cur];
        const u16* oc = cnts[cur];
        // (a) recount old candidates touching i or j (their counts only drop)
        for (int t = tid; t < m; t += NT) {
            const u32 kk = ok[t];
            const int a = key_i(kk), b = key_j(kk);
            tcnt[t] = (a == i || a == j || b == i || b == j) ? u16(count_pair(a, b, key_neg(kk))) : oc[t];
        }
        // (b) the new variable's pairs (x, k, +/-)
        const u64* pk = P(k - 1);
        const u64* nk = N(k - 1);
        for (int x = tid + 1; x < k; x += NT) {
            const u64* px = P(x - 1);
            const u64* nx = N(x - 1);
            int cp = 0, cn = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                cp += __popcll(px[w] & pk[w]) + __popcll(nx[w] & nk[w]);
                cn += __popcll(px[w] & nk[w]) + __popcll(nx[w] & pk[w]);
            }
            ncp[x] = u16(cp);
            ncn[x] = u16(cn);
        }
        __syncthreads();
        // (c) one packed scan: low 16 bits old survivors, high 16 bits new pairs
        const int L = m + 2 * (k - 1);
        const int E = (L + NT - 1) / NT;
        const int e0 = min(L, tid * E), e1 = min(L, e0 + E);
        u32 local = 0;
        for (int e = e0; e < e1; ++e) {
            if (e < m) {
                local += tcnt[e] >= 2 ? 1u : 0u;
            } else {
                const int x = ((e - m) >> 1) + 1;
                const u16 c = ((e - m) & 1) ? ncn[x] : ncp[x];
                local += c >= 2 ? 0x10000u : 0u;
            }
        }
        u32 total;
        const u32 excl = block_scan<NT>(local, red, &total);
        const u32 n_old = total & 0xffffu, n_new = total >> 16;
        u32 o = excl & 0xffffu, n = excl >> 16;
        for (int e = e0; e < e1; ++e) {
            if (e < m) {
                aux[e] = o;
                o += tcnt[e] >= 2 ? 1u : 0u;
            } else {
                const int x = ((e - m) >> 1) + 1;
                const int sg = (e - m) & 1;
                if (!sg)
                    newexcl[x] = n;
                n += ((sg ? ncn[x] : ncp[x]) >= 2) ? 1u : 0u;
            }
        }
        __syncthreads();
        u32* dk = keys[cur ^ 1];
        u16* dc = cnts[cur ^ 1];
        o = excl & 0xffffu;
        n = excl >> 16;
        for (int e = e0; e < e1; ++e) {
            if (e < m) {
                if (tcnt[e] >= 2) {
                    const u32 kk = ok[e];
                    const u32 dest = o + newexcl[key_i(kk)];
                    dk[dest] = kk;
                    dc[dest] = tcnt[e];
                    ++o;
                }
            } else {
                const int x = ((e - m) >> 1) + 1;
                const int sg = (e - m) & 1;
                const u16 c = sg ? ncn[x] : ncp[x];
                if (c >= 2) {
                    // old survivors before (x, k, .) are those with i <= x
                    const u32 bound = u32(x + 1) << 17;
                    int lo = 0, hi = m;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (ok[mid] < bound)
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
        cur ^= 1;
        m = int(n_old + n_new);
    }

    // ---- selection strategies (strategies.hpp); return a candidate index

    // greedy_from (61-69): first maximum in canonical order
    __device__ int sel_greedy() {
        const u16* c = cnts[cur];
        u32 best = 0;
        for (int t = tid; t < m; t += NT)
            best = max(best, (u32(c[t]) << 16) | (0xffffu - u32(t)));
        best = block_max<NT>(best, red);
        return int(0xffffu - (best & 0xffffu));
    }

    // greedy_alternative_from (71-83): uniform over the argmax set
    __device__ int sel_ga() {
        const u16* c = cnts[cur];
        u32 mx = 0;
        for (int t = tid; t < m; t += NT)
            mx = max(mx, u32(c[t]));
        mx = block_max<NT>(mx, red);
        u32 cnt = 0;
        for (int t = tid; t < m; t += NT)
            cnt += c[t] == mx ? 1u : 0u;
        cnt = block_sum<NT>(cnt, red);
        const u32 r = u32(nd(cnt));
        const int E = (m + NT - 1) / NT;
        const int e0 = min(m, tid * E), e1 = min(m, e0 + E);
        u32 local = 0;
        for (int e = e0; e < e1; ++e)
            local += c[e] == mx ? 1u : 0u;
        u32 total;
        u32 ex = block_scan<NT>(local, red, &total);
        for (int e = e0; e < e1; ++e)
            if (c[e] == mx) {
                if (ex == r)
                    redi[NW + 1] = e;
                ++ex;
            }
        __syncthreads();
        const int pick = redi[NW + 1];
        __syncthreads();
        return pick;
    }

    // weighted_random_from (85-98): first q with prefix(c - 1) > u * total
    __device__ int sel_wr() {
        const u16* c = cnts[cur];
        u32 tot = 0;
        for (int t = tid; t < m; t += NT)
            tot += u32(c[t]) - 1u;
        tot = block_sum<NT>(tot, red);
        const double target = __dmul_rn(uniform_real(draw(), 0.0, 1.0), double(tot));
        if (tid == 0)
            redi[NW + 1] = m - 1;
        const int E = (m + NT - 1) / NT;
        const int e0 = min(m, tid * E), e1 = min(m, e0 + E);
        u32 local = 0;
        for (int e = e0; e < e1; ++e)
            local += u32(c[e]) - 1u;
        u32 total;
        u32 s = block_scan<NT>(local, red, &total);
        for (int e = e0; e < e1; ++e) {
            const u32 s1 = s + u32(c[e]) - 1u;
            if (double(s1) > target && double(s) <= target)
                redi[NW + 1] = e;
            s = s1;
        }
        __syncthreads();
        const int pick = redi[NW + 1];
        __syncthreads();
        return pick;
    }

    // select_greedy_random (119-124)
    __device__ int sel_gr(double p_greedy) {
        if (uniform_real(draw(), 0.0, 1.0) < p_greedy)
            return sel_ga();
        return sel_wr();
    }

    // select_greedy_intersections (162-176) with score_intersections_from
    // (136-153): per candidate q, a sequential double sum over all other
    // candidates in canonical order (disjoint: c-1; intersecting: one coin,
    // beta*(c-1) on heads), coins drawn in (q, s) order from the stream
    __device__ int sel_gi(double alpha, double beta) {
        if (alpha == 0.0)
            return sel_greedy();  // gain only; no coins are drawn (140-141)
        const u32* ks = keys[cur];
        const u16* c = cnts[cur];
        for (int v = tid; v <= V; v += NT)
            nvar[v] = 0u;
        __syncthreads();
        for (int t = tid; t < m; t += NT) {
            const u32 kk = ks[t];
            atomicAdd(&nvar[key_i(kk)], 1u);
            atomicAdd(&nvar[key_j(kk)], 1u);
            const double w = double(int(c[t]) - 1);
            wd[t] = w;
            wb[t] = __dmul_rn(beta, w);
        }
        __syncthreads();
        // coins per q = candidates sharing a variable, minus q itself (and
        // its opposite-sign twin, counted under both variables)
        const int E = (m + NT - 1) / NT;
        const int e0 = min(m, tid * E), e1 = min(m, e0 + E);
        u32 local = 0;
        for (int e = e0; e < e1; ++e) {
            const u32 kk = ks[e];
            const u32 twin = (e + 1 < m && ks[e + 1] == (kk | 1u) && !(kk & 1u)) ||
                                     (e > 0 && (kk & 1u) && ks[e - 1] == (kk & ~1u))
                                 ? 1u
                                 : 0u;
            local += nvar[key_i(kk)] + nvar[key_j(kk)] - 2u - twin;
        }
        u32 D;
        u32 ex = block_scan<NT>(local, red, &D);
        for (int e = e0; e < e1; ++e) {
            const u32 kk = ks[e];
            const u32 twin = (e + 1 < m && ks[e + 1] == (kk | 1u) && !(kk & 1u)) ||
                                     (e > 0 && (kk & 1u) && ks[e - 1] == (kk & ~1u))
                                 ? 1u
                                 : 0u;
            qbase[e] = ex;
            ex += nvar[key_i(kk)] + nvar[key_j(kk)] - 2u - twin;
        }
        if (tid == 0)
            qbase[m] = D;
        last_coins = D;
        __syncthreads();
        double best_s = -1.0;
        int best_q = 0x7fffffff;
        constexpr u32 kCap = u32(kCoinWords) * 32u;
        int q_lo = 0;
        while (q_lo < m) {
            const u32 c0 = qbase[q_lo];
            // largest q_hi in (q_lo, m] with qbase[q_hi] - c0 <= kCap
            int lo = q_lo + 1, hi = m;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (qbase[mid] - c0 <= kCap)
                    lo = mid;
                else
                    hi = mid - 1;
            }
            const int q_hi = lo;
            draw_coins(qbase[q_hi] - c0);
            for (int q = q_lo + tid; q < q_hi; q += NT) {
                const u32 kq = ks[q];
                const int qi = key_i(kq), qj = key_j(kq);
                u32 ptr = qbase[q] - c0;
                double fut = 0.0;
                for (int s = 0; s < m; ++s) {
                    if (s == q)
                        continue;
                    const u32 kk = ks[s];
                    const int si = key_i(kk), sj = key_j(kk);
                    const bool inter = (si == qi) | (si == qj) | (sj == qi) | (sj == qj);
                    double add;
                    if (inter) {
                        const u32 bit = (coin[ptr >> 5] >> (ptr & 31u)) & 1u;
                        ++ptr;
                        add = bit ? wb[s] : 0.0;
                    } else {
                        add = wd[s];
                    }
                    fut = __dadd_rn(fut, add);
                }
                const double h = __dadd_rn(wd[q], __dmul_rn(alpha, fut));
                if (h > best_s || best_q == 0x7fffffff) {
                    best_s = h;
                    best_q = q;
                }
            }
            __syncthreads();
            q_lo = q_hi;
        }
        return block_argmax_double<NT>(best_s, best_q, reds, redi);
    }

    // select_greedy_potential (196-220): (c-1) + alpha * created, where
    // created = pairs with the trial variable k reaching frequency >= 2
    // (only pairs with k can newly become substitutable: counts touching
    // i or j drop, all others are unchanged)
    __device__ int sel_gp(double alpha) {
        if (alpha == 0.0)
            return sel_greedy();
        const u32* ks = keys[cur];
        const u16* c = cnts[cur];
        double best_s = -1.0;
        int best_q = 0x7fffffff;
        for (int q = tid; q < m; q += NT) {
            const u32 kq = ks[q];
            const int qi = key_i(kq), qj = key_j(kq), neg = key_neg(kq);
            u64 rp[W], rn[W];
#pragma unroll
            for (int w = 0; w < W; ++w) {
                rp[w] = P(qi - 1)[w] & (neg ? N(qj - 1)[w] : P(qj - 1)[w]);
                rn[w] = N(qi - 1)[w] & (neg ? P(qj - 1)[w] : N(qj - 1)[w]);
            }
            int created = 0;
            for (int x = 1; x <= V; ++x) {
                if (x == qi || x == qj)
                    continue;
                const u64* px = P(x - 1);
                const u64* nx = N(x - 1);
                int cp = 0, cn = 0;
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    cp += __popcll(px[w] & rp[w]) + __popcll(nx[w] & rn[w]);
                    cn += __popcll(px[w] & rn[w]) + __popcll(nx[w] & rp[w]);
                }
                created += (cp >= 2) + (cn >= 2);
            }
            const double h = __dadd_rn(double(int(c[q]) - 1), __dmul_rn(alpha, double(created)));
            if (h > best_s || best_q == 0x7fffffff) {
                best_s = h;
                best_q = q;
            }
        }
        return block_argmax_double<NT>(best_s, best_q, reds, redi);
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
        const int subs[4] = {TCSE_GREEDY_INTERSECTIONS, TCSE_GREEDY_ALTERNATIVE, TCSE_GREEDY_RANDOM,
                             TCSE_WEIGHTED_RANDOM};
        if (positive == 1)
            return subs[only];
        double target = __dmul_rn(uniform_real(draw(), 0.0, 1.0), total);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            target = __dsub_rn(target, mix[k]);
            if (target < 0.0)
                return subs[k];
        }
        return subs[3];
    }

    __device__ u64 cand_hash() {  // one thread: FNV-1a over (i, j, sign, count)
        u64 h = 0xcbf29ce484222325ULL;
        auto feed = [&](int v) {
            const u32 u = u32(v);
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                h ^= (u >> (8 * b)) & 0xffu;
                h *= 0x100000001b3ULL;
            }
        };
        for (int t = 0; t < m; ++t) {
            const u32 kk = keys[cur][t];
            feed(key_i(kk));
            feed(key_j(kk));
            feed(key_neg(kk) ? -1 : 1);
            feed(int(cnts[cur][t]));
        }
        return h;
    }

    // every pair of the current state with count >= minc, canonical order
    __device__ int all_pairs(int minc, u32* okeys, u16* ocnts, int cap) {
        int n_total = 0;
        for (int a = 1; a < V; ++a) {
            const int L = 2 * (V - a);
            const int E = (L + NT - 1) / NT;
            const int e0 = min(L, tid * E), e1 = min(L, e0 + E);
            u32 local = 0;
            for (int e = e0; e < e1; ++e)
                local += count_pair(a, a + 1 + (e >> 1), e & 1) >= minc ? 1u : 0u;
            u32 total;
            u32 ex = block_scan<NT>(local, red, &total);
            for (int e = e0; e < e1; ++e) {
                const int b = a + 1 + (e >> 1);
                const int cc = count_pair(a, b, e & 1);
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
};

__device__ __forceinline__ void set_error(const SysDesc& sd, int code, int pos) {
    if (atomicCAS(sd.err, 0, code) == 0 && sd.err_pos)
        *sd.err_pos = pos;
}

template <int W, int NT>
__global__ void __launch_bounds__(NT) search_kernel(const __grid_constant__ LaunchDesc L) {
    extern __shared__ __align__(16) unsigned char smem[];
    int s = 0;
#pragma unroll
    for (int t = 1; t < kMaxSys; ++t)
        if (t < L.nsys && int(blockIdx.x) >= L.sys[t].block_begin)
            s = t;
    const SysDesc& sd = L.sys[s];
    const int lp = int(blockIdx.x) - sd.block_begin;
    if (lp >= sd.n_local)
        return;

    Proc<W, NT> pr(sd, lp, smem);
    const int tid = threadIdx.x;
    constexpr int NW = NT / 32;

    // ---- process configuration (thread 0) + base state (all threads)
    __shared__ double s_cfg[4 + 4];
    __shared__ u64 s_seed;
    __shared__ int s_int[4];
    if (tid == 0) {
        int strategy;
        double alpha, beta, pg;
        u64 seed;
        double mix[4];
        if (sd.mode == kModeSearch) {
            // assign_strategies (parallel_search.hpp:183-205): first five
            // outputs of mt19937_64(mix_seed{master, salt, iteration, p})
            const u64 p = u64(sd.p0 + lp);
            const u64 ss = mix_seed4(sd.master_seed, sd.salt, u64(int64_t(sd.iteration)), p);
            u64 lo_[7], hi_[6];
            u64 x = ss;
            lo_[0] = x;
            for (u32 i = 1; i <= 161; ++i) {
                x = kMtF * (x ^ (x >> 62)) + i;
                if (i <= 6)
                    lo_[i] = x;
                if (i >= 156)
                    hi_[i - 156] = x;
            }
            u64 out[5];
#pragma unroll
            for (int t = 0; t < 5; ++t)
                out[t] = mt_temper(mt_mix(lo_[t], lo_[t + 1], hi_[t]));
            alpha = uniform_real(out[0], 0.0, 0.5);
            beta = uniform_real(out[1], 0.5, 1.0);
            pg = uniform_real(out[2], 0.5, 1.0);
            int used = 3;
            if (sd.forced >= 0) {
                strategy = sd.forced;
            } else if (sd.iteration == 1 && p == 0) {
                strategy = TCSE_GREEDY;
            } else {
                double target = __dmul_rn(uniform_real(out[3], 0.0, 1.0), sd.weight_total);
                strategy = TCSE_GREEDY;
                for (int k = 0; k < 7; ++k) {
                    target = __dsub_rn(target, sd.weights[k]);
                    if (target < 0.0) {
                        strategy = k;
                        break;
                    }
                }
                used = 4;
            }
            seed = out[used];
            for (int k = 0; k < 4; ++k)
                mix[k] = sd.mix[k];
        } else if (sd.mode == kModeRun) {
            const tcse_process_config& c = sd.cfgs[lp];
            strategy = c.strategy;
            alpha = c.alpha;
            beta = c.beta;
            pg = c.p_greedy;
            seed = c.seed;
            for (int k = 0; k < 4; ++k)
                mix[k] = c.mix_weights[k];
        } else {
            strategy = TCSE_GREEDY;
            alpha = beta = pg = 0.0;
            seed = 0;
            for (int k = 0; k < 4; ++k)
                mix[k] = 0.0;
        }
        const int reinit = (sd.mode == kModeSearch && sd.reinit && sd.reinit[lp]) ? 1 : 0;
        const bool rng = reinit || strategy == TCSE_GREEDY_ALTERNATIVE || strategy == TCSE_WEIGHTED_RANDOM ||
                         strategy == TCSE_GREEDY_RANDOM || strategy == TCSE_MIXED ||
                         (strategy == TCSE_GREEDY_INTERSECTIONS && alpha != 0.0);
        s_int[0] = strategy;
        s_int[1] = reinit;
        s_int[2] = rng ? 1 : 0;
        s_cfg[0] = alpha;
        s_cfg[1] = beta;
        s_cfg[2] = pg;
        for (int k = 0; k < 4; ++k)
            s_cfg[4 + k] = mix[k];
        s_seed = seed;
        if (rng)
            pr.seed_rng(seed);
    }
    {
        const size_t nw = size_t(sd.n_x) * 2 * W;
        for (size_t t = tid; t < nw; t += NT)
            pr.mask[t] = sd.base_masks[t];
        if (sd.base_keys) {
            for (int t = tid; t < sd.base_m; t += NT) {
                pr.keys[0][t] = sd.base_keys[t];
                pr.cnts[0][t] = sd.base_cnts[t];
            }
        }
    }
    __syncthreads();
    const int strategy = s_int[0];
    const int reinit = s_int[1];
    const double alpha = s_cfg[0], beta = s_cfg[1], p_greedy = s_cfg[2];
    double mix[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
        mix[k] = s_cfg[4 + k];
    const u64 seed = s_seed;
    pr.V = sd.n_x;
    pr.cur = 0;
    pr.cost = sd.naive;
    pr.n_rec = 0;
    pr.n_own = 0;
    pr.mti = 312;
    pr.wops = 0;
    pr.last_coins = 0;
    if (sd.base_keys) {
        pr.m = sd.base_m;
    } else {
        pr.m = pr.all_pairs(2, pr.keys[0], pr.cnts[0], sd.mcap);
        if (pr.m > sd.mcap) {
            set_error(sd, TCSE_ECAPACITY, pr.m);
            return;
        }
    }

    // ---- prefix: reinit from the incumbent (parallel_search.hpp:242-248) or a
    // fixed replay (cse_engine.hpp:47-57)
    const u32* pre = nullptr;
    int n_pre = 0;
    if (reinit) {
        const u64 k_max = u64(3 * sd.inc_len / 4);
        n_pre = int(1 + pr.nd(k_max));
        pre = sd.inc_keys;
    } else if (sd.mode != kModeSearch && sd.prefix_len > 0) {
        n_pre = sd.prefix_len;
        pre = sd.prefix;
    }
    u32* rec = sd.out_subs ? sd.out_subs + size_t(lp) * size_t(sd.sub_cap) : nullptr;
    for (int t = 0; t < n_pre; ++t) {
        const u32 q = pre[t];
        const int qi = key_i(q), qj = key_j(q);
        if (qi < 1 || qj <= qi || qj > pr.V || pr.apply(q) == 0) {
            set_error(sd, TCSE_EREPLAY, t);
            if (tid == 0 && sd.out_cost)
                sd.out_cost[lp] = -1;
            return;
        }
        pr.update(q);
    }
    if (reinit) {
        for (int t = tid; t < n_pre; t += NT)
            rec[t] = pre[t];
        pr.n_rec = n_pre;
    }

    if (sd.mode == kModeDump) {
        if (sd.dump_min_count >= 2) {
            for (int t = tid; t < pr.m && t < sd.dump_cap; t += NT) {
                sd.dump_keys[t] = pr.keys[pr.cur][t];
                sd.dump_cnts[t] = pr.cnts[pr.cur][t];
            }
            if (tid == 0)
                *sd.dump_n = pr.m;
        } else {
            const int n = pr.all_pairs(sd.dump_min_count, sd.dump_keys, sd.dump_cnts, sd.dump_cap);
            if (tid == 0)
                *sd.dump_n = n;
        }
        return;
    }

    // ---- run_cse main loop (cse_engine.hpp:33-40)
    u64* trace = sd.trace ? sd.trace + size_t(lp) * size_t(sd.trace_stride) : nullptr;
    for (int step = 0;; ++step) {
        if (trace && tid == 0 && step < sd.trace_stride)
            trace[step] = pr.cand_hash();
        if (pr.m == 0)
            break;
        int pick;
        int strat = strategy;
        if (strat == TCSE_MIXED)
            strat = pr.mixed_sub(mix);  // select_mixed (strategies.hpp:260-269)
        switch (strat) {
            case TCSE_GREEDY: pick = pr.sel_greedy(); break;
            case TCSE_GREEDY_ALTERNATIVE: pick = pr.sel_ga(); break;
            case TCSE_WEIGHTED_RANDOM: pick = pr.sel_wr(); break;
            case TCSE_GREEDY_RANDOM: pick = pr.sel_gr(p_greedy); break;
            case TCSE_GREEDY_INTERSECTIONS: pick = pr.sel_gi(alpha, beta); break;
            default: pick = pr.sel_gp(alpha); break;
        }
        const u32 q = pr.keys[pr.cur][pick];
        {
            // recount 12(V-1)W_E + substitution 8 W_E + selection
            // (m for g/ga/wr/gr; m + sum deg for gi; m (V-2) 4 W_E for gp)
            const u64 Vt = u64(pr.V), mt_ = u64(pr.m), we = u64(sd.words);
            u64 sel = mt_;
            if (strat == TCSE_GREEDY_INTERSECTIONS && alpha != 0.0)
                sel += pr.last_coins;
            if (strat == TCSE_GREEDY_POTENTIAL && alpha != 0.0)
                sel += mt_ * (Vt - 2) * 4 * we;
            pr.wops += 12 * (Vt - 1) * we + 8 * we + sel;
        }
        pr.apply(q);
        pr.update(q);
        if (tid == 0) {
            if (pr.n_rec < sd.sub_cap)
                rec[pr.n_rec] = q;
        }
        ++pr.n_rec;
        ++pr.n_own;
        if (pr.n_rec > sd.sub_cap) {
            set_error(sd, TCSE_ECAPACITY, pr.n_rec);
            return;
        }
    }
    if (tid == 0) {
        sd.out_cost[lp] = pr.cost;
        sd.out_len[lp] = pr.n_rec;
        sd.out_own[lp] = pr.n_own;
        sd.out_strategy[lp] = strategy;
        sd.out_seed[lp] = seed;
        if (sd.out_wops)
            sd.out_wops[lp] = pr.wops;
    }
    (void)NW;
}

// ----------------------------------------------------------------- K2

struct ReduceDesc {
    int32_t n;                // processes (global)
    const int32_t* costs;     // [n] global order
    // record source: arrays indexed by (p - rec_base) for p in [rec_base, rec_base + rec_n)
    int32_t rec_base, rec_n;
    const int32_t* lens;
    const int32_t* strategies;
    const u64* seeds;
    const u32* subs;
    int32_t stride;
    const int32_t* own;      // [own_n] selected-substitution counts of this rank's processes
    const int32_t* own_len;  // [own_n] their record lengths (prefix included)
    const u64* own_wops;     // [own_n] algorithmic word-ops
    int32_t own_n;
    IncState* inc;
    u32* inc_keys;
    u8* reinit_next;  // [n] flags for the next iteration
    double fraction;
    int32_t hist_n;  // costs lie in [0, hist_n)
};

struct ReduceLaunch {
    int32_t nsys;
    ReduceDesc r[kMaxSys];
};

constexpr int kRedNT = 1024;

__global__ void __launch_bounds__(kRedNT) reduce_kernel(const __grid_constant__ ReduceLaunch RL) {
    extern __shared__ int hist[];
    const ReduceDesc& R = RL.r[blockIdx.x];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ u64 s_min[32];
    __shared__ u64 s_sum[32];
    __shared__ u64 s_rep[32];
    __shared__ u64 s_wop[32];
    __shared__ u32 s_red[34];
    __shared__ int s_thr[2];
    // argmin over (cost, process id) — lowest index wins ties (255-260)
    u64 best = ~0ULL;
    u64 steps = 0;
    for (int p = tid; p < R.n; p += kRedNT)
        best = min(best, (u64(u32(R.costs[p])) << 32) | u64(u32(p)));
    u64 replayed = 0, wops = 0;
    for (int p = tid; p < R.own_n; p += kRedNT) {
        steps += u64(R.own[p]);
        replayed += u64(R.own_len[p] - R.own[p]);
        wops += R.own_wops[p];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        best = min(best, __shfl_down_sync(FULLMASK, best, o));
        steps += __shfl_down_sync(FULLMASK, steps, o);
        replayed += __shfl_down_sync(FULLMASK, replayed, o);
        wops += __shfl_down_sync(FULLMASK, wops, o);
    }
    if (lane == 0) {
        s_min[warp] = best;
        s_sum[warp] = steps;
        s_rep[warp] = replayed;
        s_wop[warp] = wops;
    }
    for (int v = tid; v < R.hist_n; v += kRedNT)
        hist[v] = 0;
    __syncthreads();
    if (tid == 0) {
        u64 b = s_min[0], st = 0, rp = 0, wo = 0;
        for (int w = 0; w < kRedNT / 32; ++w) {
            b = min(b, s_min[w]);
            st += s_sum[w];
            rp += s_rep[w];
            wo += s_wop[w];
        }
        const int bp = int(b & 0xffffffffu);
        const int bc = int(b >> 32);
        IncState* inc = R.inc;
        inc->best_p = bp;
        inc->best_cost = bc;
        inc->steps += st;
        inc->replayed += rp;
        inc->wops += wo;
        if (!inc->have || bc < inc->cost) {  // strictly better (261-266)
            inc->have = 1;
            inc->cost = bc;
            inc->len = R.lens[bp - R.rec_base];
            inc->strategy = R.strategies[bp - R.rec_base];
            inc->seed = R.seeds[bp - R.rec_base];
            inc->improved = 1;
        } else {
            inc->improved = 0;
        }
        s_thr[0] = inc->improved ? bp : -1;
        s_thr[1] = inc->len;
    }
    __syncthreads();
    const int bp = s_thr[0];
    const int inc_len = s_thr[1];
    if (bp >= 0)
        for (int t = tid; t < inc_len; t += kRedNT)
            R.inc_keys[t] = R.subs[size_t(bp - R.rec_base) * size_t(R.stride) + size_t(t)];
    // pick_reinit (149-163) for the next iteration, only if the incumbent can
    // share a prefix (235-237)
    long long want = llround(__dmul_rn(R.fraction, double(R.n)));
    const int count = inc_len >= 2 ? int(min(want, (long long)R.n)) : 0;
    if (count <= 0) {
        for (int p = tid; p < R.n; p += kRedNT)
            R.reinit_next[p] = 0;
        return;
    }
    for (int p = tid; p < R.n; p += kRedNT)
        atomicAdd(&hist[min(max(R.costs[p], 0), R.hist_n - 1)], 1);
    __syncthreads();
    if (tid == 0) {
        // threshold cost c*: all costs > c* are chosen, plus the first `need`
        // processes (by index) with cost == c* (stable order, 158-160)
        int acc = 0, cstar = 0, need = 0;
        for (int c = R.hist_n - 1; c >= 0; --c) {
            if (acc + hist[c] >= count) {
                cstar = c;
                need = count - acc;
                break;
            }
            acc += hist[c];
        }
        s_thr[0] = cstar;
        s_thr[1] = need;
    }
    __syncthreads();
    const int cstar = s_thr[0], need = s_thr[1];
    const int E = (R.n + kRedNT - 1) / kRedNT;
    const int e0 = min(R.n, tid * E), e1 = min(R.n, e0 + E);
    u32 local = 0;
    for (int e = e0; e < e1; ++e)
        local += R.costs[e] == cstar ? 1u : 0u;
    const u32 inc_ = warp_incl_scan(local, lane);
    if (lane == 31)
        s_red[warp] = inc_;
    __syncthreads();
    if (warp == 0) {
        const u32 w = s_red[lane];
        const u32 wi = warp_incl_scan(w, lane);
        s_red[lane] = wi - w;
    }
    __syncthreads();
    u32 ex = s_red[warp] + inc_ - local;
    for (int e = e0; e < e1; ++e) {
        const int c = R.costs[e];
        u8 f = 0;
        if (c > cstar) {
            f = 1;
        } else if (c == cstar) {
            f = ex < u32(need) ? 1 : 0;
            ++ex;
        }
        R.reinit_next[e] = f;
    }
}

// ------------------------------------------------------------ dispatch

template <int W, int NT>
static cudaError_t launch_w(const LaunchDesc& L, int smem, cudaStream_t st) {
    auto k = search_kernel<W, NT>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess)
        return e;
    k<<<L.total_blocks, NT, smem, st>>>(L);
    return cudaGetLastError();
}

cudaError_t launch_search(const LaunchDesc& L, int W, int nt, int smem, cudaStream_t st) {
    if (nt == 128) {
        switch (W) {
            case 1: return launch_w<1, 128>(L, smem, st);
            case 2: return launch_w<2, 128>(L, smem, st);
            case 3: return launch_w<3, 128>(L, smem, st);
            case 4: return launch_w<4, 128>(L, smem, st);
            case 8: return launch_w<8, 128>(L, smem, st);
            default: break;
        }
    } else if (nt == 64) {
        switch (W) {
            case 1: return launch_w<1, 64>(L, smem, st);
            case 2: return launch_w<2, 64>(L, smem, st);
            default: break;
        }
    } else if (nt == 256) {
        switch (W) {
            case 1: return launch_w<1, 256>(L, smem, st);
            case 3: return launch_w<3, 256>(L, smem, st);
            default: break;
        }
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_reduce(const ReduceLaunch& RL, int hist_n, cudaStream_t st) {
    const int smem = hist_n * int(sizeof(int));
    cudaError_t e = cudaFuncSetAttribute(reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess)
        return e;
    reduce_kernel<<<RL.nsys, kRedNT, smem, st>>>(RL);
    return cudaGetLastError();
}

int search_smem_attr_max() { return 227 * 1024; }

}  // namespace tcse
