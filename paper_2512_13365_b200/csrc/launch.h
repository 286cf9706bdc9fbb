// launch.h — host/device launch descriptors of the search kernels.
//
// One launch runs the CSE processes of up to TCSE_MAX_SYS systems (the U, V,
// W expression sets of a scheme run concurrently); block b belongs to the
// system whose [block_begin, block_begin + n_local) range holds b, and runs
// local process b - block_begin (global process id p0 + that).
#pragma once

#include <stdint.h>

#include "../../include/tcse.h"

namespace tcse {

typedef unsigned long long u64;
typedef uint32_t u32;
typedef uint16_t u16;
typedef uint8_t u8;

constexpr int kMaxSys = 4;
// RNG hand-off: the prep kernel runs each process's 311-step mt19937_64
// seeding chain and keeps every kCkptStride-th state word; the search block
// restarts kCkpt short chains from them in parallel (one lane each)
constexpr int kCkpt = 32;
constexpr int kCkptStride = 10;  // 32 x 10 >= 312
constexpr int kCoinWords = 512;  // 16384 coin bits per gi scoring chunk
// placement histogram per system: (strategy, work class) counts, then cursors;
// class 0 = fresh processes, 1..4 = reinit ones by replayed-prefix quartile
constexpr int kWorkClasses = 5;
constexpr int kHistStride = 2 * 8 * kWorkClasses;

// pair key: canonical order == unsigned key order (linear_system.hpp:32-36)
//   bits 31..17: i (1-based, < 2^15), 16..1: j (< 2^16), 0: rel_sign < 0
constexpr int kMaxVars = 32767;

enum Mode : int32_t {
    kModeSearch = 0,  // optimize_system iteration: slot from (master, salt, iteration, p)
    kModeRun = 1,     // explicit ProcessConfig per process (run_cse parity hook)
    kModeDump = 2     // replay prefix, dump pairs (count_pairs parity hook / base candidates)
};

// kernel forms (dense Greedy-Intersections layouts): the bitmap-pruned
// scoring (gi_score_bm) and the small-list loop (gi_dense_small) are each
// compiled only into the instantiations whose systems run them, so no
// instantiation carries the others' code and registers
constexpr int kFormBm = 1;     // per-variable candidate bitmaps (the system's gi_bm)
constexpr int kFormSmall = 2;  // lists of at most 32 candidates, no pruning (bitmaps too)

// device -> host only: a candidate list outgrew a shrunk session capacity
// (the session re-runs the iteration at full capacity; never user-visible)
constexpr int kErrCandOverflow = -100;

// Device-resident loop state of one system (optimize_system's loop variables,
// parallel_search.hpp:226-271): the incumbent, the iteration counter, patience
// and the active flag live in HBM and are advanced by the barrier kernel, so
// iterations run back to back without the host (CUDA graph replays); the host
// reads this struct after a batch.
struct IncState {
    int32_t have;
    int32_t cost;
    int32_t len;
    int32_t strategy;
    u64 seed;
    int32_t improved;   // set by the last barrier
    int32_t best_p;     // global id of the iteration's best process
    int32_t best_cost;
    int32_t iteration;  // iterations completed
    int32_t active;     // 1 while searching (cleared by patience / max_iterations)
    int32_t unchanged;  // iterations without improvement (patience counter)
    u64 steps;          // accumulated selected substitutions
    u64 replayed;
    u64 wops;           // accumulated algorithmic word-ops
    u64 steps_by_strategy[8];  // selected substitutions per StrategyKind of the process
};

// Device clock of a session (%globaltimer, ns): per launch group the first
// search block's start and the last one's end in the current iteration, the
// exchange start, and the accumulated spans (graph replays included).
struct LoopClock {
    u64 gstart[kMaxSys];
    u64 gend[kMaxSys];
    u64 xstart;
    u64 group_ns[kMaxSys];
    u64 search_ns;    // union of the iteration's search-group spans
    u64 exchange_ns;  // pack -> end of the barrier kernels
    u64 iterations;   // iterations the clock saw
    u64 t_begin;      // the search's first launch (wall budget origin)
};

struct SysDesc {
    // problem (base state, shared read-only by every block of the system)
    int32_t n_x, n_e, naive;
    int32_t words;    // ceil(n_e / 64): words a mask needs (the launch may use more)
    int32_t coin_words;  // gi coin buffer (u32 words) per block
    int32_t gi_dense;    // 1: gi by the reference's O(m) loop per candidate; 0: O(deg) walk
    int32_t gi_bm;       // dense: per-variable candidate bitmaps in the layout (O(m/32 + deg) scoring)
    int32_t gi_prune;    // > 0: near-best pruning (walk: exact folds only near the best; dense: from gi_prune candidates on); 0: off
    int32_t vcap;     // variable capacity = n_x + naive
    int32_t mcap;     // candidate capacity (<= pair occurrences / 2)
    int32_t sub_cap;  // record stride (u32 keys) = naive + 1
    const u64* base_masks;  // [n_x][2W]: P words then N words per variable
    const u32* base_keys;   // base candidate list (canonical order) or null
    const u16* base_cnts;
    int32_t base_m;

    int32_t mode;
    int32_t n_local;      // processes of this system in this launch
    int32_t p0;           // global process id of local process 0
    int32_t p_stride;     // global id of local process lp = p0 + lp * p_stride (flip mode: M)
    int32_t stream_comp;  // >= 0: process stream = mt19937_64(mix_seed{slot.seed, comp}) (flip mode)
    int32_t block_begin;  // first block of this system

    // kModeSearch slot derivation (assign_strategies, parallel_search.hpp:172-208)
    u64 master_seed;
    u64 salt;
    int32_t iteration;
    int32_t forced;  // -1 none
    double weights[7];
    double weight_total;
    double mix[4];
    // kModeRun
    const tcse_process_config* cfgs;  // [n_local]

    // prefixes
    const u8* reinit;     // [n_local] or null (search mode)
    const u32* inc_keys;  // incumbent record (reinit prefix source)
    int32_t inc_len;
    // session: iteration, incumbent length and the active flag come from the
    // device loop state instead of iteration / inc_len (null: host-driven)
    const IncState* loop;
    // prefix snapshots (session search mode, else null): the state after k
    // substitutions of the incumbent, k = 1..snap_k, published by the
    // launch's builder block as it replays (snap_ready = newest k, reset by
    // the prep kernel); snapshot k at snap + (k - 1) * snap_stride:
    // [V, m, cost, 0] | masks u64[V][2W] | keys u32 at snap_koff | cnts u16 at snap_coff
    unsigned char* snap;
    u32* snap_ready;
    int32_t snap_k, snap_stride, snap_koff, snap_coff;
    const u32* prefix;  // fixed prefix (run / dump modes)
    int32_t prefix_len;

    // dump mode
    int32_t dump_min_count;
    int32_t dump_cap;
    u32* dump_keys;
    u16* dump_cnts;
    int32_t* dump_n;

    // outputs, indexed by local process
    int32_t* out_cost;
    int32_t* out_len;  // record length (prefix + own)
    int32_t* out_own;  // substitutions selected by this process (steps)
    int32_t* out_strategy;
    u64* out_seed;
    u64* out_wops;  // algorithmic word-ops per process (roofline), may be null
    u32* out_subs;  // [n_local][sub_cap]
    u64* trace;     // [n_local][trace_stride] or null
    int32_t trace_stride;
    int32_t* err;   // first error code of the launch (0 = none)
    int32_t* err_pos;
};

// per-process configuration handed from the prep kernel to the search kernel
struct SlotRec {
    int32_t strategy;  // -1: skip (system inactive or the launch hit an error)
    int32_t reinit;    // > 0: restart from a prefix of the incumbent, whose length this is
    int32_t rng;     // the process draws from its mt19937_64 stream
    int32_t pad;
    double alpha, beta, p_greedy;
    u64 seed;
    double mix[4];
};

struct LaunchDesc {
    int32_t nsys;
    int32_t total_blocks;
    SlotRec* slots;  // [total_blocks]
    u64* rng;        // [total_blocks][kCkpt] checkpoints of the mt19937_64 seeding chain
    int32_t* perm;   // [total_blocks] launch order -> block (grouped by strategy), or null
    int32_t* hist;   // [kMaxSys][kHistStride] (strategy, work class) histogram + placement cursors
    const SysDesc* table;  // > kMaxSys systems (flip mode): device table, blocks contiguous per system
    int32_t table_n;
    int32_t group;         // launch group index (clock stamps)
    int32_t n_builders;    // blocks 0..n_builders-1 build sys[b]'s prefix snapshots; processes follow
    LoopClock* clock;      // or null
    SysDesc sys[kMaxSys];
};

// Exchange payload of one rank for one system (int32 words, fixed size):
//   [0, n_max)            this rank's per-process costs (global ids part(r)..)
//   n_max + 0             1 if the rank ran at least one process
//   n_max + 1             global id of the rank's best process (min cost, lowest id)
//   n_max + 2, 3, 4..5    its record length, strategy, seed (lo, hi)
//   n_max + 6             the rank's launch error (0 = none): every rank then
//                         skips the barrier and reports it (a capacity retry
//                         re-runs the iteration on every rank)
//   n_max + 7             1 if the rank's clock passed the wall budget at pack
//                         time (rank 0's word stops every rank)
//   n_max + kHdr ..       its record (u32 pair keys), sub_cap entries
// With world = 1 the gathered buffer is this payload itself, so one code
// path serves every world size.
constexpr int kHdr = 8;

struct XchgDesc {
    int32_t n, world, n_max, sys_off, words_total;  // layout (words)
    int32_t n_local, p0, sub_cap;
    const int32_t* cost;
    const int32_t* len;
    const int32_t* own;
    const int32_t* strat;
    const u64* seed;
    const u64* wops;
    const u32* subs;
    int32_t* send;        // this rank's payload (all systems), device
    const int32_t* recv;  // [world][words_total], device
    IncState* inc;
    u32* inc_keys;
    u8* reinit_next;  // [n]
    double fraction;
    int32_t hist_n;
    int32_t patience, max_iterations;
    // barrier scratch: nblk tally blocks over the n gathered costs; the last
    // one to arrive (done counter) runs the barrier itself
    int32_t nblk;
    u64* part_min;       // [nblk] (cost << 32 | p)
    int32_t* part_hist;  // [nblk][hist_n] cost histograms
    u64* part_sums;      // [nblk][3 + 8]: steps, replayed, word-ops, steps per strategy
    int32_t* done;       // arrival counter of this system's tally blocks (reset by the last)
    int32_t* sel;        // [4]: reinit threshold cost, ties to take, count (flags kernel)
};

struct XchgLaunch {
    int32_t nsys;
    int32_t* err;       // the launch error word of this rank (shared with the search launches)
    int32_t* all_done;  // arrival counter of every barrier block of the launch (clock)
    LoopClock* clock;
    u64 budget_ns;      // wall budget (0 = none): rank 0's clock decides for every rank
    XchgDesc x[kMaxSys];
};

// Shared-memory carve of one process (block).  Byte offsets; the update view
// (candidate merge scratch, including the copy of the old keys the list is
// rewritten from) and the gi view (adjacency lists, prefix sums, coin bits)
// are never live at the same time and share one region.
struct Lay {
    u32 mask, keys0, cnts0;
    u32 tcnt, ncp, ncn, aux, newexcl, kcopy;                        // update view
    u32 qbase, wp, nA, nB, aoff, bs, cursor, alist, wbt, coin, bm;  // gi view
    u32 coin_cap;  // coin bits of the gi view
    u32 total;     // bytes
};

__host__ __device__ inline u32 al16(u32 x) { return (x + 15u) & ~15u; }

// row stride (u32 words) of the per-variable candidate bitmaps: odd, so the
// rows of 32 different variables start in 32 different shared-memory banks
// (an even stride of 8 words put them in 4 banks: 8-way conflicts on every
// row access)
__host__ __device__ inline u32 bm_stride(int mcap) { return (u32(mcap + 31) >> 5) | 1u; }

__host__ __device__ inline u32 carve(Lay* L, int W, int nt, int vcap, int mcap, int n_e, int coin_words,
                                      int gi_dense, int gi_bm) {
    const u32 NW = u32(nt / 32);
    const u32 vc = u32(vcap), mc = u32(mcap);
    u32 o = 0;
    L->mask = o;  // must stay 0: search.cu mask_base() relies on it
    o += al16(vc * 2u * u32(W) * 8u);
    // one candidate list: the update copies the old keys into its scratch
    // (kcopy) and rewrites the list in place
    L->keys0 = o;
    o += al16(mc * 4u);
    L->cnts0 = o;
    o += al16(mc * 2u);
    const u32 uni = o;
    L->tcnt = o;
    o += al16(mc * 2u);
    L->ncp = o;
    o += al16((vc + 1u) * 2u);
    L->ncn = o;
    o += al16((vc + 1u) * 2u);
    L->aux = o;
    o += al16(mc * 4u);
    L->newexcl = o;
    o += al16((vc + 2u) * 4u);
    L->kcopy = o;
    o += al16(mc * 4u);
    const u32 end_upd = o;
    o = uni;
    L->qbase = o;
    o += al16((mc + 1u) * 4u);
    L->nA = o;
    o += al16((vc + 1u) * 4u);
    if (!gi_dense) {  // walk view: prefix sums and per-variable adjacency
        L->wp = o;
        o += al16((mc + 1u) * 4u);
        L->nB = o;
        o += al16((vc + 1u) * 4u);
        L->aoff = o;
        o += al16((vc + 1u) * 4u);
        L->bs = o;
        o += al16((vc + 1u) * 4u);
        L->cursor = o;
        o += al16((vc + 1u) * 4u);
        L->alist = o;
        o += al16(mc * 2u);
        L->bm = L->nA;
    } else {  // dense view: prefix sums for the exact folds of near-best candidates,
              // per-variable candidate bitmaps (bit s of row v: candidate s holds v)
        L->wp = o;
        o += al16((mc + 1u) * 4u);
        L->bm = o;
        if (gi_bm)
            o += al16((vc + 1u) * bm_stride(mcap) * 4u);
        L->nB = L->aoff = L->bs = L->cursor = L->alist = L->nA;
    }
    L->wbt = o;
    o += al16(u32(n_e + 2) * 8u);
    L->coin = o;
    L->coin_cap = u32(coin_words) * 32u;
    o += al16(u32(coin_words + 2) * 4u);  // + 2: the scoring windows read two words past a candidate's coins
    o = o > end_upd ? o : end_upd;
    (void)NW;
    L->total = o;
    return o;
}

// static shared memory of a search block next to the carved dynamic part
// (search.cu: the mt19937_64 state, reduction slots, broadcast words, the
// layout itself and the kernel's per-process scalars), an upper bound for
// occupancy estimates and the 227 KB limit
constexpr int kStaticSmem = 4096;

}  // namespace tcse
