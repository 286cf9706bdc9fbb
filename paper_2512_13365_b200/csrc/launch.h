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
constexpr int kCoinWords = 512;  // 16384 coin bits per gi scoring chunk

// pair key: canonical order == unsigned key order (linear_system.hpp:32-36)
//   bits 31..17: i (1-based, < 2^15), 16..1: j (< 2^16), 0: rel_sign < 0
constexpr int kMaxVars = 32767;

enum Mode : int32_t {
    kModeSearch = 0,  // optimize_system iteration: slot from (master, salt, iteration, p)
    kModeRun = 1,     // explicit ProcessConfig per process (run_cse parity hook)
    kModeDump = 2     // replay prefix, dump pairs (count_pairs parity hook / base candidates)
};

struct SysDesc {
    // problem (base state, shared read-only by every block of the system)
    int32_t n_x, n_e, naive;
    int32_t words;    // ceil(n_e / 64): words a mask needs (the launch may use more)
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

struct LaunchDesc {
    int32_t nsys;
    int32_t total_blocks;
    SysDesc sys[kMaxSys];
};

// per-system state of the iteration reduce (K2)
struct IncState {
    int32_t have;
    int32_t cost;
    int32_t len;
    int32_t strategy;
    u64 seed;
    int32_t improved;  // set by the last reduce
    int32_t best_p;    // global id of the iteration's best process
    int32_t best_cost;
    int32_t reserved;
    u64 steps;         // accumulated selected substitutions
    u64 replayed;
    u64 wops;          // accumulated algorithmic word-ops
};

// smem bytes one block of this system needs at launch word count W
inline int64_t smem_bytes(int W, int vcap, int mcap, int nt) {
    auto al = [](int64_t x) { return (x + 15) & ~int64_t(15); };
    int64_t b = 0;
    b += al(int64_t(vcap) * 2 * W * 8);           // masks
    b += al(int64_t(mcap) * 4) * 2;               // keys x2
    b += al(int64_t(mcap) * 2) * 2;               // cnts x2
    int64_t upd = al(int64_t(mcap) * 2)           // tcnt
                + al(int64_t(vcap + 1) * 2) * 2   // ncp, ncn
                + al(int64_t(mcap) * 4)           // aux
                + al(int64_t(vcap + 2) * 4);      // newexcl
    int64_t gi = al(int64_t(kCoinWords) * 4)      // coin bits
               + al(int64_t(mcap + 1) * 4)        // qbase
               + al(int64_t(vcap + 1) * 4)        // nvar
               + al(int64_t(mcap) * 8) * 2;       // wd, wb
    b += upd > gi ? upd : gi;
    b += 312 * 8;                                 // mt19937_64 state
    b += al(int64_t(nt / 32 + 2) * 8) * 3;        // reduction scratch
    return b;
}

}  // namespace tcse
