/*
 * tcse.h — C ABI of the B200-native ternary-CSE search path.
 *
 * This is the ONLY way host code reaches the CUDA kernels.  Every entry point
 * replaces one function of the reference's header-only C++ library
 * (/root/reference/proj/include/terncse/, "terncse"); the citation next to each
 * declaration names the function it stands in for.  The reference has no
 * plugin/FFI layer of its own, so the seam is the function
 * contract of optimize_system / optimize_scheme; include/tcse/terncse_gpu.hpp
 * is the C++ adapter a maintainer drops into the reference, and INTEGRATION.md
 * shows the ctypes / C++ bindings.
 *
 * Conventions (all mirror the reference):
 *   - variable ids are signed and 1-based (+i = coefficient +1 on x_i,
 *     linear_system.hpp:63-65); fresh variable t gets id n_x + t
 *     (linear_system.hpp:72-75);
 *   - a pair is (i, j, rel_sign) with i < j, meaning x_i + rel_sign*x_j
 *     (CanonicalPair, linear_system.hpp:20-28); canonical order is
 *     (i, j, '+' before '-') (linear_system.hpp:30-36);
 *   - every call is synchronous; buffers are caller-allocated; no
 *     library-owned heap crosses the ABI;
 *   - return 0 on success or a negative TCSE_E* code; tcse_last_error()
 *     (thread-local) carries the reference's message text where one exists
 *     ("search config: ...", "replay_prefix: unreplayable pair at position N",
 *     parallel_search.hpp:117-140, cse_engine.hpp:53).
 *
 * Results never depend on the device, the number of devices or any execution
 * knob: slots are keyed by (master_seed, salt, iteration, GLOBAL process id)
 * exactly as assign_strategies does (parallel_search.hpp:172-208), and every
 * process replays the reference's std::mt19937_64 stream bit-for-bit.
 */
#ifndef TCSE_H
#define TCSE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TCSE_ABI_VERSION 2

/* error codes */
enum {
    TCSE_OK = 0,
    TCSE_EINVAL = -1,    /* bad argument / config ("search config: ...") */
    TCSE_EREPLAY = -2,   /* replay_prefix: unreplayable pair (cse_engine.hpp:50-54) */
    TCSE_ECAPACITY = -3, /* caller buffer or device capacity too small */
    TCSE_ECUDA = -4,     /* CUDA runtime error or no device */
    TCSE_ENCCL = -5,     /* multi-rank exchange failed */
    TCSE_EVERIFY = -6    /* optimize_scheme: internal verification failed (parallel_search.hpp:332-333) */
};

/* StrategyKind, same order and values (strategies.hpp:13-21) */
enum {
    TCSE_GREEDY = 0,
    TCSE_GREEDY_ALTERNATIVE = 1,
    TCSE_WEIGHTED_RANDOM = 2,
    TCSE_GREEDY_RANDOM = 3,
    TCSE_GREEDY_INTERSECTIONS = 4,
    TCSE_MIXED = 5,
    TCSE_GREEDY_POTENTIAL = 6,
    TCSE_STRATEGY_COUNT = 7
};

/* CanonicalPair (linear_system.hpp:22-28) */
typedef struct tcse_pair {
    int32_t i;
    int32_t j;
    int32_t rel_sign; /* +1 or -1 */
} tcse_pair;

/* PairCount (linear_system.hpp:125-128) */
typedef struct tcse_pair_count {
    tcse_pair pair;
    int32_t count;
} tcse_pair_count;

/* LinearSystem without fresh definitions (linear_system.hpp:76-122), CSR:
 * expression r holds terms[row_ptr[r] .. row_ptr[r+1]), signed 1-based ids in
 * [1, n_x]; the same validation as the LinearSystem constructor applies. */
typedef struct tcse_system {
    int32_t n_x;
    int32_t n_e;
    const int32_t* row_ptr; /* n_e + 1 entries */
    const int32_t* terms;
} tcse_system;

/* ProcessConfig (strategies.hpp:46-53) */
typedef struct tcse_process_config {
    int32_t strategy;
    int32_t reserved;
    double alpha;
    double beta;
    double p_greedy;
    uint64_t seed;
    double mix_weights[4]; /* gi, ga, gr, wr */
} tcse_process_config;

/* SearchConfig (parallel_search.hpp:44-53) minus flip mode and threads, plus
 * three stop knobs that are not in the reference (0 = off).  Call
 * tcse_default_search_config() to get the reference defaults. */
typedef struct tcse_search_config {
    int32_t n_processes; /* 0 = 256, as optimize_system does (parallel_search.hpp:224) */
    int32_t patience;
    double strategy_weights[TCSE_STRATEGY_COUNT];
    double reinit_fraction;
    uint64_t master_seed;
    int32_t forced_strategy; /* -1 = none (draw from weights) */
    int32_t max_iterations;  /* 0 = until patience (reference behaviour) */
    double mix_weights[4];   /* ProcessConfig default {8,4,2,1} */
    double wall_budget_s;    /* 0 = none; else every system stops at the first iteration
                                barrier after this much device time from the search's first
                                launch — the fixed-wall-time run SURVEY.md 8(d) drives through
                                on_iteration, decided on the device (rank 0's clock for every
                                rank), so it needs no host turn per iteration */
} tcse_search_config;

/* SolutionRecord (cse_engine.hpp:18-23).  subs is caller-allocated with room
 * for cap pairs; cap >= naive_cost(system) always suffices because every
 * substitution lowers the cost by at least one. */
typedef struct tcse_record {
    tcse_pair* subs;
    int32_t cap;
    int32_t n_subs;
    int32_t cost;
    int32_t strategy;
    uint64_t seed;
} tcse_record;

/* A matrix multiplication scheme (m, n, p : r) with ternary coefficients
 * (Scheme, scheme.hpp:20-27), row-major int8 in {-1, 0, 1}:
 * u is r x (m*n), v is r x (n*p), w is (m*p) x r. */
typedef struct tcse_scheme {
    int32_t m, n, p, r;
    const int8_t* u;
    const int8_t* v;
    const int8_t* w;
} tcse_scheme;

/* CheckMethod (scheme.hpp:29); TCSE_CHECK_AUTO = check_scheme_auto's rule
 * (parallel_search.hpp:296-302: rank >= 200 -> randomized product check) */
enum { TCSE_CHECK_AUTO = -1, TCSE_CHECK_BRENT = 0, TCSE_CHECK_PRODUCT = 1 };

/* SchemeCheckReport (scheme.hpp:31-35); first_violation is "" when valid,
 * else the reference's wording: "brent(i,j,k,l,i2,j2)" or
 * "trial T mismatch at c[i][j]". */
typedef struct tcse_check_report {
    int32_t valid;
    int32_t method; /* TCSE_CHECK_BRENT or TCSE_CHECK_PRODUCT */
    char first_violation[64];
} tcse_check_report;

/* FlipModeConfig (parallel_search.hpp:24-29) */
typedef struct tcse_flip_config {
    int32_t m_schemes;
    int32_t flips_min;
    int32_t flips_max;
    int32_t reserved;
} tcse_flip_config;

/* optimize_with_flips result (SearchReport of flip mode): the carried scheme
 * (caller-allocated u/v/w with the input's shapes), the three component
 * records (caller-allocated, cap >= r * max(m*n, n*p) suffices), their naive
 * costs on the carried scheme, and the winning scheme's id: slot 0 =
 * "original", else "flip-<scheme_iteration>-<scheme_slot>". */
typedef struct tcse_flip_result {
    int8_t* u;
    int8_t* v;
    int8_t* w;
    tcse_record comp[3];
    int32_t naive[3];
    int32_t iterations;
    int32_t scheme_iteration;
    int32_t scheme_slot;
    int32_t total;
} tcse_flip_result;

/* execution counters (not part of any reference result) */
typedef struct tcse_stats {
    uint64_t steps;        /* selected substitutions (replayed prefixes excluded) */
    uint64_t replayed;     /* prefix substitutions replayed by reinit processes */
    uint64_t processes;    /* process runs (iterations x processes of the systems still searching) */
    uint64_t launches;     /* search-kernel launches (one per launch group per iteration) */
    int32_t iterations;    /* iteration barriers passed (max over systems) */
    int32_t retries;       /* iterations re-run at full candidate capacity (session layouts are
                              sized from the starting list; results never depend on it) */
    double kernel_ms;      /* device clock: summed spans of the iterations' search kernels
                              (first search block start -> last block end, all groups) */
    double step_ms;        /* summed device time of the iterations (CUDA events around them) */
    double wall_ms;        /* whole call, host clock */
    double exchange_ms;    /* device clock: pack -> all-gather -> barrier kernels, summed */
    uint64_t h2d_bytes;    /* host->device bytes copied by the call */
    uint64_t d2h_bytes;    /* device->host bytes copied by the call */
    uint64_t wops;         /* algorithmic word-intersections (SURVEY.md 8(d) model) */
    uint64_t steps_by_strategy[TCSE_STRATEGY_COUNT]; /* steps by the process's StrategyKind */
    int32_t n_groups;      /* launch groups (one kernel instantiation each) */
    int32_t group_nt[4];   /* threads per process of each group */
    int32_t group_words[4];/* mask words W of each group */
    int32_t reserved;
    double group_ms[4];    /* device clock: summed search-kernel span of each group */
    uint64_t group_wops[4];/* word-ops of each group's systems */
    uint64_t graph_launches; /* iterations replayed from the captured CUDA graph */
    uint64_t host_syncs;   /* host synchronisations (one per batch of iterations) */
    uint64_t kernel_launches; /* kernels launched for the kept iterations */
} tcse_stats;

/* Called on the calling thread after every iteration barrier, like
 * optimize_system's on_iteration (parallel_search.hpp:222, 267-268).  A
 * nonzero return stops the search at this barrier (fixed wall-time budgets). */
typedef int (*tcse_iter_cb)(int32_t system_index, int32_t iteration,
                            const tcse_record* incumbent, void* user);

/* Multi-rank exchange: all-gather of `bytes` bytes from every rank into
 * recv (world * bytes, rank-major).  Returns 0 on success. */
typedef int (*tcse_allgather_fn)(const void* send, void* recv, size_t bytes, void* user);

typedef struct tcse_ctx tcse_ctx;
typedef struct tcse_search tcse_search;

const char* tcse_last_error(void);
int32_t tcse_abi_version(void);
int32_t tcse_device_count(void);

/* reference defaults: weights {0,4,1,2,8,0.1,0.01}, reinit 0.40, patience 10,
 * seed 0, no forced strategy (parallel_search.hpp:31-53) */
void tcse_default_search_config(tcse_search_config* cfg);

/* upper bound on record length for a system (= its naive cost) */
int32_t tcse_naive_cost(const tcse_system* sys);

/* Owns the device, its stream, device pools and (optionally) the rank
 * partition.  NULL on failure (see tcse_last_error). */
tcse_ctx* tcse_create(int32_t device);
void tcse_destroy(tcse_ctx* ctx);

/* Launch on a caller-owned cudaStream_t (NULL = the context's own stream),
 * e.g. torch.cuda.current_stream().cuda_stream so that caller-side CUDA
 * events bracket the work. */
int tcse_set_stream(tcse_ctx* ctx, void* stream);

/* Several devices of this process as ONE context: one
 * sub-context per device with its own stream and an NCCL communicator
 * (ncclCommInitAll).  tcse_optimize_system(s) on it partitions the processes
 * across the devices (rank r = devices[r]) and runs one host thread per
 * device; each iteration's payload all-gather is an ncclAllGather over
 * NVLink on the device streams, inside the iteration's CUDA graph.  Results
 * are identical to one device.  Other calls run on devices[0].  NULL on
 * failure (no NCCL, duplicate device). */
tcse_ctx* tcse_create_devices(const int32_t* devices, int32_t n_devices);
int32_t tcse_context_devices(const tcse_ctx* ctx);

/* One process per GPU (torchrun / MPI style): rank 0 makes an NCCL unique
 * id (128 bytes), the caller broadcasts it, every rank attaches it to its
 * context; the library then runs the payload all-gather itself
 * (ncclAllGather on the context stream, captured in the iteration graph).
 * NCCL is bound at run time (the copy already in the process, else
 * TCSE_NCCL_LIBRARY, else libnccl.so.2); tcse_nccl_available() says whether
 * it could be loaded. */
int32_t tcse_nccl_available(void);
int tcse_nccl_unique_id(void* unique_id_128);
int tcse_set_nccl(tcse_ctx* ctx, const void* unique_id_128, int32_t rank, int32_t world);

/* Process partition across ranks: this rank runs global process ids
 * [floor(n*rank/world), floor(n*(rank+1)/world)) of every iteration; the
 * per-iteration payloads (costs + local best record) are exchanged either by
 * the host allgather callback or by a caller-run device collective around
 * tcse_search_step_begin/end.  world = 1 (default) needs neither.  The
 * result is identical for every world size. */
int tcse_set_partition(tcse_ctx* ctx, int32_t rank, int32_t world,
                       tcse_allgather_fn allgather, void* user);

/* count_pairs (linear_system.hpp:151-161) of the state replay_prefix(sys,
 * prefix) (cse_engine.hpp:47-57), computed on the device.  min_count = 1
 * returns every pair by popcount of the occurrence masks; min_count = 2
 * returns the kernel's incrementally maintained candidate list
 * (PairStats::candidates, linear_system.hpp:141-148).  Output in canonical
 * order; *n_out = number of pairs (may exceed cap -> TCSE_ECAPACITY). */
int tcse_count_pairs(tcse_ctx* ctx, const tcse_system* sys, const tcse_pair* prefix,
                     int32_t n_prefix, int32_t min_count, tcse_pair_count* out,
                     int32_t cap, int32_t* n_out);

/* n independent run_cse calls (cse_engine.hpp:29-43) in one launch:
 * process b runs `std::mt19937_64 rng(cfgs[b].seed); run_cse(replay_prefix(
 * sys, prefix), cfgs[b], rng)`.  out[b].subs receives only the substitutions
 * run_cse selected (the prefix is not repeated); out[b].cost is total_cost of
 * the final state.  trace (optional, n * trace_stride entries): per process,
 * the FNV-1a-64 hash of the candidate list (pair, count) seen at each step,
 * in canonical order, as the oracle computes it. */
int tcse_run_cse(tcse_ctx* ctx, const tcse_system* sys, const tcse_pair* prefix,
                 int32_t n_prefix, const tcse_process_config* cfgs, int32_t n,
                 tcse_record* out, uint64_t* trace, int32_t trace_stride,
                 tcse_stats* stats);

/* optimize_system (parallel_search.hpp:220-273): portfolio search over one
 * expression set.  best receives the incumbent record (prefix included),
 * *iterations the iteration count of SystemSearchResult. */
int tcse_optimize_system(tcse_ctx* ctx, const tcse_system* sys, const tcse_search_config* cfg,
                         uint64_t stream_salt, tcse_iter_cb cb, void* user,
                         tcse_record* best, int32_t* iterations, tcse_stats* stats);

/* n_systems independent optimize_system calls run CONCURRENTLY in shared
 * launches (system s uses stream salt salts[s]); result s is identical to
 * tcse_optimize_system(systems[s], cfg, salts[s]).  optimize_scheme runs U, V
 * and W this way instead of sequentially (parallel_search.hpp:329-341). */
int tcse_optimize_systems(tcse_ctx* ctx, int32_t n_systems, const tcse_system* systems,
                          const tcse_search_config* cfg, const uint64_t* salts,
                          tcse_iter_cb cb, void* user, tcse_record* best,
                          int32_t* iterations, tcse_stats* stats);

/* The same search, advanced one iteration barrier at a time (what
 * tcse_optimize_systems loops over): create uploads and prepares the systems,
 * each step runs one iteration for every still-active system and reports how
 * many remain active (0 = all converged or the callback stopped the search),
 * result copies the incumbents out. */
int tcse_search_create(tcse_ctx* ctx, int32_t n_systems, const tcse_system* systems,
                       const tcse_search_config* cfg, const uint64_t* salts, tcse_iter_cb cb,
                       void* user, tcse_search** out);
int tcse_search_step(tcse_search* search, int32_t* n_active);

/* Up to max_iterations iterations as a device-resident loop: the iteration
 * (prep, place, search, pack, [NCCL all-gather], barrier) is a captured CUDA
 * graph replayed back to back, patience and max_iterations are evaluated on
 * the device, and the host synchronises once per batch (a batch = the
 * iterations the search is certain to run).  An on_iteration callback or a
 * host all-gather callback needs a host turn per iteration and runs them one
 * at a time.  tcse_optimize_systems is create + run + result. */
int tcse_search_run(tcse_search* search, int32_t max_iterations, int32_t* n_active);

/* The same iteration in two phases around a caller-run collective (world > 1
 * without an allgather callback, e.g. ncclAllGather / torch.distributed
 * all_gather_into_tensor over NVLink).  begin launches the iteration on the
 * context's stream and writes this rank's exchange payload (per-process
 * costs of its slice + its best record, tcse_search_payload_bytes() bytes)
 * to send_dev; the caller all-gathers every rank's payload into recv_dev
 * (world x payload bytes, rank order) ordered after that stream; end runs the
 * iteration barrier from recv_dev.  NULL buffers = the library's own (world
 * 1, or the host callback). */
size_t tcse_search_payload_bytes(tcse_search* search);
int tcse_search_step_begin(tcse_search* search, void* send_dev);
int tcse_search_step_end(tcse_search* search, const void* recv_dev, int32_t* n_active);
int tcse_search_result(tcse_search* search, tcse_record* best, int32_t* iterations,
                       tcse_stats* stats);
void tcse_search_destroy(tcse_search* search);

/* optimize_with_flips (parallel_search.hpp:354-518) with the search on the
 * device: every iteration M scheme variants (slot 0 the input, the others
 * random_flip chains seeded by mix_seed{master, 0xf11b5, iteration, slot},
 * each validity-checked), processes dealt round-robin to the variants, all
 * (process, component) runs in one launch, prefix sharing for the original,
 * per-variant component minima.  Requires m_schemes >= 2 (m_schemes = 1 is
 * plain optimize_scheme) and world = 1. */
int tcse_optimize_with_flips(tcse_ctx* ctx, const tcse_scheme* scheme, const tcse_search_config* cfg,
                             const tcse_flip_config* flip, tcse_flip_result* out, tcse_stats* stats);

/* Measured shared-memory word-op peak of this device (roofline
 * denominator): a microbenchmark of the search kernel's inner operation
 * (two 8-byte LDS, AND, POPC, accumulate) over every SM.  *gops = Gword-ops/s. */
int tcse_microbench_wordops(tcse_ctx* ctx, double* gops);

/* Measured integer issue peaks of this device (the search kernel's
 * instruction mix): gops[0..5] = G thread-operations/s of
 * IADD3, LOP3, POPC, SHFL, 4-byte LDS and 8-byte LDS, each from 8
 * independent chains per thread on every SM at full occupancy. */
int tcse_microbench_pipes(tcse_ctx* ctx, double* gops);

/* Batched scheme verification on the device: for every
 * scheme, check_structure (scheme.hpp:54-62; ternary coefficients, positive
 * dimensions) then verify_brent (scheme.hpp:68-95: every Brent identity,
 * exact integers, first violation in (i,j,k,l,i2,j2) order) or
 * verify_by_product (scheme.hpp:99-137: `trials` random integer products,
 * entries uniform_int(-8,8) from mt19937_64(seed), first mismatch in
 * (trial,i,j) order) as `method` says; TCSE_CHECK_AUTO picks per scheme like
 * check_scheme_auto.  Reports are identical to the reference's.  Errors:
 * TCSE_EINVAL with check_structure's message ("scheme: ...") for the first
 * malformed scheme, or "verify_by_product: trials must be >= 1". */
int tcse_verify_schemes(tcse_ctx* ctx, const tcse_scheme* schemes, int32_t count, int32_t method,
                        int32_t trials, uint64_t seed, tcse_check_report* out);

/* A flip-graph walk on the host (no GPU): `flips` consecutive random_flip
 * moves (scheme.hpp:204-276) drawn from std::mt19937_64 `rng_seed`, as the
 * reference's fixture generator and optimize_with_flips chain them.  u/v/w
 * are caller-allocated with the input's shapes.  Identical output to the
 * reference with the same libstdc++ (the walk uses std::shuffle). */
int tcse_flip_walk(const tcse_scheme* scheme, uint64_t rng_seed, int32_t flips,
                   int8_t* u, int8_t* v, int8_t* w);

/* Host-side result/verification API kept from the reference (no GPU):
 * replay_prefix + total_cost + expand_and_verify (linear_system.hpp:193-258,
 * cse_engine.hpp:47-57).  Returns 1 if the record replays, its cost matches
 * *cost_out (written) and the expansion equals the original, 0 if not, <0 on
 * a replay error. */
int tcse_verify_record(const tcse_system* sys, const tcse_pair* subs, int32_t n_subs,
                       int32_t* cost_out);

#ifdef __cplusplus
}
#endif

#endif /* TCSE_H */
