/*
 * tcse_oracle.h — CPU restatement of the reference's search path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this code, and
 * only as the checker.  The product (paper_2512_13365_b200/libtcse.so) never
 * links or calls it.
 *
 * Plain C11 restatement of /root/reference/proj/include/terncse/{rng,
 * linear_system,strategies,cse_engine,parallel_search}.hpp, including the
 * exact libstdc++ (GCC 13) semantics of std::mt19937_64,
 * std::uniform_int_distribution (Lemire nearly-divisionless, 128-bit) and
 * std::uniform_real_distribution / generate_canonical, so that stochastic
 * trajectories are bit-identical to the reference built with its own Release
 * flags (no FMA contraction).  Pinned against oracle/_ref (the reference
 * compiled from /root/reference) by tests/test_oracle_pin.py and against the
 * golden vectors under tests/golden/.
 *
 * Types are those of the product ABI (include/tcse.h) so results compare
 * field by field.
 */
#ifndef TCSE_ORACLE_H
#define TCSE_ORACLE_H

#include "../include/tcse.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* or_last_error(void);

/* std::mt19937_64 stream: out[0..n) = first n outputs of mt19937_64(seed) */
void or_mt19937_64(uint64_t seed, int32_t n, uint64_t* out);
/* splitmix64 / mix_seed (rng.hpp:8-23) */
uint64_t or_mix_seed(const uint64_t* parts, int32_t n_parts);
/* uniform_int_distribution<size_t>(a, b) and uniform_real_distribution<double>
 * (a, b) draws from mt19937_64(seed): n draws each */
void or_uniform_int(uint64_t seed, uint64_t a, uint64_t b, int32_t n, uint64_t* out);
void or_uniform_real(uint64_t seed, double a, double b, int32_t n, double* out);

/* count_pairs of replay_prefix(sys, prefix); pairs with count >= min_count in
 * canonical order (linear_system.hpp:141-161) */
int or_count_pairs(const tcse_system* sys, const tcse_pair* prefix, int32_t n_prefix,
                   int32_t min_count, tcse_pair_count* out, int32_t cap, int32_t* n_out);

/* std::mt19937_64 rng(cfg->seed); run_cse(replay_prefix(sys, prefix), *cfg, rng)
 * (cse_engine.hpp:29-43); trace as in tcse_run_cse */
int or_run_cse(const tcse_system* sys, const tcse_pair* prefix, int32_t n_prefix,
               const tcse_process_config* cfg, tcse_record* out, uint64_t* trace,
               int32_t trace_cap);

/* one process of an optimize_system iteration (the parallel_for body,
 * parallel_search.hpp:240-252): rng = mt19937_64(slot->seed); if reinit,
 * k ~ U[1, 3*len/4] and replay of the incumbent prefix; then run_cse.  out
 * receives prefix + own substitutions; *own = own substitutions. */
int or_run_process(const tcse_system* sys, const tcse_process_config* slot, int32_t reinit,
                   const tcse_pair* incumbent, int32_t inc_len, tcse_record* out, int32_t* own);

/* assign_strategies (parallel_search.hpp:172-208); out[n] */
int or_assign_strategies(const tcse_search_config* cfg, int32_t iteration, int32_t n,
                         uint64_t salt, tcse_process_config* out);

/* pick_reinit (parallel_search.hpp:149-163) */
int or_pick_reinit(const int32_t* last_cost, int32_t n, double fraction, uint8_t* out);

/* optimize_system (parallel_search.hpp:220-273), sequential; *steps = number
 * of substitutions selected by run_cse (replayed prefixes excluded) */
int or_optimize_system(const tcse_system* sys, const tcse_search_config* cfg, uint64_t salt,
                       tcse_record* best, int32_t* iterations, uint64_t* steps);

/* replay + total_cost + expand_and_verify (linear_system.hpp:193-258) */
int or_verify_record(const tcse_system* sys, const tcse_pair* subs, int32_t n_subs,
                     int32_t* cost_out);

/* FNV-1a-64 over little-endian int32 (i, j, rel_sign) triples */
uint64_t or_sequence_fnv(const tcse_pair* subs, int32_t n);

#ifdef __cplusplus
}
#endif

#endif
