// ref_shim.cpp — C entry points over the REFERENCE ITSELF.
//
// TEST INFRASTRUCTURE ONLY (see oracle/tcse_oracle.h).  Compiled by
// oracle/Makefile against the unmodified headers under
// /root/reference/proj/include (no reference source is copied into this
// repository) into oracle/_ref/libterncse_ref.so, with the reference's own
// Release flags (-O3 -DNDEBUG -std=c++20, baseline x86-64).  Used to pin the C
// restatement (tcse_oracle.c), to generate golden vectors, and as the
// "reference" CPU baseline in bench.py.
//
// The only new logic here is ref_optimize_system_counted: optimize_system
// (parallel_search.hpp:220-273) re-expressed on top of the reference's own
// public pieces (assign_strategies, detail::pick_reinit, detail::parallel_for,
// replay_prefix, run_cse) so that substitution steps can be counted and a
// wall budget enforced at an iteration barrier; tests assert it returns the
// same record as the real optimize_system.
#include <terncse/io.hpp>
#include <terncse/parallel_search.hpp>

#include <atomic>
#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include "../include/tcse.h"

using namespace terncse;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& what) {
    g_err = what;
    return code;
}

LinearSystem to_system(const tcse_system* s) {
    std::vector<std::vector<int>> rows(std::size_t(s->n_e));
    for (int r = 0; r < s->n_e; ++r)
        for (int t = s->row_ptr[r]; t < s->row_ptr[r + 1]; ++t)
            rows[std::size_t(r)].push_back(s->terms[t]);
    return LinearSystem(s->n_x, rows);
}

std::vector<CanonicalPair> to_pairs(const tcse_pair* p, int n) {
    std::vector<CanonicalPair> out;
    for (int t = 0; t < n; ++t)
        out.push_back({p[t].i, p[t].j, p[t].rel_sign});
    return out;
}

ProcessConfig to_pc(const tcse_process_config* c) {
    ProcessConfig pc;
    pc.strategy = StrategyKind(c->strategy);
    pc.alpha = c->alpha;
    pc.beta = c->beta;
    pc.p_greedy = c->p_greedy;
    pc.seed = c->seed;
    for (int k = 0; k < 4; ++k)
        pc.mix_weights[std::size_t(k)] = c->mix_weights[k];
    return pc;
}

void from_pc(const ProcessConfig& pc, tcse_process_config* c) {
    std::memset(c, 0, sizeof *c);
    c->strategy = int32_t(pc.strategy);
    c->alpha = pc.alpha;
    c->beta = pc.beta;
    c->p_greedy = pc.p_greedy;
    c->seed = pc.seed;
    for (int k = 0; k < 4; ++k)
        c->mix_weights[k] = pc.mix_weights[std::size_t(k)];
}

SearchConfig to_cfg(const tcse_search_config* c, unsigned threads) {
    SearchConfig cfg;
    cfg.n_processes = c->n_processes;
    for (int k = 0; k < 7; ++k)
        cfg.strategy_weights[std::size_t(k)] = c->strategy_weights[k];
    cfg.reinit_fraction = c->reinit_fraction;
    cfg.patience = c->patience;
    cfg.master_seed = c->master_seed;
    if (c->forced_strategy >= 0)
        cfg.forced_strategy = StrategyKind(c->forced_strategy);
    cfg.threads = threads;
    return cfg;
}

int put_record(const SolutionRecord& rec, tcse_record* out) {
    if (int(rec.substitutions.size()) > out->cap)
        return fail(TCSE_ECAPACITY, "record capacity exceeded");
    for (std::size_t t = 0; t < rec.substitutions.size(); ++t)
        out->subs[t] = {rec.substitutions[t].i, rec.substitutions[t].j, rec.substitutions[t].rel_sign};
    out->n_subs = int32_t(rec.substitutions.size());
    out->cost = rec.cost;
    out->strategy = int32_t(rec.strategy);
    out->seed = rec.seed;
    return TCSE_OK;
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        return fn();
    } catch (const std::exception& e) {
        const std::string what = e.what();
        if (what.rfind("replay_prefix", 0) == 0)
            return fail(TCSE_EREPLAY, what);
        return fail(TCSE_EINVAL, what);
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_mt19937_64(uint64_t seed, int32_t n, uint64_t* out) {
    std::mt19937_64 g(seed);
    for (int32_t t = 0; t < n; ++t)
        out[t] = g();
}

uint64_t ref_mix_seed(const uint64_t* parts, int32_t n_parts) {
    // mix_seed takes an initializer_list; fold the same way through the
    // public splitmix64 for arbitrary part counts, and cross-check the
    // 4-part form used by assign_strategies
    if (n_parts == 4)
        return mix_seed({parts[0], parts[1], parts[2], parts[3]});
    if (n_parts == 2)
        return mix_seed({parts[0], parts[1]});
    std::uint64_t h = 0x5851f42d4c957f2dULL;
    for (int32_t t = 0; t < n_parts; ++t)
        h = splitmix64(h ^ parts[t]);
    return h;
}

void ref_uniform_int(uint64_t seed, uint64_t a, uint64_t b, int32_t n, uint64_t* out) {
    std::mt19937_64 g(seed);
    std::uniform_int_distribution<std::size_t> d(a, b);
    for (int32_t t = 0; t < n; ++t)
        out[t] = d(g);
}

void ref_uniform_real(uint64_t seed, double a, double b, int32_t n, double* out) {
    std::mt19937_64 g(seed);
    std::uniform_real_distribution<double> d(a, b);
    for (int32_t t = 0; t < n; ++t)
        out[t] = d(g);
}

int ref_count_pairs(const tcse_system* sys, const tcse_pair* prefix, int32_t n_prefix,
                    int32_t min_count, tcse_pair_count* out, int32_t cap, int32_t* n_out) {
    return guarded([&]() -> int {
        const auto state = replay_prefix(to_system(sys), to_pairs(prefix, n_prefix));
        const auto stats = count_pairs(state);
        std::vector<PairCount> all;
        for (const auto& [pair, c] : stats.freq)
            if (c >= min_count)
                all.push_back({pair, c});
        std::sort(all.begin(), all.end(), [](const PairCount& a, const PairCount& b) { return a.pair < b.pair; });
        *n_out = int32_t(all.size());
        for (std::size_t t = 0; t < all.size() && int(t) < cap; ++t)
            out[t] = {{all[t].pair.i, all[t].pair.j, all[t].pair.rel_sign}, all[t].count};
        return int(all.size()) > cap ? fail(TCSE_ECAPACITY, "capacity") : TCSE_OK;
    });
}

int ref_run_cse(const tcse_system* sys, const tcse_pair* prefix, int32_t n_prefix,
                const tcse_process_config* cfg, tcse_record* out) {
    return guarded([&]() -> int {
        const auto state = replay_prefix(to_system(sys), to_pairs(prefix, n_prefix));
        std::mt19937_64 rng(cfg->seed);
        return put_record(run_cse(state, to_pc(cfg), rng), out);
    });
}

int ref_assign_strategies(const tcse_search_config* cfg, int32_t iteration, int32_t n,
                          uint64_t salt, tcse_process_config* out) {
    return guarded([&]() -> int {
        const auto slots = assign_strategies(to_cfg(cfg, 1), iteration, n, salt);
        for (std::size_t p = 0; p < slots.size(); ++p)
            from_pc(slots[p], &out[p]);
        return TCSE_OK;
    });
}

int ref_pick_reinit(const int32_t* last_cost, int32_t n, double fraction, uint8_t* out) {
    const auto chosen = detail::pick_reinit(std::vector<int>(last_cost, last_cost + n), fraction);
    for (int32_t p = 0; p < n; ++p)
        out[p] = uint8_t(chosen[std::size_t(p)]);
    return TCSE_OK;
}

// The real optimize_system, unchanged.
int ref_optimize_system(const tcse_system* sys, const tcse_search_config* cfg, uint64_t salt,
                        uint32_t threads, tcse_record* best, int32_t* iterations) {
    return guarded([&]() -> int {
        const auto result = optimize_system(to_system(sys), to_cfg(cfg, threads), salt);
        *iterations = result.iterations;
        return put_record(result.best, best);
    });
}

// optimize_system re-expressed with the reference's own building blocks plus
// a substitution-step counter and optional stop knobs (max_iterations,
// wall_budget_s checked at the barrier like an on_iteration abort).
int ref_optimize_system_timed(const tcse_system* sys, const tcse_search_config* c, uint64_t salt,
                              uint32_t threads, double wall_budget_s, tcse_record* best,
                              int32_t* iterations, uint64_t* steps, double* seconds,
                              double* iter_secs, uint64_t* iter_steps, int32_t iter_cap) {
    return guarded([&]() -> int {
        const auto t0 = std::chrono::steady_clock::now();
        const LinearSystem base = to_system(sys);
        const SearchConfig cfg = to_cfg(c, threads);
        detail::validate_config(cfg);
        const int n = cfg.n_processes > 0 ? cfg.n_processes : 256;
        std::optional<SolutionRecord> incumbent;
        auto last_cost = std::vector<int>(std::size_t(n), 0);
        auto results = std::vector<SolutionRecord>(std::size_t(n));
        std::atomic<std::uint64_t> counted{0};
        int unchanged = 0, iteration = 0;
        auto t_iter = std::chrono::steady_clock::now();
        std::uint64_t steps_before = 0;
        for (;;) {
            ++iteration;
            const auto slots = assign_strategies(cfg, iteration, n, salt);
            std::vector<char> reinit(std::size_t(n), 0);
            if (iteration >= 2 && incumbent && incumbent->substitutions.size() >= 2)
                reinit = detail::pick_reinit(last_cost, cfg.reinit_fraction);
            detail::parallel_for(std::size_t(n), cfg.threads, [&](std::size_t p) {
                std::mt19937_64 rng(slots[p].seed);
                std::vector<CanonicalPair> prefix;
                if (reinit[p]) {
                    const std::size_t k_max = 3 * incumbent->substitutions.size() / 4;
                    const std::size_t k = std::uniform_int_distribution<std::size_t>(1, k_max)(rng);
                    prefix.assign(incumbent->substitutions.begin(), incumbent->substitutions.begin() + std::ptrdiff_t(k));
                }
                SolutionRecord rec = run_cse(replay_prefix(base, prefix), slots[p], rng);
                counted.fetch_add(rec.substitutions.size(), std::memory_order_relaxed);
                rec.substitutions.insert(rec.substitutions.begin(), prefix.begin(), prefix.end());
                results[p] = std::move(rec);
            });
            std::size_t best_p = 0;
            for (std::size_t p = 0; p < std::size_t(n); ++p) {
                last_cost[p] = results[p].cost;
                if (results[p].cost < results[best_p].cost)
                    best_p = p;
            }
            if (!incumbent || results[best_p].cost < incumbent->cost) {
                incumbent = results[best_p];
                unchanged = 0;
            } else {
                ++unchanged;
            }
            const auto now = std::chrono::steady_clock::now();
            const double elapsed = std::chrono::duration<double>(now - t0).count();
            if (iter_secs && iteration - 1 < iter_cap) {
                iter_secs[iteration - 1] = std::chrono::duration<double>(now - t_iter).count();
                iter_steps[iteration - 1] = counted.load() - steps_before;
            }
            t_iter = now;
            steps_before = counted.load();
            if (unchanged >= cfg.patience)
                break;
            if (c->max_iterations > 0 && iteration >= c->max_iterations)
                break;
            if (wall_budget_s > 0.0 && elapsed >= wall_budget_s)
                break;
        }
        *iterations = iteration;
        *steps = counted.load();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return put_record(*incumbent, best);
    });
}

int ref_optimize_system_counted(const tcse_system* sys, const tcse_search_config* c, uint64_t salt,
                                uint32_t threads, double wall_budget_s, tcse_record* best,
                                int32_t* iterations, uint64_t* steps, double* seconds) {
    return ref_optimize_system_timed(sys, c, salt, threads, wall_budget_s, best, iterations, steps, seconds,
                                     nullptr, nullptr, 0);
}

int ref_verify_record(const tcse_system* sys, const tcse_pair* subs, int32_t n_subs, int32_t* cost_out) {
    return guarded([&]() -> int {
        const auto original = to_system(sys);
        const auto state = replay_prefix(original, to_pairs(subs, n_subs));
        *cost_out = total_cost(state);
        return expand_and_verify(original, state) ? 1 : 0;
    });
}

// Scheme JSON -> extract_systems -> CSR, for fixture checks.  Writes the
// three systems' CSR into caller buffers; returns the digest in digest_out.
int ref_scheme_info(const char* scheme_json, char* digest_out, int32_t* naive_out, int32_t* valid_out) {
    return guarded([&]() -> int {
        const auto s = parse_scheme(scheme_json);
        const auto d = scheme_digest(s);
        std::snprintf(digest_out, 17, "%s", d.c_str());
        const auto systems = extract_systems(s);
        for (int c = 0; c < 3; ++c)
            naive_out[c] = naive_cost(systems[std::size_t(c)]);
        *valid_out = verify_brent(s).valid ? 1 : 0;
        return TCSE_OK;
    });
}

// optimize_scheme (parallel_search.hpp:314-345) -> report_to_json (io.hpp:250-266)
int ref_optimize_scheme_json(const char* scheme_json, const tcse_search_config* c, uint32_t threads,
                             char* out, int32_t cap, int32_t* n_out) {
    return guarded([&]() -> int {
        const auto report = optimize_scheme(parse_scheme(scheme_json), to_cfg(c, threads));
        const auto text = report_to_json(report);
        *n_out = int32_t(text.size());
        if (int(text.size()) + 1 > cap)
            return fail(TCSE_ECAPACITY, "report buffer too small");
        std::memcpy(out, text.c_str(), text.size() + 1);
        return TCSE_OK;
    });
}

// optimize_with_flips (parallel_search.hpp:354-518) -> report_to_json
int ref_optimize_with_flips_json(const char* scheme_json, const tcse_search_config* c, int32_t m_schemes,
                                 int32_t flips_min, int32_t flips_max, uint32_t threads, char* out, int32_t cap,
                                 int32_t* n_out) {
    return guarded([&]() -> int {
        SearchConfig cfg = to_cfg(c, threads);
        cfg.flip_mode.enabled = true;
        cfg.flip_mode.m_schemes = m_schemes;
        cfg.flip_mode.flips_min = flips_min;
        cfg.flip_mode.flips_max = flips_max;
        const auto text = report_to_json(optimize_with_flips(parse_scheme(scheme_json), cfg));
        *n_out = int32_t(text.size());
        if (int(text.size()) + 1 > cap)
            return fail(TCSE_ECAPACITY, "report buffer too small");
        std::memcpy(out, text.c_str(), text.size() + 1);
        return TCSE_OK;
    });
}

// emit_slp (io.hpp:352-393) of a report (parse_report, io.hpp:268-291) for a scheme
int ref_emit_slp(const char* scheme_json, const char* report_json, char* out, int32_t cap, int32_t* n_out) {
    return guarded([&]() -> int {
        const auto text = emit_slp(parse_report(report_json), parse_scheme(scheme_json));
        *n_out = int32_t(text.size());
        if (int(text.size()) + 1 > cap)
            return fail(TCSE_ECAPACITY, "buffer too small");
        std::memcpy(out, text.c_str(), text.size() + 1);
        return TCSE_OK;
    });
}

// combine_componentwise (parallel_search.hpp:522-547) of several report JSONs
// separated by '\x1e', back to report JSON
int ref_combine_json(const char* reports, char* out, int32_t cap, int32_t* n_out) {
    return guarded([&]() -> int {
        std::vector<SearchReport> rs;
        std::string all(reports), cur;
        for (char ch : all) {
            if (ch == '\x1e') {
                rs.push_back(parse_report(cur));
                cur.clear();
            } else {
                cur += ch;
            }
        }
        if (!cur.empty())
            rs.push_back(parse_report(cur));
        const auto text = report_to_json(combine_componentwise(rs));
        *n_out = int32_t(text.size());
        if (int(text.size()) + 1 > cap)
            return fail(TCSE_ECAPACITY, "buffer too small");
        std::memcpy(out, text.c_str(), text.size() + 1);
        return TCSE_OK;
    });
}

// naive_scheme / random_flip (scheme.hpp:161-276) for fixture generation
int ref_flipped_naive_json(int32_t m, int32_t n, int32_t p, int32_t flips, uint64_t seed,
                           char* out, int32_t cap, int32_t* n_out) {
    return guarded([&]() -> int {
        std::mt19937_64 rng(seed);
        Scheme s = naive_scheme(m, n, p);
        for (int t = 0; t < flips; ++t)
            s = random_flip(s, rng);
        const auto text = scheme_to_json(s);
        *n_out = int32_t(text.size());
        if (int(text.size()) + 1 > cap)
            return fail(TCSE_ECAPACITY, "buffer too small");
        std::memcpy(out, text.c_str(), text.size() + 1);
        return TCSE_OK;
    });
}

// verify_brent / verify_by_product / check_scheme_auto (scheme.hpp:68-137,
// parallel_search.hpp:296-302) of a flat scheme; structural errors come back
// as TCSE_EINVAL with the reference's message.
int ref_check_scheme(const tcse_scheme* c, int32_t method, int32_t trials, uint64_t seed, tcse_check_report* out) {
    return guarded([&]() -> int {
        Scheme s;
        s.m = c->m;
        s.n = c->n;
        s.p = c->p;
        s.r = c->r;
        const std::size_t mn = std::size_t(c->m) * c->n, np = std::size_t(c->n) * c->p, mp = std::size_t(c->m) * c->p;
        if (c->r > 0 && c->m > 0 && c->n > 0 && c->p > 0) {
            for (int q = 0; q < c->r; ++q) {
                s.u.emplace_back(c->u + q * mn, c->u + (q + 1) * mn);
                s.v.emplace_back(c->v + q * np, c->v + (q + 1) * np);
            }
            for (std::size_t row = 0; row < mp; ++row)
                s.w.emplace_back(c->w + row * c->r, c->w + (row + 1) * c->r);
        }
        SchemeCheckReport rep;
        if (method == TCSE_CHECK_BRENT)
            rep = verify_brent(s);
        else if (method == TCSE_CHECK_PRODUCT)
            rep = verify_by_product(s, trials, seed);
        else
            rep = detail::check_scheme_auto(s, seed);
        std::memset(out, 0, sizeof *out);
        out->valid = rep.valid ? 1 : 0;
        out->method = rep.method == CheckMethod::exact_brent ? TCSE_CHECK_BRENT : TCSE_CHECK_PRODUCT;
        if (rep.first_violation)
            std::snprintf(out->first_violation, sizeof out->first_violation, "%s", rep.first_violation->c_str());
        return TCSE_OK;
    });
}

}  // extern "C"
