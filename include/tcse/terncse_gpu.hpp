// terncse_gpu.hpp — drop-in B200 search for the reference library (terncse).
//
// A maintainer of the reference includes this header after the reference's
// own headers and links libtcse.so (paper_2512_13365_b200/libtcse.so); the
// functions below are signature-compatible with
//
//   terncse::optimize_system   (parallel_search.hpp:220-222)
//   terncse::optimize_scheme   (parallel_search.hpp:314)
//   terncse::run_cse           (cse_engine.hpp:29), rng = mt19937_64(cfg.seed)
//   terncse::count_pairs       (linear_system.hpp:151)
//   terncse::optimize_with_flips (parallel_search.hpp:354)
//
// and return the reference's own result types.  Everything around the search
// stays the reference's code: scheme validation (check_scheme_auto),
// extract_systems, expand_and_verify, scheme_digest, the report and its JSON.
// Only the search itself crosses the C ABI (include/tcse.h) into the sm_100a
// kernels.  Results are bit-identical to the CPU implementation for every
// strategy and seed (the device replays the reference's mt19937_64 streams),
// so reports serialize to the same bytes.  Errors are thrown as
// terncse::error with the reference's messages.
#pragma once

#include <terncse/parallel_search.hpp>

#include <chrono>
#include <cstdlib>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "../tcse.h"

namespace terncse::gpu {

// One GPU, or several GPUs of this process as one context: the search then
// partitions its processes across them with one NCCL all-gather per
// iteration (tcse_create_devices), results identical to one GPU.
class Context {
public:
    explicit Context(int device = 0) : h_(tcse_create(device)) {
        if (!h_)
            throw error(tcse_last_error());
    }
    explicit Context(const std::vector<int>& devices)
        : h_(tcse_create_devices(reinterpret_cast<const int32_t*>(devices.data()), int32_t(devices.size()))) {
        if (!h_)
            throw error(tcse_last_error());
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    ~Context() { tcse_destroy(h_); }
    tcse_ctx* get() const { return h_; }
    int devices() const { return tcse_context_devices(h_); }

private:
    tcse_ctx* h_;
};

// The default context spans every visible GPU (as the reference's default
// thread count spans every core, parallel_search.hpp:41-43), or the list in
// TCSE_DEVICES ("0,1,2,3"); one GPU if NCCL is unavailable.
inline std::vector<int> default_devices() {
    std::vector<int> devs;
    if (const char* env = std::getenv("TCSE_DEVICES")) {
        std::string s(env), cur;
        for (char c : s + ",") {
            if (c == ',') {
                if (!cur.empty())
                    devs.push_back(std::stoi(cur));
                cur.clear();
            } else {
                cur += c;
            }
        }
    } else {
        for (int d = 0; d < tcse_device_count(); ++d)
            devs.push_back(d);
    }
    if (devs.empty())
        devs.push_back(0);
    if (devs.size() > 1 && !tcse_nccl_available())
        devs.resize(1);
    return devs;
}

inline Context& default_context() {
    static Context ctx(default_devices());
    return ctx;
}

namespace detail_gpu {

inline void check(int rc) {
    if (rc != TCSE_OK)
        throw error(tcse_last_error());
}

// CSR view of a LinearSystem; fresh variables already defined become base
// variables of the view (ids are unchanged: new fresh ids continue at
// var_count() + 1, as LinearSystem::next_id() does)
struct Csr {
    std::vector<int32_t> row_ptr{0}, terms;
    tcse_system sys{};
    int existing_fresh = 0;
    explicit Csr(const LinearSystem& s) {
        for (const auto& e : s.expressions) {
            std::vector<int> t(e.begin(), e.end());
            std::sort(t.begin(), t.end(), [](int a, int b) {
                return std::abs(a) != std::abs(b) ? std::abs(a) < std::abs(b) : a < b;
            });
            terms.insert(terms.end(), t.begin(), t.end());
            row_ptr.push_back(int32_t(terms.size()));
        }
        if (terms.empty())
            terms.push_back(0);
        sys.n_x = s.var_count();
        sys.n_e = int32_t(s.expressions.size());
        sys.row_ptr = row_ptr.data();
        sys.terms = terms.data();
        existing_fresh = s.fresh_count();
    }
};

inline tcse_search_config to_c(const SearchConfig& cfg) {
    tcse_search_config c;
    tcse_default_search_config(&c);
    c.n_processes = cfg.n_processes;
    for (std::size_t k = 0; k < strategy_count; ++k)
        c.strategy_weights[k] = cfg.strategy_weights[k];
    c.reinit_fraction = cfg.reinit_fraction;
    c.patience = cfg.patience;
    c.master_seed = cfg.master_seed;
    c.forced_strategy = cfg.forced_strategy ? int32_t(*cfg.forced_strategy) : -1;
    return c;
}

inline SolutionRecord from_c(const tcse_record& r, int extra_cost = 0) {
    SolutionRecord rec;
    for (int t = 0; t < r.n_subs; ++t)
        rec.substitutions.push_back({r.subs[t].i, r.subs[t].j, r.subs[t].rel_sign});
    rec.cost = r.cost + extra_cost;
    rec.strategy = StrategyKind(r.strategy);
    rec.seed = r.seed;
    return rec;
}

struct CbState {
    const std::function<void(int, const SolutionRecord&)>* fn;
    int extra;
};

inline int trampoline(int32_t, int32_t iteration, const tcse_record* inc, void* user) {
    auto* st = static_cast<CbState*>(user);
    (*st->fn)(iteration, from_c(*inc, st->extra));
    return 0;
}

}  // namespace detail_gpu

// optimize_system (parallel_search.hpp:220-273) on the device
inline SystemSearchResult optimize_system(const LinearSystem& sys, const SearchConfig& cfg,
                                          std::uint64_t stream_salt = 0,
                                          const std::function<void(int, const SolutionRecord&)>& on_iteration = {},
                                          Context& ctx = default_context()) {
    detail::validate_config(cfg);
    detail_gpu::Csr csr(sys);
    const auto c = detail_gpu::to_c(cfg);
    std::vector<tcse_pair> buf(std::size_t(naive_cost(sys) + 1));
    tcse_record rec{buf.data(), int32_t(buf.size()), 0, 0, 0, 0};
    int32_t iterations = 0;
    detail_gpu::CbState st{&on_iteration, csr.existing_fresh};
    detail_gpu::check(tcse_optimize_system(ctx.get(), &csr.sys, &c, stream_salt,
                                           on_iteration ? detail_gpu::trampoline : nullptr, &st, &rec,
                                           &iterations, nullptr));
    return {detail_gpu::from_c(rec, csr.existing_fresh), iterations};
}

// run_cse (cse_engine.hpp:29-43) with rng = std::mt19937_64(cfg.seed), the
// stream optimize_system hands every process (parallel_search.hpp:241)
inline SolutionRecord run_cse(const LinearSystem& sys, const ProcessConfig& cfg,
                              Context& ctx = default_context()) {
    detail_gpu::Csr csr(sys);
    tcse_process_config pc{};
    pc.strategy = int32_t(cfg.strategy);
    pc.alpha = cfg.alpha;
    pc.beta = cfg.beta;
    pc.p_greedy = cfg.p_greedy;
    pc.seed = cfg.seed;
    for (int k = 0; k < 4; ++k)
        pc.mix_weights[k] = cfg.mix_weights[std::size_t(k)];
    std::vector<tcse_pair> buf(std::size_t(naive_cost(sys) + 1));
    tcse_record rec{buf.data(), int32_t(buf.size()), 0, 0, 0, 0};
    detail_gpu::check(tcse_run_cse(ctx.get(), &csr.sys, nullptr, 0, &pc, 1, &rec, nullptr, 0, nullptr));
    return detail_gpu::from_c(rec, csr.existing_fresh);
}

// count_pairs (linear_system.hpp:151-161) computed on the device
inline PairStats count_pairs(const LinearSystem& sys, Context& ctx = default_context()) {
    detail_gpu::Csr csr(sys);
    const int v = sys.var_count();
    std::vector<tcse_pair_count> out(std::size_t(std::max(16, 2 * v * v)));
    int32_t n = 0;
    detail_gpu::check(tcse_count_pairs(ctx.get(), &csr.sys, nullptr, 0, 1, out.data(), int32_t(out.size()), &n));
    PairStats stats;
    for (int t = 0; t < n; ++t)
        stats.freq[{out[std::size_t(t)].pair.i, out[std::size_t(t)].pair.j, out[std::size_t(t)].pair.rel_sign}] =
            out[std::size_t(t)].count;
    return stats;
}

// optimize_scheme (parallel_search.hpp:314-345): the reference's validation,
// extraction, verification and report; U, V and W searched concurrently on
// the device instead of one after another
inline SearchReport optimize_scheme(const Scheme& s, const SearchConfig& cfg, Context& ctx = default_context()) {
    detail::validate_config(cfg);
    const auto started = std::chrono::steady_clock::now();
    const auto check = detail::check_scheme_auto(s, cfg.master_seed);
    if (!check.valid)
        throw error("optimize_scheme: scheme failed validation (" + check.first_violation.value_or("unknown") + ")");
    SearchConfig resolved = cfg;
    resolved.n_processes = detail::resolve_processes(cfg, s.r);
    const auto systems = extract_systems(s);
    std::vector<std::unique_ptr<detail_gpu::Csr>> csr;
    std::vector<tcse_system> views;
    std::vector<std::vector<tcse_pair>> bufs;
    std::vector<tcse_record> recs;
    for (const auto& sys : systems) {
        csr.push_back(std::make_unique<detail_gpu::Csr>(sys));
        views.push_back(csr.back()->sys);
        bufs.emplace_back(std::size_t(naive_cost(sys) + 1));
    }
    for (auto& b : bufs)
        recs.push_back({b.data(), int32_t(b.size()), 0, 0, 0, 0});
    const auto c = detail_gpu::to_c(resolved);
    const std::uint64_t salts[3] = {0, 1, 2};
    int32_t iters[3] = {0, 0, 0};
    detail_gpu::check(tcse_optimize_systems(ctx.get(), 3, views.data(), &c, salts, nullptr, nullptr, recs.data(),
                                            iters, nullptr));
    SearchReport report;
    report.scheme_digest = scheme_digest(s);
    report.config = resolved;
    for (std::size_t comp = 0; comp < 3; ++comp) {
        auto best = detail_gpu::from_c(recs[comp]);
        const auto final_state = replay_prefix(systems[comp], best.substitutions);
        if (total_cost(final_state) != best.cost || !expand_and_verify(systems[comp], final_state))
            throw error("optimize_scheme: internal verification failed");
        ComponentResult& result = report.components[comp];
        result.record = std::move(best);
        result.cost = result.record.cost;
        result.naive = naive_cost(systems[comp]);
        result.iterations = iters[comp];
        report.total += result.cost;
        report.iterations += result.iterations;
    }
    report.wall_ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - started)
                         .count();
    return report;
}

// optimize_with_flips (parallel_search.hpp:354-518) with the search on the
// device; the report carries the winning variant, as the reference's does
inline SearchReport optimize_with_flips(const Scheme& s, const SearchConfig& cfg, Context& ctx = default_context()) {
    detail::validate_config(cfg);
    if (!cfg.flip_mode.enabled)
        throw error("optimize_with_flips: flip mode is disabled");
    if (cfg.flip_mode.m_schemes == 1)
        return gpu::optimize_scheme(s, cfg, ctx);
    check_structure(s);
    const auto started = std::chrono::steady_clock::now();
    SearchConfig resolved = cfg;
    resolved.n_processes = detail::resolve_processes(cfg, s.r);
    std::vector<int8_t> u, v, w;
    for (const auto& row : s.u)
        u.insert(u.end(), row.begin(), row.end());
    for (const auto& row : s.v)
        v.insert(v.end(), row.begin(), row.end());
    for (const auto& row : s.w)
        w.insert(w.end(), row.begin(), row.end());
    const tcse_scheme cs{s.m, s.n, s.p, s.r, u.data(), v.data(), w.data()};
    std::vector<int8_t> ou(u.size()), ov(v.size()), ow(w.size());
    const std::size_t cap = std::size_t(s.r) * std::size_t(std::max({s.m * s.n, s.n * s.p, s.m * s.p})) + 1;
    std::vector<tcse_pair> b0(cap), b1(cap), b2(cap);
    tcse_flip_result res{};
    res.u = ou.data();
    res.v = ov.data();
    res.w = ow.data();
    res.comp[0] = {b0.data(), int32_t(cap), 0, 0, 0, 0};
    res.comp[1] = {b1.data(), int32_t(cap), 0, 0, 0, 0};
    res.comp[2] = {b2.data(), int32_t(cap), 0, 0, 0, 0};
    const auto c = detail_gpu::to_c(resolved);
    const tcse_flip_config fc{cfg.flip_mode.m_schemes, cfg.flip_mode.flips_min, cfg.flip_mode.flips_max, 0};
    detail_gpu::check(tcse_optimize_with_flips(ctx.get(), &cs, &c, &fc, &res, nullptr));
    Scheme carried = s;
    for (int q = 0; q < s.r; ++q) {
        std::copy_n(ou.data() + std::size_t(q) * std::size_t(s.m * s.n), s.m * s.n, carried.u[std::size_t(q)].begin());
        std::copy_n(ov.data() + std::size_t(q) * std::size_t(s.n * s.p), s.n * s.p, carried.v[std::size_t(q)].begin());
    }
    for (std::size_t row = 0; row < carried.w.size(); ++row)
        std::copy_n(ow.data() + row * std::size_t(s.r), s.r, carried.w[row].begin());
    SearchReport report;
    report.scheme_digest = scheme_digest(carried);
    report.config = resolved;
    report.carried_scheme = carried;
    const std::string id = res.scheme_slot == 0 ? std::string("original")
                                                : "flip-" + std::to_string(res.scheme_iteration) + "-" +
                                                      std::to_string(res.scheme_slot);
    const auto systems = extract_systems(carried);
    for (std::size_t comp = 0; comp < 3; ++comp) {
        auto best = detail_gpu::from_c(res.comp[comp]);
        const auto final_state = replay_prefix(systems[comp], best.substitutions);
        if (total_cost(final_state) != best.cost || !expand_and_verify(systems[comp], final_state))
            throw error("optimize_with_flips: internal verification failed");
        ComponentResult& result = report.components[comp];
        result.record = std::move(best);
        result.cost = result.record.cost;
        result.naive = naive_cost(systems[comp]);
        result.iterations = res.iterations;
        result.scheme_id = id;
        report.total += result.cost;
    }
    report.iterations = res.iterations;
    report.wall_ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - started)
                         .count();
    return report;
}

}  // namespace terncse::gpu
