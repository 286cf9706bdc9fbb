// adapter_check.cpp — the reference's own API with the GPU drop-in
// (include/tcse/terncse_gpu.hpp) side by side with the CPU implementation.
//
// TEST INFRASTRUCTURE: built by oracle/Makefile against the unmodified
// reference headers into oracle/_ref/adapter_check (links libtcse.so); run on
// a GPU by tests/test_gpu_adapter.py.  Every check compares the reference's
// serialized or returned results byte for byte.
#include <terncse/io.hpp>
#include <terncse/parallel_search.hpp>
#include <tcse/terncse_gpu.hpp>

#include <cstdio>
#include <fstream>
#include <random>
#include <sstream>

using namespace terncse;

static int failures = 0;

static void report(bool ok, const std::string& what) {
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok)
        ++failures;
}

static std::string slurp(const std::string& path) {
    std::ifstream in(path);
    std::ostringstream b;
    b << in.rdbuf();
    return b.str();
}

static LinearSystem random_system(std::mt19937_64& rng, int max_exprs, int max_vars) {
    const int n_x = std::uniform_int_distribution<int>(2, max_vars)(rng);
    const int n_e = std::uniform_int_distribution<int>(1, max_exprs)(rng);
    std::vector<std::vector<int>> exprs;
    std::vector<int> ids;
    for (int i = 0; i < n_x; ++i)
        ids.push_back(i + 1);
    for (int e = 0; e < n_e; ++e) {
        std::shuffle(ids.begin(), ids.end(), rng);
        const int terms = std::uniform_int_distribution<int>(0, n_x)(rng);
        std::vector<int> expr;
        for (int t = 0; t < terms; ++t)
            expr.push_back(std::uniform_int_distribution<int>(0, 1)(rng) ? ids[std::size_t(t)] : -ids[std::size_t(t)]);
        exprs.push_back(std::move(expr));
    }
    return LinearSystem(n_x, exprs);
}

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : "tests/golden/schemes";
    // 1. optimize_scheme: byte-identical report JSON (io.hpp:250-266)
    struct Case {
        const char* name;
        int n;
        int patience;
        std::uint64_t seed;
    };
    for (const Case& c : {Case{"strassen", 16, 2, 0}, Case{"laderman", 64, 3, 7}, Case{"sxs", 48, 2, 11},
                          Case{"laderman", 0, 2, 5}}) {
        const Scheme s = parse_scheme(slurp(dir + "/" + c.name + ".json"));
        SearchConfig cfg;
        cfg.n_processes = c.n;
        cfg.patience = c.patience;
        cfg.master_seed = c.seed;
        const auto cpu = report_to_json(optimize_scheme(s, cfg));
        const auto gpu = report_to_json(gpu::optimize_scheme(s, cfg));
        report(cpu == gpu, std::string("optimize_scheme report bytes: ") + c.name + " n=" + std::to_string(c.n));
    }
    // 1b. optimize_with_flips (parallel_search.hpp:354-518): byte-identical report
    for (const Case& c : {Case{"strassen", 9, 2, 3}, Case{"laderman", 32, 2, 5}}) {
        const Scheme s = parse_scheme(slurp(dir + "/" + c.name + ".json"));
        SearchConfig cfg;
        cfg.n_processes = c.n;
        cfg.patience = c.patience;
        cfg.master_seed = c.seed;
        cfg.flip_mode.enabled = true;
        cfg.flip_mode.m_schemes = 4;
        const auto cpu = report_to_json(optimize_with_flips(s, cfg));
        const auto gpu = report_to_json(gpu::optimize_with_flips(s, cfg));
        report(cpu == gpu, std::string("optimize_with_flips report bytes: ") + c.name);
    }
    // 2. optimize_system with on_iteration (parallel_search.hpp:220-273)
    std::mt19937_64 gen(1234);
    for (int round = 0; round < 6; ++round) {
        const auto sys = random_system(gen, 20, 10);
        SearchConfig cfg;
        cfg.n_processes = 12;
        cfg.patience = 3;
        cfg.master_seed = gen();
        std::vector<int> a, b;
        const auto cpu = optimize_system(sys, cfg, 1, [&](int, const SolutionRecord& r) { a.push_back(r.cost); });
        const auto g = gpu::optimize_system(sys, cfg, 1, [&](int, const SolutionRecord& r) { b.push_back(r.cost); });
        report(cpu.best.substitutions == g.best.substitutions && cpu.best.cost == g.best.cost &&
                   cpu.iterations == g.iterations && cpu.best.seed == g.best.seed && a == b,
               "optimize_system record + on_iteration trace, round " + std::to_string(round));
    }
    // 3. run_cse for every strategy, and count_pairs on a state with fresh variables
    for (int round = 0; round < 20; ++round) {
        const auto sys = random_system(gen, 14, 10);
        for (std::size_t k = 0; k < strategy_count; ++k) {
            ProcessConfig pc;
            pc.strategy = StrategyKind(k);
            pc.alpha = std::uniform_real_distribution<double>(0.0, 0.5)(gen);
            pc.seed = gen();
            std::mt19937_64 rng(pc.seed);
            const auto cpu = run_cse(sys, pc, rng);
            const auto g = gpu::run_cse(sys, pc);
            if (cpu.substitutions != g.substitutions || cpu.cost != g.cost)
                report(false, "run_cse " + std::string(to_string(StrategyKind(k))));
        }
        auto state = sys;
        const auto cands = count_pairs(state).candidates();
        if (!cands.empty())
            apply_substitution(state, cands[0].pair);
        const auto a = count_pairs(state), b = gpu::count_pairs(state);
        bool same = a.freq.size() == b.freq.size();
        for (const auto& [pair, cnt] : a.freq)
            same = same && b.count(pair) == cnt;
        if (!same)
            report(false, "count_pairs on a replayed state");
        // continuing from a state with fresh variables
        ProcessConfig g0;
        std::mt19937_64 r0(0);
        const auto cont_cpu = run_cse(state, g0, r0);
        const auto cont_gpu = gpu::run_cse(state, g0);
        if (cont_cpu.substitutions != cont_gpu.substitutions || cont_cpu.cost != cont_gpu.cost)
            report(false, "run_cse continuing from fresh variables");
    }
    report(failures == 0, "run_cse x 7 strategies x 20 systems, count_pairs, continuation");
    // 4. errors surface as terncse::error with the reference's messages
    try {
        SearchConfig bad;
        bad.patience = 0;
        gpu::optimize_system(LinearSystem(2, {{1, 2}, {1, 2}}), bad);
        report(false, "bad config throws");
    } catch (const error& e) {
        report(std::string(e.what()).find("patience") != std::string::npos, "bad config throws terncse::error");
    }
    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
