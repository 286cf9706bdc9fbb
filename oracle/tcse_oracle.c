/*
 * tcse_oracle.c — CPU restatement of the reference search path (TEST
 * INFRASTRUCTURE ONLY; see tcse_oracle.h).  Every function cites the
 * reference file:line it restates; paths are relative to
 * /root/reference/proj/include/terncse/.
 *
 * Build: oracle/Makefile (gcc -O2 -std=c11 -ffp-contract=off).  The
 * -ffp-contract=off matches the reference's Release build, which targets
 * baseline x86-64 (no FMA), so double arithmetic rounds after every operation.
 */
#include "tcse_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* or_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ rng */

/* splitmix64 (rng.hpp:8-13) */
static uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* mix_seed (rng.hpp:18-23) */
uint64_t or_mix_seed(const uint64_t* parts, int32_t n_parts) {
    uint64_t h = 0x5851f42d4c957f2dULL;
    for (int32_t t = 0; t < n_parts; ++t)
        h = splitmix64(h ^ parts[t]);
    return h;
}

/* std::mt19937_64 (libstdc++ mersenne_twister_engine<uint64, 64, 312, 156,
 * 31, 0xb5026f5aa96619e9, 29, 0x5555555555555555, 17, 0x71d67fffeda60000, 37,
 * 0xfff7eee000000000, 43, 6364136223846793005>) */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt_seed(mt64* g, uint64_t s) {
    g->mt[0] = s;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static void mt_twist(mt64* g) {
    const uint64_t UM = 0xffffffff80000000ULL, LM = 0x7fffffffULL, A = 0xb5026f5aa96619e9ULL;
    uint64_t* mt = g->mt;
    int i = 0;
    for (; i < 312 - 156; ++i) {
        uint64_t y = (mt[i] & UM) | (mt[i + 1] & LM);
        mt[i] = mt[i + 156] ^ (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
    }
    for (; i < 311; ++i) {
        uint64_t y = (mt[i] & UM) | (mt[i + 1] & LM);
        mt[i] = mt[i + 156 - 312] ^ (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
    }
    uint64_t y = (mt[311] & UM) | (mt[0] & LM);
    mt[311] = mt[155] ^ (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
    g->idx = 0;
}

static uint64_t mt_next(mt64* g) {
    if (g->idx >= 312)
        mt_twist(g);
    uint64_t z = g->mt[g->idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71d67fffeda60000ULL;
    z ^= (z << 37) & 0xfff7eee000000000ULL;
    z ^= (z >> 43);
    return z;
}

/* uniform_int_distribution downscaling path with a 64-bit engine:
 * __S::_S_nd<unsigned __int128>(urng, range) (bits/uniform_int_dist.h:257-281,
 * 312-319).  Returns a value in [0, range). */
static uint64_t mt_nd(mt64* g, uint64_t range) {
    unsigned __int128 product = (unsigned __int128)mt_next(g) * range;
    uint64_t low = (uint64_t)product;
    if (low < range) {
        uint64_t threshold = (0 - range) % range;
        while (low < threshold) {
            product = (unsigned __int128)mt_next(g) * range;
            low = (uint64_t)product;
        }
    }
    return (uint64_t)(product >> 64);
}

/* uniform_int_distribution<T>(a, b) for b - a < 2^64 - 1 */
static uint64_t mt_uniform_int(mt64* g, uint64_t a, uint64_t b) { return a + mt_nd(g, b - a + 1); }

/* generate_canonical<double, 53>(mt19937_64) (bits/random.tcc:3349-3381):
 * one engine call, double(x) / 2^64, clamped below 1 */
static double mt_canonical(mt64* g) {
    double r = (double)mt_next(g) / 18446744073709551616.0;
    if (r >= 1.0)
        r = nextafter(1.0, 0.0);
    return r;
}

/* uniform_real_distribution<double>(a, b): canonical * (b - a) + a */
static double mt_uniform_real(mt64* g, double a, double b) {
    double span = b - a;
    double t = mt_canonical(g) * span;
    return t + a;
}

void or_mt19937_64(uint64_t seed, int32_t n, uint64_t* out) {
    mt64 g;
    mt_seed(&g, seed);
    for (int32_t t = 0; t < n; ++t)
        out[t] = mt_next(&g);
}

void or_uniform_int(uint64_t seed, uint64_t a, uint64_t b, int32_t n, uint64_t* out) {
    mt64 g;
    mt_seed(&g, seed);
    for (int32_t t = 0; t < n; ++t)
        out[t] = mt_uniform_int(&g, a, b);
}

void or_uniform_real(uint64_t seed, double a, double b, int32_t n, double* out) {
    mt64 g;
    mt_seed(&g, seed);
    for (int32_t t = 0; t < n; ++t)
        out[t] = mt_uniform_real(&g, a, b);
}

/* ------------------------------------------------------- linear system */

/* LinearSystem (linear_system.hpp:76-122): expressions as unsorted arrays of
 * signed ids (set semantics), plus fresh definitions. */
typedef struct {
    int n_x, n_e, n_f;
    int* len;      /* n_e */
    int* cap;      /* n_e */
    int** rows;    /* n_e arrays */
    tcse_pair* defs;
    int defs_cap;
} osys;

static void osys_free(osys* s) {
    if (!s->rows)
        return;
    for (int r = 0; r < s->n_e; ++r)
        free(s->rows[r]);
    free(s->rows);
    free(s->len);
    free(s->cap);
    free(s->defs);
    memset(s, 0, sizeof *s);
}

static int row_has(const osys* s, int r, int term) {
    for (int t = 0; t < s->len[r]; ++t)
        if (s->rows[r][t] == term)
            return 1;
    return 0;
}

/* LinearSystem constructor validation (linear_system.hpp:84-101) */
static int osys_init(osys* s, const tcse_system* in) {
    memset(s, 0, sizeof *s);
    if (in->n_x < 0)
        return fail(TCSE_EINVAL, "linear system: negative variable count");
    if (in->n_e < 0)
        return fail(TCSE_EINVAL, "linear system: negative expression count");
    s->n_x = in->n_x;
    s->n_e = in->n_e;
    s->len = calloc((size_t)in->n_e + 1, sizeof(int));
    s->cap = calloc((size_t)in->n_e + 1, sizeof(int));
    s->rows = calloc((size_t)in->n_e + 1, sizeof(int*));
    s->defs_cap = 16;
    s->defs = malloc(sizeof(tcse_pair) * (size_t)s->defs_cap);
    for (int r = 0; r < in->n_e; ++r) {
        int n = in->row_ptr[r + 1] - in->row_ptr[r];
        s->cap[r] = n > 0 ? n : 1;
        s->rows[r] = malloc(sizeof(int) * (size_t)s->cap[r]);
        for (int t = 0; t < n; ++t) {
            int term = in->terms[in->row_ptr[r] + t];
            if (term == 0 || abs(term) > in->n_x) {
                int code = fail(TCSE_EINVAL, "linear system: index %d out of range in expression %d", term, r);
                osys_free(s);
                return code;
            }
            if (row_has(s, r, -term)) {
                int code = fail(TCSE_EINVAL, "linear system: expression %d contains both signs of x%d", r, abs(term));
                osys_free(s);
                return code;
            }
            if (row_has(s, r, term)) {
                int code = fail(TCSE_EINVAL, "linear system: duplicate term in expression %d", r);
                osys_free(s);
                return code;
            }
            s->rows[r][s->len[r]++] = term;
        }
    }
    return TCSE_OK;
}

static void osys_copy(osys* dst, const osys* src) {
    memset(dst, 0, sizeof *dst);
    dst->n_x = src->n_x;
    dst->n_e = src->n_e;
    dst->n_f = src->n_f;
    dst->len = malloc(sizeof(int) * ((size_t)src->n_e + 1));
    dst->cap = malloc(sizeof(int) * ((size_t)src->n_e + 1));
    dst->rows = malloc(sizeof(int*) * ((size_t)src->n_e + 1));
    for (int r = 0; r < src->n_e; ++r) {
        dst->len[r] = src->len[r];
        dst->cap[r] = src->cap[r];
        dst->rows[r] = malloc(sizeof(int) * (size_t)src->cap[r]);
        memcpy(dst->rows[r], src->rows[r], sizeof(int) * (size_t)src->len[r]);
    }
    dst->defs_cap = src->defs_cap;
    dst->defs = malloc(sizeof(tcse_pair) * (size_t)src->defs_cap);
    memcpy(dst->defs, src->defs, sizeof(tcse_pair) * (size_t)src->n_f);
}

static void row_erase(osys* s, int r, int term) {
    for (int t = 0; t < s->len[r]; ++t)
        if (s->rows[r][t] == term) {
            s->rows[r][t] = s->rows[r][--s->len[r]];
            return;
        }
}

static void row_insert(osys* s, int r, int term) {
    if (s->len[r] == s->cap[r]) {
        s->cap[r] *= 2;
        s->rows[r] = realloc(s->rows[r], sizeof(int) * (size_t)s->cap[r]);
    }
    s->rows[r][s->len[r]++] = term;
}

/* apply_substitution (linear_system.hpp:167-189); returns the number of
 * replaced occurrences (0 = the reference throws, state untouched) */
static int osys_apply(osys* s, tcse_pair q) {
    const int k = s->n_x + s->n_f + 1;
    const int first = q.i;
    const int second = q.rel_sign * q.j;
    int replaced = 0;
    for (int r = 0; r < s->n_e; ++r) {
        if (row_has(s, r, first) && row_has(s, r, second)) {
            row_erase(s, r, first);
            row_erase(s, r, second);
            row_insert(s, r, k);
            ++replaced;
        } else if (row_has(s, r, -first) && row_has(s, r, -second)) {
            row_erase(s, r, -first);
            row_erase(s, r, -second);
            row_insert(s, r, -k);
            ++replaced;
        }
    }
    if (replaced == 0)
        return 0;
    if (s->n_f == s->defs_cap) {
        s->defs_cap *= 2;
        s->defs = realloc(s->defs, sizeof(tcse_pair) * (size_t)s->defs_cap);
    }
    s->defs[s->n_f++] = q;
    return replaced;
}

/* naive_cost / total_cost (linear_system.hpp:193-204) */
static int osys_naive(const osys* s) {
    int cost = 0;
    for (int r = 0; r < s->n_e; ++r)
        if (s->len[r] > 0)
            cost += s->len[r] - 1;
    return cost;
}

static int osys_total(const osys* s) { return s->n_f + osys_naive(s); }

/* replay_prefix (cse_engine.hpp:47-57) */
static int osys_replay(osys* s, const tcse_pair* prefix, int n_prefix) {
    for (int t = 0; t < n_prefix; ++t) {
        tcse_pair q = prefix[t];
        if (q.i <= 0 || q.j <= q.i || (q.rel_sign != 1 && q.rel_sign != -1) || osys_apply(s, q) == 0)
            return fail(TCSE_EREPLAY, "replay_prefix: unreplayable pair at position %d", t);
    }
    return TCSE_OK;
}

/* pair key in canonical order (linear_system.hpp:32-36): (i, j, '+' < '-') */
static uint64_t pair_key(int i, int j, int rel) {
    return ((uint64_t)(uint32_t)i << 33) | ((uint64_t)(uint32_t)j << 1) | (uint64_t)(rel < 0);
}

static tcse_pair key_pair(uint64_t key) {
    tcse_pair q;
    q.i = (int)(key >> 33);
    q.j = (int)((key >> 1) & 0xffffffffULL);
    q.rel_sign = (key & 1ULL) ? -1 : 1;
    return q;
}

static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

typedef struct {
    uint64_t key;
    int count;
} okc;

typedef struct {
    okc* v;
    int n;
} opairs;

/* count_pairs (linear_system.hpp:151-161) with canonicalize (53-61); result
 * sorted canonically, every pair with count >= 1 */
static opairs osys_count(const osys* s) {
    size_t total = 0;
    for (int r = 0; r < s->n_e; ++r)
        total += (size_t)s->len[r] * (size_t)(s->len[r] > 0 ? s->len[r] - 1 : 0) / 2;
    uint64_t* keys = malloc(sizeof(uint64_t) * (total + 1));
    size_t n = 0;
    for (int r = 0; r < s->n_e; ++r) {
        const int* t = s->rows[r];
        for (int a = 0; a + 1 < s->len[r]; ++a)
            for (int b = a + 1; b < s->len[r]; ++b) {
                int x = t[a], y = t[b];
                if (abs(x) > abs(y)) {
                    int tmp = x;
                    x = y;
                    y = tmp;
                }
                int rel = ((x > 0) == (y > 0)) ? 1 : -1;
                keys[n++] = pair_key(abs(x), abs(y), rel);
            }
    }
    qsort(keys, n, sizeof(uint64_t), cmp_u64);
    opairs out;
    out.v = malloc(sizeof(okc) * (n + 1));
    out.n = 0;
    for (size_t t = 0; t < n;) {
        size_t u = t;
        while (u < n && keys[u] == keys[t])
            ++u;
        out.v[out.n].key = keys[t];
        out.v[out.n].count = (int)(u - t);
        ++out.n;
        t = u;
    }
    free(keys);
    return out;
}

/* PairStats::candidates (linear_system.hpp:141-148) */
static opairs candidates_of(const opairs* all) {
    opairs c;
    c.v = malloc(sizeof(okc) * ((size_t)all->n + 1));
    c.n = 0;
    for (int t = 0; t < all->n; ++t)
        if (all->v[t].count >= 2)
            c.v[c.n++] = all->v[t];
    return c;
}

static int stats_count(const opairs* all, uint64_t key) {
    int lo = 0, hi = all->n;
    while (lo < hi) {
        int mid = (lo + hi) / 2;
        if (all->v[mid].key < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return (lo < all->n && all->v[lo].key == key) ? all->v[lo].count : 0;
}

/* ---------------------------------------------------------- strategies */

/* greedy_from (strategies.hpp:61-69) */
static int greedy_from(const opairs* c) {
    if (c->n == 0)
        return -1;
    int best = 0;
    for (int t = 0; t < c->n; ++t)
        if (c->v[t].count > c->v[best].count)
            best = t;
    return best;
}

/* greedy_alternative_from (strategies.hpp:71-83) */
static int greedy_alternative_from(const opairs* c, mt64* g) {
    if (c->n == 0)
        return -1;
    int max_c = 0;
    for (int t = 0; t < c->n; ++t)
        if (c->v[t].count > max_c)
            max_c = c->v[t].count;
    int n_arg = 0;
    for (int t = 0; t < c->n; ++t)
        n_arg += c->v[t].count == max_c;
    uint64_t pick = mt_uniform_int(g, 0, (uint64_t)n_arg - 1);
    for (int t = 0; t < c->n; ++t)
        if (c->v[t].count == max_c && pick-- == 0)
            return t;
    return -1;
}

/* weighted_random_from (strategies.hpp:85-98) */
static int weighted_random_from(const opairs* c, mt64* g) {
    if (c->n == 0)
        return -1;
    double total = 0.0;
    for (int t = 0; t < c->n; ++t)
        total += (double)(c->v[t].count - 1);
    double target = mt_uniform_real(g, 0.0, 1.0) * total;
    for (int t = 0; t < c->n; ++t) {
        target -= (double)(c->v[t].count - 1);
        if (target < 0.0)
            return t;
    }
    return c->n - 1;
}

/* select_greedy_random (strategies.hpp:119-124) */
static int greedy_random_from(const opairs* c, const tcse_process_config* cfg, mt64* g) {
    if (mt_uniform_real(g, 0.0, 1.0) < cfg->p_greedy)
        return greedy_alternative_from(c, g);
    return weighted_random_from(c, g);
}

/* pairs_intersect (strategies.hpp:127-129) */
static int keys_intersect(uint64_t a, uint64_t b) {
    tcse_pair p = key_pair(a), q = key_pair(b);
    return p.i == q.i || p.i == q.j || p.j == q.i || p.j == q.j;
}

/* score_intersections_from (strategies.hpp:136-153) */
static double score_intersections_from(uint64_t q, int c_q, const opairs* c,
                                       const tcse_process_config* cfg, mt64* g) {
    const double gain = (double)(c_q - 1);
    if (cfg->alpha == 0.0)
        return gain;
    double future = 0.0;
    for (int t = 0; t < c->n; ++t) {
        if (c->v[t].key == q)
            continue;
        if (!keys_intersect(q, c->v[t].key))
            future += (double)(c->v[t].count - 1);
        else if (mt_uniform_int(g, 0, 1))
            future += cfg->beta * (double)(c->v[t].count - 1);
    }
    return gain + cfg->alpha * future;
}

/* select_greedy_intersections (strategies.hpp:162-176) */
static int greedy_intersections_from(const opairs* c, const tcse_process_config* cfg, mt64* g) {
    if (c->n == 0)
        return -1;
    int best = -1;
    double best_score = 0.0;
    for (int t = 0; t < c->n; ++t) {
        double h = score_intersections_from(c->v[t].key, c->v[t].count, c, cfg, g);
        if (best < 0 || h > best_score) {
            best = t;
            best_score = h;
        }
    }
    return best;
}

/* select_greedy_potential (strategies.hpp:196-220): trial substitution on a
 * scratch copy, count pairs reaching frequency 2 that were below 2 before */
static int greedy_potential_from(const osys* s, const opairs* all, const opairs* c, double alpha) {
    if (c->n == 0)
        return -1;
    int best = -1;
    double best_score = 0.0;
    for (int t = 0; t < c->n; ++t) {
        double score = (double)(c->v[t].count - 1);
        if (alpha != 0.0) {
            osys trial;
            osys_copy(&trial, s);
            osys_apply(&trial, key_pair(c->v[t].key));
            opairs after = osys_count(&trial);
            int created = 0;
            for (int u = 0; u < after.n; ++u)
                if (after.v[u].count >= 2 && stats_count(all, after.v[u].key) < 2)
                    ++created;
            free(after.v);
            osys_free(&trial);
            score += alpha * (double)created;
        }
        if (best < 0 || score > best_score) {
            best = t;
            best_score = score;
        }
    }
    return best;
}

/* pick_mixed_substrategy (strategies.hpp:236-258) */
static int pick_mixed_substrategy(const tcse_process_config* cfg, mt64* g, int* err) {
    static const int subs[4] = {TCSE_GREEDY_INTERSECTIONS, TCSE_GREEDY_ALTERNATIVE,
                                TCSE_GREEDY_RANDOM, TCSE_WEIGHTED_RANDOM};
    double total = 0.0;
    int positive = 0, only = 0;
    for (int k = 0; k < 4; ++k) {
        if (cfg->mix_weights[k] < 0.0) {
            *err = fail(TCSE_EINVAL, "mixed strategy: negative weight");
            return -1;
        }
        if (cfg->mix_weights[k] > 0.0) {
            ++positive;
            only = k;
        }
        total += cfg->mix_weights[k];
    }
    if (positive == 0) {
        *err = fail(TCSE_EINVAL, "mixed strategy: all weights are zero");
        return -1;
    }
    if (positive == 1)
        return subs[only];
    double target = mt_uniform_real(g, 0.0, 1.0) * total;
    for (int k = 0; k < 4; ++k) {
        target -= cfg->mix_weights[k];
        if (target < 0.0)
            return subs[k];
    }
    return subs[3];
}

/* select_pair (strategies.hpp:273-285); returns candidate index or -1 */
static int select_pair(const osys* s, const opairs* all, const opairs* c,
                       const tcse_process_config* cfg, mt64* g, int* err) {
    switch (cfg->strategy) {
        case TCSE_GREEDY: return greedy_from(c);
        case TCSE_GREEDY_ALTERNATIVE: return greedy_alternative_from(c, g);
        case TCSE_WEIGHTED_RANDOM: return weighted_random_from(c, g);
        case TCSE_GREEDY_RANDOM: return greedy_random_from(c, cfg, g);
        case TCSE_GREEDY_INTERSECTIONS: return greedy_intersections_from(c, cfg, g);
        case TCSE_MIXED: {
            /* select_mixed (strategies.hpp:260-269) */
            int sub = pick_mixed_substrategy(cfg, g, err);
            switch (sub) {
                case TCSE_GREEDY_INTERSECTIONS: return greedy_intersections_from(c, cfg, g);
                case TCSE_GREEDY_ALTERNATIVE: return greedy_alternative_from(c, g);
                case TCSE_GREEDY_RANDOM: return greedy_random_from(c, cfg, g);
                case TCSE_WEIGHTED_RANDOM: return weighted_random_from(c, g);
                default: return -1;
            }
        }
        case TCSE_GREEDY_POTENTIAL: return greedy_potential_from(s, all, c, cfg->alpha);
        default: *err = fail(TCSE_EINVAL, "select_pair: unknown strategy"); return -1;
    }
}

/* FNV-1a over little-endian int32 words */
static uint64_t fnv_i32(uint64_t h, int32_t v) {
    uint32_t u = (uint32_t)v;
    for (int b = 0; b < 4; ++b) {
        h ^= (u >> (8 * b)) & 0xffu;
        h *= 0x100000001b3ULL;
    }
    return h;
}

uint64_t or_sequence_fnv(const tcse_pair* subs, int32_t n) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (int32_t t = 0; t < n; ++t) {
        h = fnv_i32(h, subs[t].i);
        h = fnv_i32(h, subs[t].j);
        h = fnv_i32(h, subs[t].rel_sign);
    }
    return h;
}

static uint64_t candidates_fnv(const opairs* c) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (int t = 0; t < c->n; ++t) {
        tcse_pair q = key_pair(c->v[t].key);
        h = fnv_i32(h, q.i);
        h = fnv_i32(h, q.j);
        h = fnv_i32(h, q.rel_sign);
        h = fnv_i32(h, c->v[t].count);
    }
    return h;
}

/* run_cse (cse_engine.hpp:29-43) on state s (consumed), rng g */
static int run_cse_state(osys* s, const tcse_process_config* cfg, mt64* g, tcse_record* out,
                         uint64_t* trace, int trace_cap) {
    out->n_subs = 0;
    out->strategy = cfg->strategy;
    out->seed = cfg->seed;
    int step = 0;
    for (;;) {
        opairs all = osys_count(s);
        opairs c = candidates_of(&all);
        if (trace && step < trace_cap)
            trace[step] = candidates_fnv(&c);
        ++step;
        int err = 0;
        int pick = select_pair(s, &all, &c, cfg, g, &err);
        if (err) {
            free(all.v);
            free(c.v);
            return err;
        }
        if (pick < 0) {
            free(all.v);
            free(c.v);
            break;
        }
        tcse_pair q = key_pair(c.v[pick].key);
        free(all.v);
        free(c.v);
        osys_apply(s, q);
        if (out->n_subs >= out->cap)
            return fail(TCSE_ECAPACITY, "run_cse: record capacity %d exceeded", out->cap);
        out->subs[out->n_subs++] = q;
    }
    out->cost = osys_total(s);
    return TCSE_OK;
}

int or_count_pairs(const tcse_system* sys, const tcse_pair* prefix, int32_t n_prefix,
                   int32_t min_count, tcse_pair_count* out, int32_t cap, int32_t* n_out) {
    osys s;
    int rc = osys_init(&s, sys);
    if (rc)
        return rc;
    rc = osys_replay(&s, prefix, n_prefix);
    if (rc) {
        osys_free(&s);
        return rc;
    }
    opairs all = osys_count(&s);
    int n = 0;
    for (int t = 0; t < all.n; ++t) {
        if (all.v[t].count < min_count)
            continue;
        if (n < cap) {
            out[n].pair = key_pair(all.v[t].key);
            out[n].count = all.v[t].count;
        }
        ++n;
    }
    free(all.v);
    osys_free(&s);
    *n_out = n;
    return n > cap ? fail(TCSE_ECAPACITY, "count_pairs: %d pairs exceed capacity %d", n, cap) : TCSE_OK;
}

int or_run_cse(const tcse_system* sys, const tcse_pair* prefix, int32_t n_prefix,
               const tcse_process_config* cfg, tcse_record* out, uint64_t* trace,
               int32_t trace_cap) {
    osys s;
    int rc = osys_init(&s, sys);
    if (rc)
        return rc;
    rc = osys_replay(&s, prefix, n_prefix);
    if (rc == TCSE_OK) {
        mt64 g;
        mt_seed(&g, cfg->seed);
        rc = run_cse_state(&s, cfg, &g, out, trace, trace_cap);
    }
    osys_free(&s);
    return rc;
}

/* ------------------------------------------------------ orchestration */

int or_run_process(const tcse_system* sys, const tcse_process_config* slot, int32_t reinit,
                   const tcse_pair* incumbent, int32_t inc_len, tcse_record* out, int32_t* own) {
    osys s;
    int rc = osys_init(&s, sys);
    if (rc)
        return rc;
    mt64 g;
    mt_seed(&g, slot->seed);
    int k = 0;
    if (reinit) {
        const uint64_t k_max = (uint64_t)(3 * inc_len / 4);
        k = (int)mt_uniform_int(&g, 1, k_max);
        rc = osys_replay(&s, incumbent, k);
        if (rc) {
            osys_free(&s);
            return rc;
        }
    }
    tcse_record rec = *out;
    rec.subs = out->subs + k;
    rec.cap = out->cap - k;
    rc = run_cse_state(&s, slot, &g, &rec, NULL, 0);
    osys_free(&s);
    if (rc)
        return rc;
    memcpy(out->subs, incumbent, sizeof(tcse_pair) * (size_t)k);
    out->n_subs = k + rec.n_subs;
    out->cost = rec.cost;
    out->strategy = rec.strategy;
    out->seed = rec.seed;
    *own = rec.n_subs;
    return TCSE_OK;
}

/* validate_config (parallel_search.hpp:117-140), flip mode excluded */
static int validate_config(const tcse_search_config* cfg) {
    if (cfg->n_processes < 0)
        return fail(TCSE_EINVAL, "search config: n_processes must be >= 0");
    if (cfg->reinit_fraction < 0.0 || cfg->reinit_fraction > 1.0)
        return fail(TCSE_EINVAL, "search config: reinit_fraction must be in [0, 1]");
    if (cfg->patience < 1)
        return fail(TCSE_EINVAL, "search config: patience must be >= 1");
    if (cfg->forced_strategy < 0) {
        double total = 0.0;
        for (int k = 0; k < TCSE_STRATEGY_COUNT; ++k) {
            if (cfg->strategy_weights[k] < 0.0)
                return fail(TCSE_EINVAL, "search config: strategy weights must be >= 0");
            total += cfg->strategy_weights[k];
        }
        if (total <= 0.0)
            return fail(TCSE_EINVAL, "search config: all strategy weights are zero");
    }
    return TCSE_OK;
}

/* assign_strategies (parallel_search.hpp:172-208) */
int or_assign_strategies(const tcse_search_config* cfg, int32_t iteration, int32_t n,
                         uint64_t salt, tcse_process_config* out) {
    int rc = validate_config(cfg);
    if (rc)
        return rc;
    if (n < 1)
        return fail(TCSE_EINVAL, "assign_strategies: need at least one process");
    double weight_total = 0.0;
    for (int k = 0; k < TCSE_STRATEGY_COUNT; ++k)
        weight_total += cfg->strategy_weights[k];
    for (int32_t p = 0; p < n; ++p) {
        const uint64_t parts[4] = {cfg->master_seed, salt, (uint64_t)(int64_t)iteration, (uint64_t)p};
        mt64 prng;
        mt_seed(&prng, or_mix_seed(parts, 4));
        tcse_process_config* pc = &out[p];
        memset(pc, 0, sizeof *pc);
        for (int k = 0; k < 4; ++k)
            pc->mix_weights[k] = cfg->mix_weights[k];
        pc->alpha = mt_uniform_real(&prng, 0.0, 0.5);
        pc->beta = mt_uniform_real(&prng, 0.5, 1.0);
        pc->p_greedy = mt_uniform_real(&prng, 0.5, 1.0);
        if (cfg->forced_strategy >= 0) {
            pc->strategy = cfg->forced_strategy;
        } else if (iteration == 1 && p == 0) {
            pc->strategy = TCSE_GREEDY;
        } else {
            double target = mt_uniform_real(&prng, 0.0, 1.0) * weight_total;
            pc->strategy = TCSE_GREEDY;
            for (int k = 0; k < TCSE_STRATEGY_COUNT; ++k) {
                target -= cfg->strategy_weights[k];
                if (target < 0.0) {
                    pc->strategy = k;
                    break;
                }
            }
        }
        pc->seed = mt_next(&prng);
    }
    return TCSE_OK;
}

/* pick_reinit (parallel_search.hpp:149-163): worst llround(f*n) by cost,
 * stable ties by index */
int or_pick_reinit(const int32_t* last_cost, int32_t n, double fraction, uint8_t* out) {
    memset(out, 0, (size_t)n);
    long long want = llround(fraction * (double)n);
    int32_t count = want < (long long)n ? (int32_t)want : n;
    if (count <= 0)
        return TCSE_OK;
    /* stable order by cost descending = sort by (cost desc, index asc) */
    for (int32_t p = 0; p < n; ++p) {
        int32_t rank = 0;
        for (int32_t q = 0; q < n; ++q)
            if (last_cost[q] > last_cost[p] || (last_cost[q] == last_cost[p] && q < p))
                ++rank;
        out[p] = rank < count;
    }
    return TCSE_OK;
}

typedef struct {
    tcse_pair* subs;
    int n, cost, strategy;
    uint64_t seed;
} orec;

/* optimize_system (parallel_search.hpp:220-273), processes run in index
 * order (the reference's outcome does not depend on scheduling) */
int or_optimize_system(const tcse_system* sys, const tcse_search_config* cfg, uint64_t salt,
                       tcse_record* best, int32_t* iterations, uint64_t* steps) {
    int rc = validate_config(cfg);
    if (rc)
        return rc;
    osys base;
    rc = osys_init(&base, sys);
    if (rc)
        return rc;
    const int n = cfg->n_processes > 0 ? cfg->n_processes : 256;
    const int cap = osys_naive(&base) + 1;
    orec* results = calloc((size_t)n, sizeof(orec));
    for (int p = 0; p < n; ++p)
        results[p].subs = malloc(sizeof(tcse_pair) * (size_t)cap);
    int32_t* last_cost = calloc((size_t)n, sizeof(int32_t));
    uint8_t* reinit = calloc((size_t)n, 1);
    tcse_process_config* slots = malloc(sizeof(tcse_process_config) * (size_t)n);
    tcse_pair* inc = malloc(sizeof(tcse_pair) * (size_t)cap);
    int have_inc = 0, inc_n = 0, inc_cost = 0, inc_strategy = 0;
    uint64_t inc_seed = 0, total_steps = 0;
    int unchanged = 0, iteration = 0;
    for (;;) {
        ++iteration;
        rc = or_assign_strategies(cfg, iteration, n, salt, slots);
        if (rc)
            goto done;
        memset(reinit, 0, (size_t)n);
        if (iteration >= 2 && have_inc && inc_n >= 2)
            or_pick_reinit(last_cost, n, cfg->reinit_fraction, reinit);
        for (int p = 0; p < n; ++p) {
            mt64 g;
            mt_seed(&g, slots[p].seed);
            osys s;
            osys_copy(&s, &base);
            int k = 0;
            if (reinit[p]) {
                const uint64_t k_max = (uint64_t)(3 * inc_n / 4);
                k = (int)mt_uniform_int(&g, 1, k_max);
                rc = osys_replay(&s, inc, k);
                if (rc) {
                    osys_free(&s);
                    goto done;
                }
            }
            tcse_record rec;
            rec.subs = results[p].subs + k;
            rec.cap = cap - k;
            rc = run_cse_state(&s, &slots[p], &g, &rec, NULL, 0);
            osys_free(&s);
            if (rc)
                goto done;
            memcpy(results[p].subs, inc, sizeof(tcse_pair) * (size_t)k);
            results[p].n = k + rec.n_subs;
            results[p].cost = rec.cost;
            results[p].strategy = rec.strategy;
            results[p].seed = rec.seed;
            total_steps += (uint64_t)rec.n_subs;
        }
        int best_p = 0;
        for (int p = 0; p < n; ++p) {
            last_cost[p] = results[p].cost;
            if (results[p].cost < results[best_p].cost)
                best_p = p;
        }
        if (!have_inc || results[best_p].cost < inc_cost) {
            have_inc = 1;
            inc_n = results[best_p].n;
            inc_cost = results[best_p].cost;
            inc_strategy = results[best_p].strategy;
            inc_seed = results[best_p].seed;
            memcpy(inc, results[best_p].subs, sizeof(tcse_pair) * (size_t)inc_n);
            unchanged = 0;
        } else {
            ++unchanged;
        }
        if (unchanged >= cfg->patience)
            break;
        if (cfg->max_iterations > 0 && iteration >= cfg->max_iterations)
            break;
    }
    if (inc_n > best->cap) {
        rc = fail(TCSE_ECAPACITY, "optimize_system: record capacity %d < %d", best->cap, inc_n);
        goto done;
    }
    memcpy(best->subs, inc, sizeof(tcse_pair) * (size_t)inc_n);
    best->n_subs = inc_n;
    best->cost = inc_cost;
    best->strategy = inc_strategy;
    best->seed = inc_seed;
    *iterations = iteration;
    if (steps)
        *steps = total_steps;
done:
    for (int p = 0; p < n; ++p)
        free(results[p].subs);
    free(results);
    free(last_cost);
    free(reinit);
    free(slots);
    free(inc);
    osys_free(&base);
    return rc;
}

/* expand_and_verify (linear_system.hpp:208-258) of replay_prefix(sys, subs) */
int or_verify_record(const tcse_system* sys, const tcse_pair* subs, int32_t n_subs,
                     int32_t* cost_out) {
    osys s;
    int rc = osys_init(&s, sys);
    if (rc)
        return rc;
    rc = osys_replay(&s, subs, n_subs);
    if (rc) {
        osys_free(&s);
        return rc;
    }
    *cost_out = osys_total(&s);
    /* expansion of every variable as a dense coefficient vector over x_1..x_nx */
    const int nv = s.n_x + s.n_f;
    long long* ex = calloc((size_t)(nv + 1) * (size_t)(s.n_x + 1), sizeof(long long));
    for (int v = 1; v <= s.n_x; ++v)
        ex[(size_t)v * (size_t)(s.n_x + 1) + (size_t)v] = 1;
    for (int t = 0; t < s.n_f; ++t) {
        const int id = s.n_x + t + 1;
        const tcse_pair q = s.defs[t];
        long long* row = ex + (size_t)id * (size_t)(s.n_x + 1);
        for (int b = 1; b <= s.n_x; ++b)
            row[b] = ex[(size_t)q.i * (size_t)(s.n_x + 1) + (size_t)b]
                   + (long long)q.rel_sign * ex[(size_t)q.j * (size_t)(s.n_x + 1) + (size_t)b];
    }
    int ok = 1;
    long long* acc = calloc((size_t)s.n_x + 1, sizeof(long long));
    for (int r = 0; r < s.n_e && ok; ++r) {
        memset(acc, 0, sizeof(long long) * ((size_t)s.n_x + 1));
        for (int t = 0; t < s.len[r]; ++t) {
            int term = s.rows[r][t];
            long long sign = term > 0 ? 1 : -1;
            for (int b = 1; b <= s.n_x; ++b)
                acc[b] += sign * ex[(size_t)abs(term) * (size_t)(s.n_x + 1) + (size_t)b];
        }
        int nonzero = 0;
        for (int b = 1; b <= s.n_x && ok; ++b) {
            if (acc[b] == 0)
                continue;
            ++nonzero;
            if (acc[b] != 1 && acc[b] != -1) {
                ok = 0;
                break;
            }
            /* original expression must hold the signed term */
            int want = acc[b] > 0 ? b : -b, found = 0;
            for (int t = sys->row_ptr[r]; t < sys->row_ptr[r + 1]; ++t)
                found |= sys->terms[t] == want;
            if (!found)
                ok = 0;
        }
        if (ok && nonzero != sys->row_ptr[r + 1] - sys->row_ptr[r])
            ok = 0;
    }
    free(acc);
    free(ex);
    osys_free(&s);
    return ok;
}
