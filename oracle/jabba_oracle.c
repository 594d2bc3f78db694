/*
 * jabba_oracle.c — TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * Plain-C restatement of the reference JABBA path. Every function cites the
 * reference file:line it restates; paths are relative to
 * /root/reference/proj/include/jabba/. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this code.
 *
 * Floating point: compiled with -O2 -ffp-contract=off and no -march, which
 * matches the reference's own build (proj/CMakeLists.txt:5-10: -O3, no
 * -march => SSE2 binary64, no FMA contraction).
 *
 * RNG: std::mt19937_64 plus libstdc++ (GCC 13.3) uniform_int_distribution
 * (128-bit Lemire "nearly divisionless" downscaling for a full 64-bit engine)
 * and uniform_real_distribution (generate_canonical<double,53>: one engine
 * draw, double(x) / 2^64, clamped below 1). Pinned draw-for-draw against the
 * real std:: implementation by tests/test_oracle_golden.py (test_rng_matches_libstdcxx).
 */
#include "jabba_oracle.h"

#include <float.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* jo_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* std::mt19937_64 (ISO C++ [rand.eng.mers], parameters of mt19937_64)       */

typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt_next(mt64* g) {
    if (g->idx >= 312) {
        const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

/* uniform_int_distribution<size_t>(lo, hi): libstdc++ bits/uniform_int_dist.h,
 * engine range 2^64-1 > urange -> _S_nd<unsigned __int128> (Lemire). Used by
 * clustering.hpp:80 (sample_indices) and :103-104 (first D^2 center). */
static uint64_t uniform_int(mt64* g, uint64_t lo, uint64_t hi) {
    const uint64_t urange = hi - lo;
    if (urange == UINT64_MAX) return mt_next(g) + lo;
    const uint64_t erange = urange + 1;
    unsigned __int128 prod = (unsigned __int128)mt_next(g) * erange;
    uint64_t low = (uint64_t)prod;
    if (low < erange) {
        const uint64_t thresh = (0 - erange) % erange;
        while (low < thresh) {
            prod = (unsigned __int128)mt_next(g) * erange;
            low = (uint64_t)prod;
        }
    }
    return (uint64_t)(prod >> 64) + lo;
}

/* uniform_real_distribution<double>(lo, hi): generate_canonical<double,53>
 * (one draw for a 64-bit engine) * (hi - lo) + lo. clustering.hpp:61. */
static double uniform_real(mt64* g, double lo, double hi) {
    double c = (double)mt_next(g) / 18446744073709551616.0;
    if (c >= 1.0) c = nextafter(1.0, 0.0);
    return c * (hi - lo) + lo;
}

void jo_mt_stream(uint64_t seed, uint64_t count, uint64_t* out) {
    mt64 g;
    mt_seed(&g, seed);
    for (uint64_t i = 0; i < count; ++i) out[i] = mt_next(&g);
}

uint64_t jo_uniform_int_stream(uint64_t seed, uint64_t lo, uint64_t hi, uint64_t count,
                               uint64_t* out) {
    mt64 g;
    mt_seed(&g, seed);
    for (uint64_t i = 0; i < count; ++i) out[i] = uniform_int(&g, lo, hi);
    return 0;
}

void jo_uniform_real_stream(uint64_t seed, double lo, double hi, uint64_t count, double* out) {
    mt64 g;
    mt_seed(&g, seed);
    for (uint64_t i = 0; i < count; ++i) out[i] = uniform_real(&g, lo, hi);
}

/* ------------------------------------------------------------------------ */
/* Segment planning: Dataset factories core.hpp:73-98, split_series
 * compression.hpp:140-160, partitional_compress checks :167-184.            */

int jo_plan_segments(const int64_t* series_lengths, int64_t n_series, int32_t layout,
                     int64_t parts, int64_t* seg_first, int64_t* seg_steps,
                     int64_t* n_seg_out) {
    if (n_series <= 0) return fail(JO_INVALID_INPUT, "empty dataset");
    if (layout == 0 && n_series != 1)
        return fail(JO_LAYOUT_ERROR,
                    "univariate-partitioned dataset must hold exactly one series");
    if (layout == 1)
        for (int64_t s = 1; s < n_series; ++s)
            if (series_lengths[s] != series_lengths[0])
                return fail(JO_LAYOUT_ERROR, "multivariate dataset has ragged dimensions");
    int64_t nseg = 0, first = 0;
    for (int64_t s = 0; s < n_series; ++s) {
        const int64_t len = series_lengths[s];
        const int64_t steps = len == 0 ? 0 : len - 1;
        if (parts == 1 && layout != 0) {
            seg_first[nseg] = first;
            seg_steps[nseg] = steps;
            ++nseg;
        } else {
            if (parts == 0) return fail(JO_INVALID_PARTITION, "partition count must be >= 1");
            if (parts > steps)
                return fail(JO_INVALID_PARTITION, "cannot split %lld steps into %lld segments",
                            (long long)steps, (long long)parts);
            const int64_t base = steps / parts, extra = steps % parts;
            int64_t begin = first;
            for (int64_t p = 0; p < parts; ++p) {
                const int64_t st = base + (p < extra ? 1 : 0);
                seg_first[nseg] = begin;
                seg_steps[nseg] = st;
                ++nseg;
                begin += st;
            }
        }
        first += len;
    }
    *n_seg_out = nseg;
    return JO_OK;
}

/* ------------------------------------------------------------------------ */
/* Compression: detail::compress_range compression.hpp:31-66                 */

typedef struct {
    int64_t* len;
    double* inc;
    int64_t n, cap;
} piece_vec;

static void pv_push(piece_vec* v, int64_t len, double inc) {
    if (v->n == v->cap) {
        v->cap = v->cap ? v->cap * 2 : 1024;
        v->len = (int64_t*)realloc(v->len, sizeof(int64_t) * v->cap);
        v->inc = (double*)realloc(v->inc, sizeof(double) * v->cap);
    }
    v->len[v->n] = len;
    v->inc[v->n] = inc;
    ++v->n;
}

static void compress_range(const double* v, int64_t first, int64_t last, double tol,
                           int64_t max_piece_len, piece_vec* out) {
    const double tol2 = tol * tol;
    int64_t start = first;
    while (start < last) {
        const double base = v[start];
        double s2 = 0.0, s3 = 0.0; /* s1 (:37,44) is dead in the reference */
        int64_t end = start;
        for (;;) {
            const int64_t cand = end + 1;
            if (cand > last) break;
            const double y = v[cand] - base;
            const double d = (double)(cand - start);
            const double ns2 = s2 + y * y;
            const double ns3 = s3 + d * y;
            const double len = d;
            const double inc = y;
            const double sum_d2 = len * (len + 1.0) * (2.0 * len + 1.0) / 6.0;
            const double sq_dev = inc * inc / (len * len) * sum_d2 - 2.0 * inc / len * ns3 + ns2;
            if (sq_dev > (len - 1.0) * tol2 && cand > start + 1) break;
            end = cand;
            s2 = ns2;
            s3 = ns3;
            if (max_piece_len > 0 && end - start >= max_piece_len) break;
        }
        pv_push(out, end - start, v[end] - base);
        start = end;
    }
}

/* compress (compression.hpp:70-83) over every segment, joined in input order
 * (partitional_compress :167-193; the fork-join result is thread-count
 * independent, parallel.hpp:3-5, so the sequential loop is the contract). */
int jo_compress(const double* values, const int64_t* seg_first, const int64_t* seg_steps,
                int64_t n_seg, double tol, int64_t max_piece_len, int64_t* piece_offsets,
                int64_t** piece_len, double** piece_inc) {
    if (!(tol > 0.0)) return fail(JO_INVALID_INPUT, "compression tol must be > 0");
    if (max_piece_len < 0) return fail(JO_INVALID_INPUT, "max_piece_len must be >= 0");
    if (n_seg <= 0) return fail(JO_INVALID_INPUT, "empty dataset");
    for (int64_t s = 0; s < n_seg; ++s) {
        if (seg_steps[s] < 1)
            return fail(JO_INVALID_INPUT, "compression needs at least 2 samples");
        for (int64_t i = seg_first[s]; i <= seg_first[s] + seg_steps[s]; ++i)
            if (!isfinite(values[i]))
                return fail(JO_INVALID_INPUT, "compression input has non-finite values");
    }
    piece_vec pv = {0};
    piece_offsets[0] = 0;
    for (int64_t s = 0; s < n_seg; ++s) {
        compress_range(values, seg_first[s], seg_first[s] + seg_steps[s], tol, max_piece_len,
                       &pv);
        piece_offsets[s + 1] = pv.n;
    }
    *piece_len = pv.len;
    *piece_inc = pv.inc;
    return JO_OK;
}

/* ------------------------------------------------------------------------ */
/* Clustering (clustering.hpp)                                               */

static inline double dist2(const double* a, const double* b) { /* :52-56 */
    const double dx = a[0] - b[0];
    const double dy = a[1] - b[1];
    return dx * dx + dy * dy;
}

/* detail::weighted_index :59-71 */
static int64_t weighted_index(const double* w, int64_t n, double total, mt64* rng) {
    const double u = uniform_real(rng, 0.0, total);
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        acc += w[i];
        if (u < acc) return i;
    }
    for (int64_t i = n; i-- > 0;)
        if (w[i] > 0.0) return i;
    return n - 1;
}

/* detail::sample_indices :74-85 (partial Fisher-Yates over iota(n)) */
static uint64_t* sample_indices(uint64_t n, uint64_t s, mt64* rng) {
    uint64_t* idx = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    for (uint64_t i = 0; i < n; ++i) idx[i] = i;
    for (uint64_t i = 0; i < s; ++i) {
        const uint64_t j = i + uniform_int(rng, 0, n - 1 - i);
        const uint64_t t = idx[i];
        idx[i] = idx[j];
        idx[j] = t;
    }
    return idx;
}

int jo_sample_indices(uint64_t n, uint64_t sample_size, uint64_t seed, uint64_t* out) {
    mt64 g;
    mt_seed(&g, seed);
    uint64_t* idx = sample_indices(n, sample_size, &g);
    memcpy(out, idx, sizeof(uint64_t) * sample_size);
    free(idx);
    return JO_OK;
}

/* d2_seed :92-131 */
static int d2_seed(const double* pts, int64_t n, uint64_t k, mt64* rng, double* centers) {
    if (k < 1) return fail(JO_INVALID_INPUT, "d2_seed: k must be >= 1");
    if ((int64_t)k > n) return fail(JO_INVALID_INPUT, "d2_seed: k exceeds points");
    char* chosen = (char*)calloc(n, 1);
    double* d2 = (double*)malloc(sizeof(double) * n);
    double* w = (double*)malloc(sizeof(double) * n);
    const uint64_t first = uniform_int(rng, 0, (uint64_t)n - 1);
    centers[0] = pts[2 * first];
    centers[1] = pts[2 * first + 1];
    chosen[first] = 1;
    for (int64_t i = 0; i < n; ++i) d2[i] = dist2(pts + 2 * i, centers);
    for (uint64_t c = 1; c < k; ++c) {
        double total = 0.0;
        for (int64_t i = 0; i < n; ++i) total += chosen[i] ? 0.0 : d2[i];
        int64_t next;
        if (total > 0.0) {
            for (int64_t i = 0; i < n; ++i) w[i] = chosen[i] ? 0.0 : d2[i];
            next = weighted_index(w, n, total, rng);
        } else {
            next = 0;
            while (next < n && chosen[next]) ++next;
        }
        chosen[next] = 1;
        centers[2 * c] = pts[2 * next];
        centers[2 * c + 1] = pts[2 * next + 1];
        for (int64_t i = 0; i < n; ++i) {
            const double dd = dist2(pts + 2 * i, centers + 2 * c);
            if (dd < d2[i]) d2[i] = dd; /* std::min(a,b) == (b < a) ? b : a */
        }
    }
    free(chosen);
    free(d2);
    free(w);
    return JO_OK;
}

/* detail::nearest_center :146-157 */
static uint32_t nearest_center(const double* p, const double* centers, uint64_t k) {
    uint32_t best = 0;
    double best_d = INFINITY;
    for (uint64_t c = 0; c < k; ++c) {
        const double d = dist2(p, centers + 2 * c);
        if (d < best_d) {
            best_d = d;
            best = (uint32_t)c;
        }
    }
    return best;
}

static void assign_all(const double* pts, int64_t n, const double* centers, uint64_t k,
                       uint32_t* labels) { /* :159-163 */
    for (int64_t i = 0; i < n; ++i) labels[i] = nearest_center(pts + 2 * i, centers, k);
}

/* detail::update_means :167-198 (with empty-cluster re-seeding) */
static void update_means(const double* pts, int64_t n, uint32_t* labels, double* centers,
                         uint64_t k) {
    double* sums = (double*)calloc(2 * k, sizeof(double));
    uint64_t* counts = (uint64_t*)calloc(k, sizeof(uint64_t));
    for (int64_t i = 0; i < n; ++i) {
        sums[2 * labels[i]] += pts[2 * i];
        sums[2 * labels[i] + 1] += pts[2 * i + 1];
        ++counts[labels[i]];
    }
    for (uint64_t c = 0; c < k; ++c)
        if (counts[c] > 0) {
            centers[2 * c] = sums[2 * c] / (double)counts[c];
            centers[2 * c + 1] = sums[2 * c + 1] / (double)counts[c];
        }
    for (uint64_t c = 0; c < k; ++c) {
        if (counts[c] > 0) continue;
        int64_t far_i = 0;
        double far_d = -1.0;
        for (int64_t i = 0; i < n; ++i) {
            if (counts[labels[i]] <= 1) continue;
            const double d = dist2(pts + 2 * i, centers + 2 * labels[i]);
            if (d > far_d) {
                far_d = d;
                far_i = i;
            }
        }
        --counts[labels[far_i]];
        labels[far_i] = (uint32_t)c;
        counts[c] = 1;
        centers[2 * c] = pts[2 * far_i];
        centers[2 * c + 1] = pts[2 * far_i + 1];
    }
    free(sums);
    free(counts);
}

/* sse metrics.hpp:52-64 */
static double sse(const double* pts, int64_t n, const uint32_t* labels, const double* centers) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double* c = centers + 2 * labels[i];
        const double dx = pts[2 * i] - c[0];
        const double dy = pts[2 * i + 1] - c[1];
        acc += dx * dx + dy * dy;
    }
    return acc;
}

/* detail::lloyd_once :200-220. labels/centers are outputs. */
static int lloyd_once(const double* pts, int64_t n, uint64_t k, uint64_t max_iters, mt64* rng,
                      uint32_t* labels, double* centers, double* sse_out, uint64_t* iters) {
    int st = d2_seed(pts, n, k, rng, centers);
    if (st) return st;
    assign_all(pts, n, centers, k, labels);
    uint32_t* next = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    uint64_t it = 0;
    for (; it < max_iters; ++it) {
        update_means(pts, n, labels, centers, k);
        /* sse_trace (:208) only feeds the dead trace; skipped */
        assign_all(pts, n, centers, k, next);
        if (memcmp(next, labels, sizeof(uint32_t) * n) == 0) {
            ++it;
            break;
        }
        memcpy(labels, next, sizeof(uint32_t) * n);
    }
    *iters = it;
    free(next);
    update_means(pts, n, labels, centers, k);
    *sse_out = sse(pts, n, labels, centers);
    return JO_OK;
}

static int validate_vq(uint64_t k, double r, uint64_t max_iters, uint64_t n_init) {
    if (k < 1) return fail(JO_INVALID_INPUT, "VQConfig: k must be >= 1");
    if (!(r > 0.0 && r <= 1.0)) return fail(JO_INVALID_INPUT, "VQConfig: r must be in (0,1]");
    if (max_iters < 1) return fail(JO_INVALID_INPUT, "VQConfig: max_iters must be >= 1");
    if (n_init < 1) return fail(JO_INVALID_INPUT, "VQConfig: n_init must be >= 1");
    return JO_OK;
}

/* best of n_init lloyd_once runs on one rng stream (kmeans :224-236,
 * sampling_kmeans inner loop :266-270) */
static int lloyd_best(const double* pts, int64_t n, uint64_t k, uint64_t max_iters,
                      uint64_t n_init, mt64* rng, uint32_t* labels, double* centers,
                      uint64_t* iterations) {
    uint32_t* rl = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    double* rc = (double*)malloc(sizeof(double) * 2 * k);
    double best_sse = 0.0;
    for (uint64_t r = 0; r < n_init; ++r) {
        double s;
        uint64_t it;
        int st = lloyd_once(pts, n, k, max_iters, rng, rl, rc, &s, &it);
        if (st) {
            free(rl);
            free(rc);
            return st;
        }
        if (r == 0 || s < best_sse) {
            best_sse = s;
            memcpy(labels, rl, sizeof(uint32_t) * n);
            memcpy(centers, rc, sizeof(double) * 2 * k);
            *iterations = it;
        }
    }
    free(rl);
    free(rc);
    return JO_OK;
}

int jo_kmeans(const double* pts, int64_t n, uint64_t k, uint64_t max_iters, uint64_t n_init,
              uint64_t seed, uint32_t* labels, double* centers, uint64_t* iterations) {
    int st = validate_vq(k, 1.0, max_iters, n_init);
    if (st) return st;
    if ((int64_t)k > n) return fail(JO_INVALID_INPUT, "kmeans: k exceeds points");
    mt64 g;
    mt_seed(&g, seed);
    return lloyd_best(pts, n, k, max_iters, n_init, &g, labels, centers, iterations);
}

/* ------------------------------------------------------------------------ */
/* Greedy aggregation :292-375                                               */

static const double* g_sort_keys;
static int cmp_key_stable(const void* a, const void* b) {
    const int64_t ia = *(const int64_t*)a, ib = *(const int64_t*)b;
    const double ka = g_sort_keys[ia], kb = g_sort_keys[ib];
    if (ka < kb) return -1;
    if (kb < ka) return 1;
    return ia < ib ? -1 : (ia > ib);
}

/* detail::sort_keys :292-324 */
static void sort_keys(const double* pts, int64_t n, int32_t key, double* keys) {
    if (key == 1) {
        for (int64_t i = 0; i < n; ++i)
            keys[i] = sqrt(pts[2 * i] * pts[2 * i] + pts[2 * i + 1] * pts[2 * i + 1]);
        return;
    }
    const double dn = (double)n;
    double mx = 0.0, my = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        mx += pts[2 * i];
        my += pts[2 * i + 1];
    }
    mx /= dn;
    my /= dn;
    double sxx = 0.0, sxy = 0.0, syy = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double dx = pts[2 * i] - mx, dy = pts[2 * i + 1] - my;
        sxx += dx * dx;
        sxy += dx * dy;
        syy += dy * dy;
    }
    const double theta = 0.5 * atan2(2.0 * sxy, sxx - syy);
    double vx = cos(theta), vy = sin(theta);
    if (vx < 0.0 || (vx == 0.0 && vy < 0.0)) {
        vx = -vx;
        vy = -vy;
    }
    for (int64_t i = 0; i < n; ++i)
        keys[i] = vx * (pts[2 * i] - mx) + vy * (pts[2 * i + 1] - my);
}

/* greedy_aggregate :328-375. centers (2*groups) optional. */
static int greedy_aggregate(const double* pts, int64_t n, double alpha, int32_t sort_key,
                            int32_t early_stop, uint32_t* labels, int64_t* n_groups,
                            int64_t* starting_points, double** centers_out) {
    if (!(alpha > 0.0)) return fail(JO_INVALID_INPUT, "GAConfig: alpha must be > 0");
    if (n <= 0) return fail(JO_INVALID_INPUT, "greedy_aggregate: no points");
    const double alpha2 = alpha * alpha;
    double* keys = (double*)malloc(sizeof(double) * n);
    sort_keys(pts, n, sort_key, keys);
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * n);
    for (int64_t i = 0; i < n; ++i) order[i] = i;
    g_sort_keys = keys; /* std::stable_sort == sort by (key, index) */
    qsort(order, n, sizeof(int64_t), cmp_key_stable);
    char* assigned = (char*)calloc(n, 1);
    double* sums = (double*)malloc(sizeof(double) * 2 * n);
    int64_t* counts = (int64_t*)malloc(sizeof(int64_t) * n);
    int64_t groups = 0;
    for (int64_t si = 0; si < n; ++si) {
        const int64_t sp = order[si];
        if (assigned[sp]) continue;
        const uint32_t g = (uint32_t)groups;
        if (starting_points) starting_points[groups] = sp;
        sums[2 * g] = pts[2 * sp];
        sums[2 * g + 1] = pts[2 * sp + 1];
        counts[g] = 1;
        ++groups;
        assigned[sp] = 1;
        labels[sp] = g;
        for (int64_t sj = si + 1; sj < n; ++sj) {
            const int64_t j = order[sj];
            if (early_stop && keys[j] - keys[sp] > alpha) break;
            if (assigned[j]) continue;
            if (dist2(pts + 2 * sp, pts + 2 * j) <= alpha2) {
                assigned[j] = 1;
                labels[j] = g;
                sums[2 * g] += pts[2 * j];
                sums[2 * g + 1] += pts[2 * j + 1];
                ++counts[g];
            }
        }
    }
    if (centers_out) {
        double* c = (double*)malloc(sizeof(double) * 2 * (groups ? groups : 1));
        for (int64_t g = 0; g < groups; ++g) {
            c[2 * g] = sums[2 * g] / (double)counts[g];
            c[2 * g + 1] = sums[2 * g + 1] / (double)counts[g];
        }
        *centers_out = c;
    }
    *n_groups = groups;
    free(keys);
    free(order);
    free(assigned);
    free(sums);
    free(counts);
    return JO_OK;
}

int jo_greedy_aggregate(const double* pts, int64_t n, double alpha, int32_t sort_key,
                        int32_t early_stop, uint32_t* labels, int64_t* n_groups,
                        int64_t* starting_points) {
    return greedy_aggregate(pts, n, alpha, sort_key, early_stop, labels, n_groups,
                            starting_points, NULL);
}

/* auto_alpha digitization.hpp:66-75 */
double jo_auto_alpha(int64_t n, int64_t N, double tol, double eta, int* status) {
    *status = JO_OK;
    if (N < 1 || n <= N) {
        *status = fail(JO_INVALID_INPUT, "auto_alpha: requires n > N >= 1");
        return 0.0;
    }
    if (!(tol > 0.0)) {
        *status = fail(JO_INVALID_INPUT, "auto_alpha: tol must be > 0");
        return 0.0;
    }
    if (!(eta > 0.0)) {
        *status = fail(JO_INVALID_INPUT, "auto_alpha: eta must be > 0");
        return 0.0;
    }
    const double dn = (double)n, dN = (double)N;
    const double poly = 3.0 * dn * dn * dn * dn + 2.0 - 5.0 * dn * dn;
    const double num = 60.0 * dn * (dn - dN) * tol * tol;
    return pow(num / (dN * eta * eta * poly), 0.25);
}

/* ------------------------------------------------------------------------ */
/* Digitization: scale_pieces digitization.hpp:25-59, run_backend :131-198,
 * digitize :207-293                                                         */

typedef struct {
    uint32_t* labels;
    uint64_t k;
    uint64_t* sample;
    uint32_t* sample_labels;
    uint64_t sample_size;
    double* backend_centers;
    uint64_t iterations;
} cluster_run;

static uint64_t* g_pair_keys;
static int cmp_u64_idx(const void* a, const void* b) {
    const int64_t ia = *(const int64_t*)a, ib = *(const int64_t*)b;
    const uint64_t ka = g_pair_keys[ia], kb = g_pair_keys[ib];
    if (ka != kb) return ka < kb ? -1 : 1;
    return ia < ib ? -1 : (ia > ib);
}

static int run_backend(const double* pts, int64_t n, int64_t total_steps, const jo_config* cfg,
                       cluster_run* run) {
    memset(run, 0, sizeof *run);
    run->labels = (uint32_t*)malloc(sizeof(uint32_t) * n);
    int st;
    switch (cfg->backend) {
        case 0: { /* vq :135-143, r forced to 1 */
            st = validate_vq(cfg->k, 1.0, cfg->max_iters, cfg->n_init);
            if (st) return st;
            if ((int64_t)cfg->k > n) return fail(JO_INVALID_INPUT, "kmeans: k exceeds points");
            mt64 g;
            mt_seed(&g, cfg->seed);
            run->backend_centers = (double*)malloc(sizeof(double) * 2 * cfg->k);
            st = lloyd_best(pts, n, cfg->k, cfg->max_iters, cfg->n_init, &g, run->labels,
                            run->backend_centers, &run->iterations);
            if (st) return st;
            run->k = cfg->k;
            return JO_OK;
        }
        case 1: { /* svq :144-152 -> sampling_kmeans clustering.hpp:247-275 */
            st = validate_vq(cfg->k, cfg->r, cfg->max_iters, cfg->n_init);
            if (st) return st;
            if (n <= 0) return fail(JO_INVALID_INPUT, "sampling_kmeans: no points");
            const uint64_t S = (uint64_t)llround(cfg->r * (double)n);
            if (S < cfg->k)
                return fail(JO_INVALID_INPUT,
                            "sampling_kmeans: sample of %llu points is smaller than k=%llu",
                            (unsigned long long)S, (unsigned long long)cfg->k);
            mt64 g;
            mt_seed(&g, cfg->seed);
            uint64_t* idx = sample_indices((uint64_t)n, S, &g);
            double* sp = (double*)malloc(sizeof(double) * 2 * S);
            for (uint64_t s = 0; s < S; ++s) {
                sp[2 * s] = pts[2 * idx[s]];
                sp[2 * s + 1] = pts[2 * idx[s] + 1];
            }
            run->sample = idx;
            run->sample_size = S;
            run->sample_labels = (uint32_t*)malloc(sizeof(uint32_t) * S);
            run->backend_centers = (double*)malloc(sizeof(double) * 2 * cfg->k);
            st = lloyd_best(sp, (int64_t)S, cfg->k, cfg->max_iters, cfg->n_init, &g,
                            run->sample_labels, run->backend_centers, &run->iterations);
            free(sp);
            if (st) return st;
            assign_all(pts, n, run->backend_centers, cfg->k, run->labels);
            run->k = cfg->k;
            return JO_OK;
        }
        case 2:
        case 3: { /* ga / ga-auto :153-167 */
            double alpha = cfg->alpha;
            if (cfg->backend == 3) {
                if (!(cfg->eta > 0.0))
                    return fail(JO_INVALID_INPUT, "AutoDigitizeConfig: eta must be > 0");
                alpha = jo_auto_alpha(total_steps, n, cfg->tol, cfg->eta, &st);
                if (st) return st;
            }
            if (cfg->has_alpha_len && !(cfg->alpha_len > 0.0))
                return fail(JO_INVALID_INPUT, "GAConfig: alpha_len must be > 0");
            if (cfg->has_alpha_inc && !(cfg->alpha_inc > 0.0))
                return fail(JO_INVALID_INPUT, "GAConfig: alpha_inc must be > 0");
            int64_t groups;
            st = greedy_aggregate(pts, n, alpha, cfg->sort_key, cfg->early_stop, run->labels,
                                  &groups, NULL, &run->backend_centers);
            if (st) return st;
            run->k = (uint64_t)groups;
            return JO_OK;
        }
        case 4: { /* ga-hier :168-195 */
            if (!(cfg->alpha > 0.0)) return fail(JO_INVALID_INPUT, "GAConfig: alpha must be > 0");
            if (cfg->has_alpha_len && !(cfg->alpha_len > 0.0))
                return fail(JO_INVALID_INPUT, "GAConfig: alpha_len must be > 0");
            if (cfg->has_alpha_inc && !(cfg->alpha_inc > 0.0))
                return fail(JO_INVALID_INPUT, "GAConfig: alpha_inc must be > 0");
            const double a_len = cfg->has_alpha_len ? cfg->alpha_len : cfg->alpha;
            const double a_inc = cfg->has_alpha_inc ? cfg->alpha_inc : cfg->alpha;
            double* e = (double*)malloc(sizeof(double) * 2 * n);
            uint32_t* gl = (uint32_t*)malloc(sizeof(uint32_t) * n);
            uint32_t* gi = (uint32_t*)malloc(sizeof(uint32_t) * n);
            int64_t ng;
            for (int64_t i = 0; i < n; ++i) {
                e[2 * i] = pts[2 * i];
                e[2 * i + 1] = 0.0;
            }
            st = greedy_aggregate(e, n, a_len, cfg->sort_key, cfg->early_stop, gl, &ng, NULL,
                                  NULL);
            if (!st) {
                for (int64_t i = 0; i < n; ++i) {
                    e[2 * i] = pts[2 * i + 1];
                    e[2 * i + 1] = 0.0;
                }
                st = greedy_aggregate(e, n, a_inc, cfg->sort_key, cfg->early_stop, gi, &ng,
                                      NULL, NULL);
            }
            free(e);
            if (st) {
                free(gl);
                free(gi);
                return st;
            }
            /* pair ids in order of first appearance (the std::map lookup) */
            uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * n);
            int64_t* ord = (int64_t*)malloc(sizeof(int64_t) * n);
            for (int64_t i = 0; i < n; ++i) {
                keys[i] = ((uint64_t)gl[i] << 32) | gi[i];
                ord[i] = i;
            }
            g_pair_keys = keys;
            qsort(ord, n, sizeof(int64_t), cmp_u64_idx);
            /* first occurrence of each key = head of its sorted run */
            int64_t* firstpos = (int64_t*)malloc(sizeof(int64_t) * n);
            for (int64_t a = 0; a < n;) {
                int64_t b = a;
                while (b < n && keys[ord[b]] == keys[ord[a]]) ++b;
                for (int64_t t = a; t < b; ++t) firstpos[ord[t]] = ord[a];
                a = b;
            }
            uint32_t* idmap = (uint32_t*)malloc(sizeof(uint32_t) * n);
            uint32_t next = 0;
            for (int64_t i = 0; i < n; ++i) {
                if (firstpos[i] == i) idmap[i] = next++;
                run->labels[i] = idmap[firstpos[i]];
            }
            run->k = next;
            free(keys);
            free(ord);
            free(firstpos);
            free(idmap);
            free(gl);
            free(gi);
            return JO_OK;
        }
    }
    return fail(JO_INVALID_INPUT, "unknown backend");
}

static uint64_t* g_cnt;
static uint64_t* g_first;
static int cmp_rank(const void* a, const void* b) { /* digitization.hpp:257-262 */
    const uint64_t ga = *(const uint64_t*)a, gb = *(const uint64_t*)b;
    if (g_cnt[ga] != g_cnt[gb]) return g_cnt[ga] > g_cnt[gb] ? -1 : 1;
    if (g_first[ga] != g_first[gb]) return g_first[ga] < g_first[gb] ? -1 : 1;
    return ga < gb ? -1 : (ga > gb); /* stable */
}

int jo_fit(const double* values, const int64_t* seg_first, const int64_t* seg_steps,
           int64_t n_seg, const jo_config* cfg, jo_fit_result* out) {
    memset(out, 0, sizeof *out);
    out->n_seg = n_seg;
    out->piece_offsets = (int64_t*)malloc(sizeof(int64_t) * (n_seg + 1));
    int st = jo_compress(values, seg_first, seg_steps, n_seg, cfg->tol, cfg->max_piece_len,
                         out->piece_offsets, &out->piece_len, &out->piece_inc);
    if (st) return st;
    const int64_t N = out->piece_offsets[n_seg];
    out->n_pieces = N;
    out->anchors = (double*)malloc(sizeof(double) * n_seg);
    out->source_lengths = (int64_t*)malloc(sizeof(int64_t) * n_seg);
    int64_t total_steps = 0;
    for (int64_t s = 0; s < n_seg; ++s) {
        out->anchors[s] = values[seg_first[s]];
        out->source_lengths[s] = seg_steps[s];
        total_steps += seg_steps[s];
    }
    if (N == 0) return fail(JO_INVALID_INPUT, "digitize: no pieces");
    if (cfg->scl < 0.0) return fail(JO_INVALID_INPUT, "scale_pieces: scl must be >= 0");

    /* scale_pieces :25-59 */
    const double dn = (double)N;
    double mean_len = 0.0, mean_inc = 0.0;
    for (int64_t i = 0; i < N; ++i) {
        mean_len += (double)out->piece_len[i];
        mean_inc += out->piece_inc[i];
    }
    mean_len /= dn;
    mean_inc /= dn;
    double var_len = 0.0, var_inc = 0.0;
    for (int64_t i = 0; i < N; ++i) {
        const double dl = (double)out->piece_len[i] - mean_len;
        const double di = out->piece_inc[i] - mean_inc;
        var_len += dl * dl;
        var_inc += di * di;
    }
    double sl = N > 1 ? sqrt(var_len / (dn - 1.0)) : 0.0;
    double si = N > 1 ? sqrt(var_inc / (dn - 1.0)) : 0.0;
    if (sl <= 0.0) sl = 1.0;
    if (si <= 0.0) si = 1.0;
    out->scaling[0] = cfg->scl;
    out->scaling[1] = sl;
    out->scaling[2] = si;
    double* pts = (double*)malloc(sizeof(double) * 2 * N);
    for (int64_t i = 0; i < N; ++i) { /* ScalingParams::apply core.hpp:130-132 */
        pts[2 * i] = cfg->scl * (double)out->piece_len[i] / sl;
        pts[2 * i + 1] = out->piece_inc[i] / si;
    }

    cluster_run run;
    st = run_backend(pts, N, total_steps, cfg, &run);
    if (st) {
        free(pts);
        free(run.labels);
        free(run.sample);
        free(run.sample_labels);
        free(run.backend_centers);
        return st;
    }
    out->iterations = run.iterations;
    out->sample_size = run.sample_size;

    /* group statistics :217-253 */
    const uint64_t k = run.k;
    double* sums = (double*)calloc(2 * k, sizeof(double));
    double* len_sums = (double*)calloc(k, sizeof(double));
    uint64_t* counts = (uint64_t*)calloc(k, sizeof(uint64_t));
    uint64_t* first_seen = (uint64_t*)malloc(sizeof(uint64_t) * k);
    for (uint64_t g = 0; g < k; ++g) first_seen[g] = UINT64_MAX;
    for (int64_t i = 0; i < N; ++i) {
        const uint32_t g = run.labels[i];
        sums[2 * g] += pts[2 * i];
        sums[2 * g + 1] += pts[2 * i + 1];
        len_sums[g] += (double)out->piece_len[i];
        ++counts[g];
        if (first_seen[g] == UINT64_MAX) first_seen[g] = (uint64_t)i;
    }
    double* centers = (double*)malloc(sizeof(double) * 2 * k);
    double* mean_lengths = (double*)malloc(sizeof(double) * k);
    for (uint64_t g = 0; g < k; ++g) {
        if (counts[g] > 0) {
            centers[2 * g] = sums[2 * g] / (double)counts[g];
            centers[2 * g + 1] = sums[2 * g + 1] / (double)counts[g];
            mean_lengths[g] = len_sums[g] / (double)counts[g];
        } else {
            centers[2 * g] = run.backend_centers[2 * g];
            centers[2 * g + 1] = run.backend_centers[2 * g + 1];
            double ls = 0.0;
            uint64_t lc = 0;
            for (uint64_t s = 0; s < run.sample_size; ++s) {
                if (run.sample_labels[s] != g) continue;
                ls += (double)out->piece_len[run.sample[s]];
                ++lc;
            }
            mean_lengths[g] = lc > 0 ? ls / (double)lc : 1.0;
        }
    }
    /* rank order :255-264 */
    uint64_t* order = (uint64_t*)malloc(sizeof(uint64_t) * (k ? k : 1));
    for (uint64_t g = 0; g < k; ++g) order[g] = g;
    g_cnt = counts;
    g_first = first_seen;
    qsort(order, k, sizeof(uint64_t), cmp_rank);
    uint32_t* rank_of = (uint32_t*)malloc(sizeof(uint32_t) * (k ? k : 1));
    for (uint64_t r = 0; r < k; ++r) rank_of[order[r]] = (uint32_t)r;
    out->k = k;
    out->centers = (double*)malloc(sizeof(double) * 2 * (k ? k : 1));
    out->mean_lengths = (double*)malloc(sizeof(double) * (k ? k : 1));
    for (uint64_t r = 0; r < k; ++r) {
        out->centers[2 * r] = centers[2 * order[r]];
        out->centers[2 * r + 1] = centers[2 * order[r] + 1];
        out->mean_lengths[r] = mean_lengths[order[r]];
        if (!isfinite(out->centers[2 * r]) || !isfinite(out->centers[2 * r + 1]))
            st = fail(JO_INVALID_INPUT, "codebook: non-finite center"); /* core.hpp:173-175 */
    }
    out->labels = (uint32_t*)malloc(sizeof(uint32_t) * N);
    for (int64_t i = 0; i < N; ++i) out->labels[i] = rank_of[run.labels[i]]; /* :280-291 */

    free(pts);
    free(sums);
    free(len_sums);
    free(counts);
    free(first_seen);
    free(centers);
    free(mean_lengths);
    free(order);
    free(rank_of);
    free(run.labels);
    free(run.sample);
    free(run.sample_labels);
    free(run.backend_centers);
    return st;
}

void jo_fit_free(jo_fit_result* r) {
    free(r->piece_offsets);
    free(r->piece_len);
    free(r->piece_inc);
    free(r->anchors);
    free(r->source_lengths);
    free(r->centers);
    free(r->mean_lengths);
    free(r->labels);
    memset(r, 0, sizeof *r);
}

/* ------------------------------------------------------------------------ */
/* Inverse (inverse.hpp)                                                     */

/* quantize_lengths inverse.hpp:63-74 */
void jo_quantize_lengths(const double* real_lens, int64_t n, int64_t* out) {
    double carry = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double l = real_lens[i];
        int64_t rounded = (int64_t)llround(l + carry);
        if (rounded < 1) rounded = 1;
        carry = l + carry - (double)rounded;
        out[i] = rounded;
    }
}

/* detail::match_total_length inverse.hpp:81-93 */
int jo_match_total_length(int64_t* lens, int64_t n, int64_t target) {
    int64_t total = 0;
    for (int64_t i = 0; i < n; ++i) total += lens[i];
    int64_t residual = target - total;
    for (int64_t i = n; i-- > 0 && residual != 0;) {
        int64_t adjusted = lens[i] + residual;
        if (adjusted < 1) adjusted = 1;
        residual -= adjusted - lens[i];
        lens[i] = adjusted;
    }
    if (residual != 0)
        return fail(JO_INVALID_PIECE, "cannot fit %lld pieces into %lld steps", (long long)n,
                    (long long)target);
    return JO_OK;
}

/* inverse_compress compression.hpp:87-103; out holds sum(len)+1 values */
int jo_inverse_compress(const int64_t* len, const double* inc, int64_t n, double anchor,
                        double* out) {
    if (n <= 0) return fail(JO_INVALID_PIECE, "inverse_compress: empty piece sequence");
    int64_t pos = 0;
    out[pos++] = anchor;
    double v = anchor;
    for (int64_t j = 0; j < n; ++j) {
        if (len[j] < 1) return fail(JO_INVALID_PIECE, "inverse_compress: piece with len < 1");
        const double l = (double)len[j];
        for (int64_t i = 1; i <= len[j]; ++i) out[pos++] = v + inc[j] * ((double)i / l);
        v += inc[j];
    }
    return JO_OK;
}

/* symbolize_with digitization.hpp:297-307: ScalingParams::apply core.hpp:130-132,
 * Codebook::nearest core.hpp:147-160 (dx = center - q, strict <, lowest index) */
int jo_symbolize_with(const double* centers, uint64_t k, const double* scaling,
                      const int64_t* len, const double* inc, int64_t n, uint32_t* labels) {
    if (k == 0) return fail(JO_INVALID_INPUT, "symbolize_with: empty codebook");
    for (int64_t i = 0; i < n; ++i) {
        const double qx = scaling[0] * (double)len[i] / scaling[1];
        const double qy = inc[i] / scaling[2];
        uint64_t best = 0;
        double best_d = INFINITY;
        for (uint64_t c = 0; c < k; ++c) {
            const double dx = centers[2 * c] - qx;
            const double dy = centers[2 * c + 1] - qy;
            const double d = dx * dx + dy * dy;
            if (d < best_d) {
                best_d = d;
                best = c;
            }
        }
        labels[i] = (uint32_t)best;
    }
    return JO_OK;
}

int64_t jo_reconstruct_size(const int64_t* source_lengths, int64_t n_seg, int32_t layout) {
    int64_t t = 0;
    for (int64_t s = 0; s < n_seg; ++s) t += source_lengths[s] + 1;
    if (layout == 0 && n_seg > 0) t -= n_seg - 1; /* stitch_partitions :198-213 */
    return t;
}

/* reconstruct inverse.hpp:127-132 via inverse_symbolize_series :97-115 */
int jo_reconstruct(const double* centers, const double* mean_lengths, uint64_t k,
                   const double* scaling, const uint32_t* labels, const int64_t* piece_offsets,
                   const double* anchors, const int64_t* source_lengths, int64_t n_seg,
                   int32_t layout, double* out_values) {
    if (n_seg <= 0 && layout == 0) return fail(JO_INVALID_INPUT, "stitch_partitions: no segments");
    const double scl = scaling[0], sl = scaling[1], si = scaling[2];
    int64_t pos = 0;
    for (int64_t s = 0; s < n_seg; ++s) {
        const int64_t a = piece_offsets[s], b = piece_offsets[s + 1], n = b - a;
        double* rl = (double*)malloc(sizeof(double) * (n ? n : 1));
        double* ri = (double*)malloc(sizeof(double) * (n ? n : 1));
        int64_t* ql = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
        for (int64_t j = 0; j < n; ++j) { /* inverse_digitize_series :32-51 */
            const uint32_t lab = labels[a + j];
            if (lab >= k) {
                free(rl);
                free(ri);
                free(ql);
                return fail(JO_UNKNOWN_SYMBOL, "label %u not in codebook of size %llu", lab,
                            (unsigned long long)k);
            }
            rl[j] = scl > 0.0 ? centers[2 * lab] * sl / scl : mean_lengths[lab];
            ri[j] = centers[2 * lab + 1] * si;
        }
        jo_quantize_lengths(rl, n, ql);
        int st = jo_match_total_length(ql, n, source_lengths[s]);
        if (!st) {
            double* tmp = (double*)malloc(sizeof(double) * (source_lengths[s] + 1));
            st = jo_inverse_compress(ql, ri, n, anchors[s], tmp);
            if (!st) {
                /* univariate-partitioned: drop every non-final part's last sample */
                const int64_t cnt =
                    (layout == 0 && s + 1 < n_seg) ? source_lengths[s] : source_lengths[s] + 1;
                memcpy(out_values + pos, tmp, sizeof(double) * cnt);
                pos += cnt;
            }
            free(tmp);
        }
        free(rl);
        free(ri);
        free(ql);
        if (st) return st;
    }
    return JO_OK;
}
