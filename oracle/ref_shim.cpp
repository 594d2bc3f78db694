// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// Binds the UNMODIFIED reference headers (/root/reference/proj/include, added
// with -I by oracle/Makefile; nothing is copied) to the same flat C argument
// conventions as oracle/jabba_oracle.h and include/jabba_b200.h, so tests can
// run the reference itself on the same vectors. Built into
// oracle/_ref/libjabba_ref.so with the reference's own flags
// (proj/CMakeLists.txt:5-10: C++20, -O3, no -march => no FMA).
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "jabba/jabba.hpp"

extern "C" {
#include "jabba_oracle.h"
}

namespace {
thread_local std::string g_err;

int map_error(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const jabba::invalid_input*>(&e)) return 1;
    if (dynamic_cast<const jabba::invalid_piece*>(&e)) return 2;
    if (dynamic_cast<const jabba::invalid_partition*>(&e)) return 3;
    if (dynamic_cast<const jabba::unknown_symbol*>(&e)) return 4;
    if (dynamic_cast<const jabba::parse_error*>(&e)) return 5;
    if (dynamic_cast<const jabba::layout_error*>(&e)) return 6;
    if (dynamic_cast<const jabba::version_error*>(&e)) return 7;
    return 103;
}

jabba::JabbaConfig to_cfg(const jo_config* c) {
    jabba::JabbaConfig cfg;
    cfg.compression.tol = c->tol;
    cfg.compression.max_piece_len = c->max_piece_len;
    cfg.digitize.backend = static_cast<jabba::Backend>(c->backend);
    cfg.digitize.scl = c->scl;
    cfg.digitize.vq.k = c->k;
    cfg.digitize.vq.r = c->r;
    cfg.digitize.vq.max_iters = c->max_iters;
    cfg.digitize.vq.n_init = c->n_init;
    cfg.digitize.vq.seed = c->seed;
    cfg.digitize.ga.alpha = c->alpha;
    cfg.digitize.ga.sort_key = c->sort_key == 1 ? jabba::SortKey::two_norm
                                                : jabba::SortKey::first_principal_component;
    cfg.digitize.ga.early_stop = c->early_stop != 0;
    if (c->has_alpha_len) cfg.digitize.ga.alpha_len = c->alpha_len;
    if (c->has_alpha_inc) cfg.digitize.ga.alpha_inc = c->alpha_inc;
    cfg.digitize.auto_digitize.eta = c->eta;
    cfg.threads = c->threads;
    return cfg;
}

// Builds the reference Dataset for a segment table. A univariate-partitioned
// table (layout 0) is passed through Dataset::partitioned so split_series runs
// inside the reference; other layouts pass each segment as a member series.
jabba::Dataset to_dataset(const double* values, const int64_t* seg_first,
                          const int64_t* seg_steps, int64_t n_seg, int32_t layout) {
    std::vector<jabba::TimeSeries> members;
    if (layout == 0) {
        const int64_t first = seg_first[0];
        const int64_t last = seg_first[n_seg - 1] + seg_steps[n_seg - 1];
        jabba::TimeSeries ts(std::vector<double>(values + first, values + last + 1), "s");
        return jabba::Dataset::partitioned(std::move(ts), static_cast<std::size_t>(n_seg));
    }
    for (int64_t s = 0; s < n_seg; ++s)
        members.emplace_back(
            std::vector<double>(values + seg_first[s], values + seg_first[s] + seg_steps[s] + 1),
            "s" + std::to_string(s));
    if (layout == 1) return jabba::Dataset::multivariate(std::move(members));
    return jabba::Dataset::collection(std::move(members));
}
}  // namespace

extern "C" {

const char* jref_last_error(void) { return g_err.c_str(); }

// jabba_fit (jabba.hpp:30-36) on the flat segment table
int jref_fit(const double* values, const int64_t* seg_first, const int64_t* seg_steps,
             int64_t n_seg, int32_t layout, const jo_config* c, jo_fit_result* out) {
    std::memset(out, 0, sizeof *out);
    try {
        const auto ds = to_dataset(values, seg_first, seg_steps, n_seg, layout);
        const auto fit = jabba::jabba_fit(ds, to_cfg(c));
        const auto& b = fit.batch;
        const auto& sym = fit.symbolic;
        out->n_seg = static_cast<int64_t>(b.segments.size());
        out->n_pieces = static_cast<int64_t>(b.total_pieces());
        out->piece_offsets = (int64_t*)malloc(sizeof(int64_t) * (out->n_seg + 1));
        out->piece_len = (int64_t*)malloc(sizeof(int64_t) * (out->n_pieces + 1));
        out->piece_inc = (double*)malloc(sizeof(double) * (out->n_pieces + 1));
        out->labels = (uint32_t*)malloc(sizeof(uint32_t) * (out->n_pieces + 1));
        out->anchors = (double*)malloc(sizeof(double) * out->n_seg);
        out->source_lengths = (int64_t*)malloc(sizeof(int64_t) * out->n_seg);
        int64_t p = 0;
        out->piece_offsets[0] = 0;
        for (std::size_t s = 0; s < b.segments.size(); ++s) {
            const auto& seg = b.segments[s];
            for (std::size_t i = 0; i < seg.pieces.size(); ++i) {
                out->piece_len[p] = seg.pieces[i].len;
                out->piece_inc[p] = seg.pieces[i].inc;
                out->labels[p] = sym.series[s].labels[i];
                ++p;
            }
            out->piece_offsets[s + 1] = p;
            out->anchors[s] = seg.anchor;
            out->source_lengths[s] = seg.source_length;
        }
        const auto& cb = sym.codebook;
        out->k = cb.size();
        out->centers = (double*)malloc(sizeof(double) * (2 * out->k + 1));
        out->mean_lengths = (double*)malloc(sizeof(double) * (out->k + 1));
        for (std::size_t g = 0; g < cb.size(); ++g) {
            out->centers[2 * g] = cb.centers[g][0];
            out->centers[2 * g + 1] = cb.centers[g][1];
            out->mean_lengths[g] = cb.mean_lengths[g];
        }
        out->scaling[0] = cb.scaling.scl;
        out->scaling[1] = cb.scaling.sigma_len;
        out->scaling[2] = cb.scaling.sigma_inc;
        return 0;
    } catch (const std::exception& e) {
        return map_error(e);
    }
}

void jref_fit_free(jo_fit_result* r) {
    free(r->piece_offsets);
    free(r->piece_len);
    free(r->piece_inc);
    free(r->anchors);
    free(r->source_lengths);
    free(r->centers);
    free(r->mean_lengths);
    free(r->labels);
    std::memset(r, 0, sizeof *r);
}

// reconstruct (inverse.hpp:127-132) from a flat symbolic result
int jref_reconstruct(const double* centers, const double* mean_lengths, uint64_t k,
                     const double* scaling, const uint32_t* labels,
                     const int64_t* piece_offsets, const double* anchors,
                     const int64_t* source_lengths, int64_t n_seg, int32_t layout,
                     double* out_values) {
    try {
        jabba::SymbolicResult sym;
        sym.layout = static_cast<jabba::Layout>(layout);
        sym.codebook.scaling.scl = scaling[0];
        sym.codebook.scaling.sigma_len = scaling[1];
        sym.codebook.scaling.sigma_inc = scaling[2];
        for (uint64_t g = 0; g < k; ++g) {
            sym.codebook.centers.push_back({centers[2 * g], centers[2 * g + 1]});
            sym.codebook.mean_lengths.push_back(mean_lengths[g]);
            sym.codebook.symbols.push_back(jabba::symbol_token(g, k));
        }
        for (int64_t s = 0; s < n_seg; ++s) {
            jabba::SymbolicResult::Series ser;
            ser.id = "s" + std::to_string(s) + "[" + std::to_string(s) + "]";
            ser.anchor = anchors[s];
            ser.source_length = source_lengths[s];
            ser.labels.assign(labels + piece_offsets[s], labels + piece_offsets[s + 1]);
            sym.series.push_back(std::move(ser));
        }
        const auto out = jabba::reconstruct(sym);
        int64_t pos = 0;
        for (const auto& ts : out) {
            std::memcpy(out_values + pos, ts.values.data(), sizeof(double) * ts.values.size());
            pos += static_cast<int64_t>(ts.values.size());
        }
        return 0;
    } catch (const std::exception& e) {
        return map_error(e);
    }
}

// symbolize_with (digitization.hpp:297-307) through the reference's own code
int jref_symbolize_with(const double* centers, uint64_t k, const double* scaling,
                        const int64_t* len, const double* inc, int64_t n, uint32_t* labels) {
    try {
        jabba::Codebook cb;
        cb.scaling.scl = scaling[0];
        cb.scaling.sigma_len = scaling[1];
        cb.scaling.sigma_inc = scaling[2];
        for (uint64_t g = 0; g < k; ++g) {
            cb.centers.push_back({centers[2 * g], centers[2 * g + 1]});
            cb.mean_lengths.push_back(1.0);
            cb.symbols.push_back(jabba::symbol_token(g, k));
        }
        jabba::PieceSequence seq;
        for (int64_t i = 0; i < n; ++i) seq.pieces.push_back(jabba::Piece{len[i], inc[i]});
        const auto s = jabba::symbolize_with(cb, seq);
        std::memcpy(labels, s.labels.data(), sizeof(uint32_t) * s.labels.size());
        return 0;
    } catch (const std::exception& e) {
        return map_error(e);
    }
}

// --- building blocks, for pinning the restatement ---

void jref_mt_stream(uint64_t seed, uint64_t count, uint64_t* out) {
    std::mt19937_64 g(seed);
    for (uint64_t i = 0; i < count; ++i) out[i] = g();
}

void jref_uniform_int_stream(uint64_t seed, uint64_t lo, uint64_t hi, uint64_t count,
                             uint64_t* out) {
    std::mt19937_64 g(seed);
    std::uniform_int_distribution<std::size_t> d(lo, hi);
    for (uint64_t i = 0; i < count; ++i) out[i] = d(g);
}

void jref_uniform_real_stream(uint64_t seed, double lo, double hi, uint64_t count, double* out) {
    std::mt19937_64 g(seed);
    for (uint64_t i = 0; i < count; ++i) out[i] = std::uniform_real_distribution<double>(lo, hi)(g);
}

int jref_sample_indices(uint64_t n, uint64_t s, uint64_t seed, uint64_t* out) {
    std::mt19937_64 g(seed);
    const auto idx = jabba::detail::sample_indices(n, s, g);
    for (uint64_t i = 0; i < s; ++i) out[i] = idx[i];
    return 0;
}

int jref_kmeans(const double* pts, int64_t n, uint64_t k, uint64_t max_iters, uint64_t n_init,
                uint64_t seed, uint32_t* labels, double* centers, uint64_t* iterations) {
    try {
        std::vector<jabba::Point2> p(n);
        for (int64_t i = 0; i < n; ++i) p[i] = {pts[2 * i], pts[2 * i + 1]};
        jabba::VQConfig cfg;
        cfg.k = k;
        cfg.max_iters = max_iters;
        cfg.n_init = n_init;
        cfg.seed = seed;
        const auto res = jabba::kmeans(p, cfg);
        for (int64_t i = 0; i < n; ++i) labels[i] = res.labels[i];
        for (uint64_t c = 0; c < k; ++c) {
            centers[2 * c] = res.centers[c][0];
            centers[2 * c + 1] = res.centers[c][1];
        }
        *iterations = res.iterations;
        return 0;
    } catch (const std::exception& e) {
        return map_error(e);
    }
}

int jref_greedy_aggregate(const double* pts, int64_t n, double alpha, int32_t sort_key,
                          int32_t early_stop, uint32_t* labels, int64_t* n_groups,
                          int64_t* starting_points) {
    try {
        std::vector<jabba::Point2> p(n);
        for (int64_t i = 0; i < n; ++i) p[i] = {pts[2 * i], pts[2 * i + 1]};
        jabba::GAConfig cfg;
        cfg.alpha = alpha;
        cfg.sort_key = sort_key == 1 ? jabba::SortKey::two_norm
                                     : jabba::SortKey::first_principal_component;
        cfg.early_stop = early_stop != 0;
        const auto res = jabba::greedy_aggregate(p, cfg);
        for (int64_t i = 0; i < n; ++i) labels[i] = res.labels[i];
        *n_groups = static_cast<int64_t>(res.groups());
        for (std::size_t g = 0; g < res.starting_points.size(); ++g)
            starting_points[g] = static_cast<int64_t>(res.starting_points[g]);
        return 0;
    } catch (const std::exception& e) {
        return map_error(e);
    }
}

double jref_auto_alpha(int64_t n, int64_t N, double tol, double eta, int* status) {
    try {
        *status = 0;
        return jabba::auto_alpha(n, N, tol, eta);
    } catch (const std::exception& e) {
        *status = map_error(e);
        return 0.0;
    }
}

void jref_quantize_lengths(const double* real_lens, int64_t n, int64_t* out) {
    const auto q = jabba::quantize_lengths(std::vector<double>(real_lens, real_lens + n));
    for (int64_t i = 0; i < n; ++i) out[i] = q[i];
}

}  // extern "C"
