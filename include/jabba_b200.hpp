// jabba_b200.hpp — C++ drop-in for the reference's fit/reconstruct entry points.
//
// Include AFTER the reference's "jabba/jabba.hpp": the functions below take
// and return the reference's own value types, so a caller switches with a
// one-line change:
//     jabba::jabba_fit(ds, cfg)     ->  jabba_b200::fit_transform(ds, cfg)
//     jabba::reconstruct(symbolic)  ->  jabba_b200::inverse_transform(symbolic)
// Errors are rethrown as the reference's exception classes (core.hpp:20-30).
// All compute runs on the GPU through the C ABI (include/jabba_b200.h).
#pragma once

#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "jabba_b200.h"

namespace jabba_b200 {

[[noreturn]] inline void rethrow(jb_status st) {
    const std::string msg = jb_last_error();
    switch (st) {
        case JB_INVALID_INPUT: throw jabba::invalid_input(msg);
        case JB_INVALID_PIECE: throw jabba::invalid_piece(msg);
        case JB_INVALID_PARTITION: throw jabba::invalid_partition(msg);
        case JB_UNKNOWN_SYMBOL: throw jabba::unknown_symbol(msg);
        case JB_PARSE_ERROR: throw jabba::parse_error(msg);
        case JB_LAYOUT_ERROR: throw jabba::layout_error(msg);
        case JB_VERSION_ERROR: throw jabba::version_error(msg);
        default: throw jabba::error("jabba_b200: " + msg);
    }
}

inline void check(jb_status st) {
    if (st != JB_OK) rethrow(st);
}

// One CUDA context per thread (the reference's functions are reentrant).
inline jb_context* context(int device = 0) {
    struct Holder {
        jb_context* ctx = nullptr;
        ~Holder() {
            if (ctx) jb_context_destroy(ctx);
        }
    };
    thread_local Holder h;
    if (!h.ctx) check(jb_context_create(device, &h.ctx));
    return h.ctx;
}

inline jb_config to_c(const jabba::JabbaConfig& c) {
    jb_config o;
    jb_config_default(&o);
    o.tol = c.compression.tol;
    o.max_piece_len = c.compression.max_piece_len;
    o.backend = static_cast<int32_t>(c.digitize.backend);
    o.scl = c.digitize.scl;
    o.k = c.digitize.vq.k;
    o.r = c.digitize.vq.r;
    o.max_iters = c.digitize.vq.max_iters;
    o.n_init = c.digitize.vq.n_init;
    o.seed = c.digitize.vq.seed;
    o.alpha = c.digitize.ga.alpha;
    o.sort_key = c.digitize.ga.sort_key == jabba::SortKey::two_norm ? JB_SORT_TWO_NORM
                                                                     : JB_SORT_FIRST_PRINCIPAL_COMPONENT;
    o.early_stop = c.digitize.ga.early_stop ? 1 : 0;
    o.has_alpha_len = c.digitize.ga.alpha_len.has_value();
    o.alpha_len = c.digitize.ga.alpha_len.value_or(0.0);
    o.has_alpha_inc = c.digitize.ga.alpha_inc.has_value();
    o.alpha_inc = c.digitize.ga.alpha_inc.value_or(0.0);
    o.eta = c.digitize.auto_digitize.eta;
    o.threads = c.threads;
    return o;
}

// jabba::jabba_fit (jabba.hpp:30-36) on the GPU.
inline jabba::JabbaFit fit_transform(const jabba::Dataset& ds, jabba::JabbaConfig cfg) {
    if (ds.series.empty()) throw jabba::invalid_input("empty dataset");
    std::vector<int64_t> lengths;
    std::vector<double> values;
    for (const auto& s : ds.series) {
        lengths.push_back(static_cast<int64_t>(s.values.size()));
        values.insert(values.end(), s.values.begin(), s.values.end());
    }
    const int32_t layout = static_cast<int32_t>(ds.layout);
    if (layout != JB_LAYOUT_UNIVARIATE_PARTITIONED && ds.m != ds.series.size())
        throw jabba::layout_error("dataset m does not match member count");
    const int64_t parts =
        layout == JB_LAYOUT_UNIVARIATE_PARTITIONED ? static_cast<int64_t>(ds.m) : 1;
    std::vector<int64_t> first(lengths.size() * std::max<int64_t>(parts, 1)),
        steps(first.size());
    int64_t n_seg = 0;
    check(jb_plan_segments(lengths.data(), (int64_t)lengths.size(), layout, parts, first.data(),
                           steps.data(), &n_seg));
    const jb_config c = to_c(cfg);
    jb_fit* raw = nullptr;
    check(jb_fit_transform(context(), values.data(), (int64_t)values.size(), 0, first.data(),
                           steps.data(), n_seg, layout, &c, &raw));
    std::unique_ptr<jb_fit, void (*)(jb_fit*)> fit(raw, jb_fit_free);
    const int64_t N = jb_fit_n_pieces(raw);
    const uint64_t k = jb_fit_k(raw);
    std::vector<int64_t> off(n_seg + 1), len(N), sl(n_seg);
    std::vector<double> inc(N), centers(2 * k), ml(k), scaling(3), anchors(n_seg);
    std::vector<uint32_t> labels(N);
    check(jb_fit_copy_pieces(raw, off.data(), len.data(), inc.data()));
    check(jb_fit_copy_symbolic(raw, labels.data(), centers.data(), ml.data(), scaling.data(),
                               anchors.data(), sl.data()));
    // segment ids as partitional_compress / split_series name them (compression.hpp:153)
    std::vector<std::string> ids;
    if (layout == JB_LAYOUT_UNIVARIATE_PARTITIONED) {
        for (int64_t s = 0; s < n_seg; ++s)
            ids.push_back(ds.series.front().id + "[" + std::to_string(s) + "]");
    } else {
        for (const auto& s : ds.series) ids.push_back(s.id);
    }
    jabba::JabbaFit out;
    out.batch.layout = ds.layout;
    out.symbolic.layout = ds.layout;
    auto& cb = out.symbolic.codebook;
    cb.scaling.scl = scaling[0];
    cb.scaling.sigma_len = scaling[1];
    cb.scaling.sigma_inc = scaling[2];
    cb.digitizer_tag = jabba::to_string(cfg.digitize.backend);
    for (uint64_t g = 0; g < k; ++g) {
        cb.centers.push_back({centers[2 * g], centers[2 * g + 1]});
        cb.mean_lengths.push_back(ml[g]);
        cb.symbols.push_back(jabba::symbol_token(g, k));
    }
    for (int64_t s = 0; s < n_seg; ++s) {
        jabba::PieceSequence seq;
        seq.anchor = anchors[s];
        seq.source_id = ids[s];
        seq.source_length = sl[s];
        jabba::SymbolicResult::Series ser;
        ser.id = ids[s];
        ser.anchor = anchors[s];
        ser.source_length = sl[s];
        for (int64_t j = off[s]; j < off[s + 1]; ++j) {
            seq.pieces.push_back(jabba::Piece{len[j], inc[j]});
            ser.labels.push_back(labels[j]);
        }
        out.batch.segments.push_back(std::move(seq));
        out.symbolic.series.push_back(std::move(ser));
    }
    return out;
}

// jabba::reconstruct (inverse.hpp:127-132) on the GPU.
inline std::vector<jabba::TimeSeries> inverse_transform(const jabba::SymbolicResult& sym) {
    const auto& cb = sym.codebook;
    const uint64_t k = cb.size();
    std::vector<double> centers, anchors;
    for (const auto& c : cb.centers) {
        centers.push_back(c[0]);
        centers.push_back(c[1]);
    }
    const double scaling[3] = {cb.scaling.scl, cb.scaling.sigma_len, cb.scaling.sigma_inc};
    std::vector<int64_t> off{0}, sl;
    std::vector<uint32_t> labels;
    for (const auto& s : sym.series) {
        labels.insert(labels.end(), s.labels.begin(), s.labels.end());
        off.push_back((int64_t)labels.size());
        anchors.push_back(s.anchor);
        sl.push_back(s.source_length);
    }
    const int32_t layout = static_cast<int32_t>(sym.layout);
    const int64_t n_seg = (int64_t)sym.series.size();
    std::vector<double> out(std::max<int64_t>(jb_reconstruct_size(sl.data(), n_seg, layout), 1));
    check(jb_inverse_transform(context(), centers.data(), cb.mean_lengths.data(), k, scaling,
                               labels.data(), off.data(), anchors.data(), sl.data(), n_seg,
                               layout, out.data()));
    std::vector<jabba::TimeSeries> res;
    if (sym.layout == jabba::Layout::univariate_partitioned) {
        std::string id = sym.series.front().id;
        const auto b = id.find('[');
        if (b != std::string::npos) id.resize(b);
        out.resize(jb_reconstruct_size(sl.data(), n_seg, layout));
        res.emplace_back(std::move(out), id);
        return res;
    }
    int64_t pos = 0;
    for (const auto& s : sym.series) {
        const int64_t n = s.source_length + 1;
        res.emplace_back(std::vector<double>(out.begin() + pos, out.begin() + pos + n), s.id);
        pos += n;
    }
    return res;
}

// jabba::symbolize_with (digitization.hpp:297-307) on the GPU.
inline jabba::SymbolicResult::Series symbolize_with(const jabba::Codebook& codebook,
                                                    const jabba::PieceSequence& seq) {
    if (codebook.size() == 0) throw jabba::invalid_input("symbolize_with: empty codebook");
    std::vector<double> centers;
    for (const auto& c : codebook.centers) {
        centers.push_back(c[0]);
        centers.push_back(c[1]);
    }
    const double scaling[3] = {codebook.scaling.scl, codebook.scaling.sigma_len,
                               codebook.scaling.sigma_inc};
    std::vector<int64_t> len;
    std::vector<double> inc;
    for (const auto& p : seq.pieces) {
        len.push_back(p.len);
        inc.push_back(p.inc);
    }
    jabba::SymbolicResult::Series s;
    s.id = seq.source_id;
    s.anchor = seq.anchor;
    s.source_length = seq.source_length;
    s.labels.resize(len.size());
    check(jb_symbolize_with(context(), centers.data(), (uint64_t)codebook.size(), scaling,
                            len.data(), inc.data(), (int64_t)len.size(), 0, s.labels.data()));
    return s;
}

}  // namespace jabba_b200
