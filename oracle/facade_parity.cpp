// facade_parity.cpp — TEST INFRASTRUCTURE ONLY.
//
// Runs the reference's own C++ entry points (jabba::jabba_fit /
// jabba::reconstruct, the UNMODIFIED headers under /root/reference/proj) and
// the drop-in (jabba_b200::fit_transform / inverse_transform over the GPU C
// ABI) side by side in one process, on inputs built with the reference
// suite's own generators (proj/tests/oracles.hpp oracle::walk,
// bench.hpp random_walk / gaussian_noise). One PASS/FAIL line per case;
// exit code = number of failures (the acceptance.cpp convention).
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>

#include "jabba/bench.hpp"
#include "jabba/jabba.hpp"
#include "oracles.hpp"
#include "jabba_b200.hpp"

using namespace jabba;

static int failures = 0;

static void report(const std::string& name, bool ok, const std::string& why = "") {
    std::printf("%s %s%s%s\n", ok ? "PASS" : "FAIL", name.c_str(), why.empty() ? "" : ": ",
                why.c_str());
    if (!ok) ++failures;
}

static bool close_rel(double a, double b, double rel) {
    return std::abs(a - b) <= rel * std::max({1.0, std::abs(a), std::abs(b)});
}

static void compare(const std::string& name, const Dataset& ds, const JabbaConfig& cfg) {
    try {
        const JabbaFit ref = jabba_fit(ds, cfg);
        const JabbaFit got = jabba_b200::fit_transform(ds, cfg);
        std::string why;
        if (got.batch.segments.size() != ref.batch.segments.size()) why = "segment count";
        for (size_t s = 0; why.empty() && s < ref.batch.segments.size(); ++s) {
            const auto& a = ref.batch.segments[s];
            const auto& b = got.batch.segments[s];
            if (a.pieces.size() != b.pieces.size()) why = "piece count, segment " + std::to_string(s);
            for (size_t i = 0; why.empty() && i < a.pieces.size(); ++i)
                if (a.pieces[i].len != b.pieces[i].len || a.pieces[i].inc != b.pieces[i].inc)
                    why = "piece " + std::to_string(i) + " of segment " + std::to_string(s);
            if (why.empty() && (a.anchor != b.anchor || a.source_length != b.source_length ||
                                a.source_id != b.source_id))
                why = "segment metadata " + std::to_string(s);
            if (why.empty() && ref.symbolic.tokens(s) != got.symbolic.tokens(s))
                why = "symbols of segment " + std::to_string(s);
        }
        const auto& ca = ref.symbolic.codebook;
        const auto& cbk = got.symbolic.codebook;
        if (why.empty() && (ca.size() != cbk.size() || ca.symbols != cbk.symbols ||
                            ca.digitizer_tag != cbk.digitizer_tag))
            why = "codebook alphabet";
        for (size_t g = 0; why.empty() && g < ca.size(); ++g)
            if (!close_rel(ca.centers[g][0], cbk.centers[g][0], 1e-9) ||
                !close_rel(ca.centers[g][1], cbk.centers[g][1], 1e-9) ||
                !close_rel(ca.mean_lengths[g], cbk.mean_lengths[g], 1e-12))
                why = "center " + std::to_string(g);
        if (why.empty()) {
            const auto ra = reconstruct(ref.symbolic);
            const auto rb = jabba_b200::inverse_transform(got.symbolic);
            if (ra.size() != rb.size()) why = "reconstruction count";
            for (size_t s = 0; why.empty() && s < ra.size(); ++s) {
                if (ra[s].values.size() != rb[s].values.size() || ra[s].id != rb[s].id) {
                    why = "reconstruction shape " + std::to_string(s);
                    break;
                }
                for (size_t i = 0; i < ra[s].values.size(); ++i)
                    if (!close_rel(ra[s].values[i], rb[s].values[i], 1e-9)) {
                        why = "reconstructed sample " + std::to_string(i);
                        break;
                    }
            }
        }
        report(name, why.empty(), why);
    } catch (const std::exception& e) {
        report(name, false, std::string("exception: ") + e.what());
    }
}

template <class E>
static void expect_throw(const std::string& name, const std::function<void()>& f) {
    try {
        f();
        report(name, false, "no exception");
    } catch (const E&) {
        report(name, true);
    } catch (const std::exception& e) {
        report(name, false, std::string("wrong exception: ") + e.what());
    }
}

int main() {
    // test_compression.cpp / acceptance.cpp style inputs
    const auto walk = oracle::walk(4000, 99);
    for (Backend b : {Backend::vq, Backend::sampling_vq, Backend::ga, Backend::ga_auto,
                      Backend::ga_hier}) {
        JabbaConfig cfg;
        cfg.compression.tol = 0.25;
        cfg.digitize.backend = b;
        cfg.digitize.vq.k = 12;
        cfg.digitize.vq.r = 0.5;
        cfg.digitize.vq.seed = 7;
        cfg.digitize.ga.alpha = 0.4;
        compare(std::string("partitioned walk x8 ") + to_string(b), Dataset::partitioned(walk, 8),
                cfg);
    }
    {
        std::vector<TimeSeries> dims;
        for (int d = 0; d < 6; ++d) dims.push_back(oracle::walk(3000, 100 + d));
        for (auto& d : dims) d.id = "dim" + std::to_string(d.values.size());
        JabbaConfig cfg;
        cfg.compression.tol = 0.1;
        cfg.digitize.backend = Backend::sampling_vq;
        cfg.digitize.vq.k = 20;
        cfg.digitize.vq.r = 0.3;
        compare("multivariate 6x3000 svq", Dataset::multivariate(dims), cfg);
        cfg.digitize.backend = Backend::ga;
        cfg.digitize.ga.sort_key = SortKey::two_norm;
        cfg.digitize.ga.alpha = 0.2;
        compare("multivariate 6x3000 ga two-norm", Dataset::multivariate(dims), cfg);
    }
    {
        const auto noise = gaussian_noise(100000, 42);
        JabbaConfig cfg;
        cfg.compression.tol = 0.01;
        cfg.digitize.backend = Backend::ga;
        cfg.digitize.ga.alpha = 0.05;
        compare("gaussian noise 1e5 ga (PAPER.md:559 setting)", Dataset::collection({noise}), cfg);
        const auto rw = random_walk(200000, 42);
        cfg.compression.tol = 0.1;
        cfg.digitize.backend = Backend::sampling_vq;
        cfg.digitize.vq.k = 50;
        cfg.digitize.vq.r = 0.5;
        compare("random walk 2e5 svq k50", Dataset::partitioned(rw, 16), cfg);
        cfg.compression.max_piece_len = 7;
        compare("random walk 2e5 svq max_piece_len 7", Dataset::partitioned(rw, 16), cfg);
    }
    // symbolize_with (digitization.hpp:297-307): held-out pieces against a
    // fitted codebook, as test_io.cpp:108-116 / acceptance.cpp:368 use it
    for (Backend b : {Backend::vq, Backend::sampling_vq, Backend::ga}) {
        JabbaConfig cfg;
        cfg.compression.tol = 0.2;
        cfg.digitize.backend = b;
        cfg.digitize.vq.k = 16;
        cfg.digitize.vq.r = 0.5;
        cfg.digitize.ga.alpha = 0.3;
        const JabbaFit fit = jabba_fit(Dataset::partitioned(oracle::walk(20000, 5), 4), cfg);
        const PieceSequence held = compress(oracle::walk(30000, 99), {0.2, 0});
        const auto ref = symbolize_with(fit.symbolic.codebook, held);
        const auto got = jabba_b200::symbolize_with(fit.symbolic.codebook, held);
        const bool same_labels = got.labels == ref.labels;
        const bool ok = same_labels && got.anchor == ref.anchor &&
                        got.source_length == ref.source_length;
        report(std::string("symbolize_with held-out walk, ") + to_string(b) + " codebook", ok,
               ok ? "" : (same_labels ? "metadata" : "labels"));
    }
    expect_throw<invalid_input>("symbolize_with: empty codebook", [] {
        jabba_b200::symbolize_with(Codebook{}, compress(oracle::walk(100, 3), {0.2, 0}));
    });
    // error classes at the reference's call sites
    expect_throw<invalid_partition>("oversized partition count", [] {
        jabba_b200::fit_transform(Dataset::partitioned(TimeSeries{{0, 1, 2, 3}, "tiny"}, 4),
                                  JabbaConfig{});
    });
    expect_throw<invalid_input>("non-finite input", [] {
        auto ts = oracle::walk(400, 1);
        ts.values[350] = std::nan("");
        jabba_b200::fit_transform(Dataset::partitioned(ts, 8), JabbaConfig{});
    });
    expect_throw<invalid_input>("tol must be > 0", [] {
        JabbaConfig cfg;
        cfg.compression.tol = 0.0;
        jabba_b200::fit_transform(Dataset::collection({oracle::walk(100, 1)}), cfg);
    });
    expect_throw<unknown_symbol>("label outside the codebook", [] {
        JabbaConfig cfg;
        auto fit = jabba_b200::fit_transform(Dataset::collection({oracle::walk(300, 4)}), cfg);
        fit.symbolic.series[0].labels[0] = 10000;
        jabba_b200::inverse_transform(fit.symbolic);
    });
    std::printf("%d failure(s)\n", failures);
    return failures;
}
