// jabba_cli.cpp — the reference's command-line front end
// (proj/tools/jabba_cli.cpp:51-269) over the C ABI (include/jabba_b200.h):
//   jabba_b200 symbolize   --input F [--format csv-rows|csv-cols|ts-lite] [--tol] [--backend]
//                          [--k] [--alpha] [--r] [--scl] [--eta] [--partitions] [--threads]
//                          [--seed] [--model-out F] [--out F] [--json]
//   jabba_b200 reconstruct --symbols F [--model F] [--out F] [--ref F] [--ref-format]
//   jabba_b200 inspect     --model F
//   jabba_b200 bench partition-sweep [--n] [--tol] [--alpha] [--partitions 1,2,4] [--seed]
//                          [--out F] [--json-out F]
//   jabba_b200 bench multivariate --input F [--format] [--tol] [--eta] [--r] [--scl] [--seed]
//                          [--out F] [--json-out F]
// Exit codes as the reference (jabba_cli.cpp:2): 0 success, 2 usage error, 1
// data / validation error. File formats are those of io.hpp (dataset
// loaders :70-144, model / symbolic JSON :160-289, symbols text :293-338),
// written with the same JSON library the reference builds against, so a
// symbols file, a model and a reconstruction written here read back in the
// reference's CLI and vice versa. No CLI11 (absent offline): flags are
// parsed here, `--name value` and `--name=value`.
#include <charconv>
#include <chrono>
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <array>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <limits>
#include <map>
#include <memory>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include <json.hpp>

#include "../../include/jabba_b200.h"

namespace {

// ---------------------------------------------------------------------------
// errors: data errors exit 1 (the reference's jabba::error), usage errors 2

struct DataError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void check(jb_status st) {
    if (st != JB_OK) throw DataError(jb_last_error());
}

jb_context* ctx() {
    static std::unique_ptr<jb_context, void (*)(jb_context*)> c(nullptr, jb_context_destroy);
    if (!c) {
        jb_context* raw = nullptr;
        check(jb_context_create(0, &raw));
        c.reset(raw);
    }
    return c.get();
}

// ---------------------------------------------------------------------------
// value types (core.hpp:35-215, the fields the front end needs)

struct Series {
    std::string id;
    std::vector<double> values;
};

struct Dataset {
    std::vector<Series> series;
    int32_t layout = JB_LAYOUT_COLLECTION;
    int64_t m = 0;
};

struct Codebook {
    std::vector<std::array<double, 2>> centers;
    std::vector<std::string> symbols;
    std::vector<double> mean_lengths;
    double scl = 1.0, sigma_len = 1.0, sigma_inc = 1.0;
    std::string tag;

    size_t size() const { return centers.size(); }
    size_t index_of(const std::string& tok) const {
        for (size_t i = 0; i < symbols.size(); ++i)
            if (symbols[i] == tok) return i;
        throw DataError("token not in codebook alphabet: \"" + tok + "\"");
    }
    void validate() const {  // Codebook::validate core.hpp:168-180
        if (centers.size() != symbols.size() || centers.size() != mean_lengths.size())
            throw DataError("codebook: centers/symbols/mean_lengths size mismatch");
        if (sigma_len <= 0 || sigma_inc <= 0)
            throw DataError("codebook: scaling sigmas must be positive");
        for (const auto& c : centers)
            if (!std::isfinite(c[0]) || !std::isfinite(c[1]))
                throw DataError("codebook: non-finite center");
        for (size_t i = 0; i < symbols.size(); ++i)
            for (size_t j = i + 1; j < symbols.size(); ++j)
                if (symbols[i] == symbols[j])
                    throw DataError("codebook: duplicate symbol \"" + symbols[i] + "\"");
    }
};

struct SymSeries {
    std::string id;
    double anchor = 0.0;
    int64_t source_length = 0;
    std::vector<uint32_t> labels;
};

struct Symbolic {
    Codebook cb;
    std::vector<SymSeries> series;
    int32_t layout = JB_LAYOUT_COLLECTION;
};

struct Model {
    Codebook cb;
    uint64_t seed = 0;
    double tol = 0.0;
};

const char* layout_name(int32_t l) {
    switch (l) {
        case JB_LAYOUT_UNIVARIATE_PARTITIONED: return "univariate-partitioned";
        case JB_LAYOUT_MULTIVARIATE: return "multivariate";
        default: return "collection";
    }
}

int32_t layout_from(const std::string& s) {
    if (s == "univariate-partitioned") return JB_LAYOUT_UNIVARIATE_PARTITIONED;
    if (s == "multivariate") return JB_LAYOUT_MULTIVARIATE;
    if (s == "collection") return JB_LAYOUT_COLLECTION;
    throw DataError("unknown layout \"" + s + "\"");
}

const char* backend_name(int32_t b) {  // to_string(Backend) digitization.hpp:88-100
    switch (b) {
        case JB_BACKEND_VQ: return "vq";
        case JB_BACKEND_SVQ: return "svq";
        case JB_BACKEND_GA: return "ga";
        case JB_BACKEND_GA_AUTO: return "ga-auto";
        default: return "ga-hier";
    }
}

int32_t backend_from(const std::string& s) {  // backend_from_string digitization.hpp:101-108
    if (s == "vq") return JB_BACKEND_VQ;
    if (s == "svq") return JB_BACKEND_SVQ;
    if (s == "ga") return JB_BACKEND_GA;
    if (s == "ga-auto") return JB_BACKEND_GA_AUTO;
    if (s == "ga-hier") return JB_BACKEND_GA_HIER;
    throw DataError("unknown digitizer backend \"" + s + "\"");
}

std::string token(uint64_t rank, uint64_t k) {
    char buf[32];
    jb_symbol_token(rank, k, buf);
    return buf;
}

// ---------------------------------------------------------------------------
// dataset loaders (io.hpp:70-144)

std::string strip_cr(std::string s) {
    if (!s.empty() && s.back() == '\r') s.pop_back();
    return s;
}

std::vector<std::string> split(const std::string& line, char sep) {
    std::vector<std::string> out(1);
    for (char c : line) {
        if (c == sep) out.emplace_back();
        else out.back().push_back(c);
    }
    return out;
}

double parse_cell(const std::string& cell, size_t line, size_t col) {
    const char* b = cell.data();
    const char* e = b + cell.size();
    while (b < e && (*b == ' ' || *b == '\t')) ++b;
    while (e > b && (e[-1] == ' ' || e[-1] == '\t' || e[-1] == '\r')) --e;
    double v = 0.0;
    const auto r = std::from_chars(b, e, v);
    if (r.ec != std::errc{} || r.ptr != e)
        throw DataError("non-numeric cell \"" + cell + "\" at line " + std::to_string(line) +
                        ", column " + std::to_string(col));
    return v;
}

Dataset collection(std::vector<Series> s) {
    Dataset d;
    d.series = std::move(s);
    d.layout = JB_LAYOUT_COLLECTION;
    d.m = (int64_t)d.series.size();
    return d;
}

Dataset load_dataset(const std::string& path, const std::string& format) {
    if (format != "csv-rows" && format != "csv-cols" && format != "ts-lite")
        throw DataError("unknown data format \"" + format + "\"");
    std::ifstream in(path);
    if (!in) throw DataError("cannot open \"" + path + "\"");
    std::vector<std::string> lines;
    for (std::string line; std::getline(in, line);) {
        line = strip_cr(line);
        if (!line.empty()) lines.push_back(line);
    }
    if (lines.empty()) throw DataError("empty input");
    if (format == "csv-rows") {
        std::vector<Series> s;
        for (size_t li = 0; li < lines.size(); ++li) {
            Series ts;
            ts.id = std::to_string(li);
            const auto cells = split(lines[li], ',');
            for (size_t ci = 0; ci < cells.size(); ++ci)
                ts.values.push_back(parse_cell(cells[ci], li + 1, ci + 1));
            s.push_back(std::move(ts));
        }
        return collection(std::move(s));
    }
    if (format == "csv-cols") {
        const auto header = split(lines[0], ',');
        std::vector<Series> s(header.size());
        for (size_t c = 0; c < header.size(); ++c) s[c].id = header[c];
        for (size_t li = 1; li < lines.size(); ++li) {
            const auto cells = split(lines[li], ',');
            if (cells.size() != header.size())
                throw DataError("line " + std::to_string(li + 1) + " has " +
                                std::to_string(cells.size()) + " cells, header has " +
                                std::to_string(header.size()));
            for (size_t ci = 0; ci < cells.size(); ++ci)
                s[ci].values.push_back(parse_cell(cells[ci], li + 1, ci + 1));
        }
        return collection(std::move(s));
    }
    // ts-lite: series id, dimension id, values...
    std::map<std::string, std::vector<Series>> by;
    std::vector<std::string> order;
    for (size_t li = 0; li < lines.size(); ++li) {
        const auto cells = split(lines[li], ',');
        if (cells.size() < 3)
            throw DataError("ts-lite line " + std::to_string(li + 1) +
                            " needs: series id, dimension id, values...");
        Series dim;
        dim.id = cells[0] + "/" + cells[1];
        for (size_t ci = 2; ci < cells.size(); ++ci)
            dim.values.push_back(parse_cell(cells[ci], li + 1, ci + 1));
        if (by.find(cells[0]) == by.end()) order.push_back(cells[0]);
        by[cells[0]].push_back(std::move(dim));
    }
    if (order.size() == 1) {
        Dataset d;
        d.series = std::move(by[order.front()]);
        for (const auto& x : d.series)
            if (x.values.size() != d.series.front().values.size())
                throw DataError("ts-lite dimensions of series \"" + order.front() + "\" are ragged");
        d.layout = JB_LAYOUT_MULTIVARIATE;
        d.m = (int64_t)d.series.size();
        return d;
    }
    std::vector<Series> members;
    for (const auto& sid : order)
        for (auto& x : by[sid]) members.push_back(std::move(x));
    return collection(std::move(members));
}

void write_file(const std::string& path, const std::string& content) {
    std::ofstream out(path);
    if (!out) throw DataError("cannot write \"" + path + "\"");
    out << content;
}

std::string read_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw DataError("cannot open \"" + path + "\"");
    std::stringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

// ---------------------------------------------------------------------------
// persistence (io.hpp:160-338)

nlohmann::json codebook_json(const Codebook& cb) {
    nlohmann::json j;
    j["scaling"] = {{"scl", cb.scl}, {"sigma_len", cb.sigma_len}, {"sigma_inc", cb.sigma_inc}};
    j["digitizer_tag"] = cb.tag;
    auto& c = j["centers"] = nlohmann::json::array();
    for (const auto& p : cb.centers) c.push_back({p[0], p[1]});
    j["symbols"] = cb.symbols;
    j["mean_lengths"] = cb.mean_lengths;
    return j;
}

Codebook codebook_from(const nlohmann::json& j) {
    Codebook cb;
    cb.scl = j.at("scaling").at("scl").get<double>();
    cb.sigma_len = j.at("scaling").at("sigma_len").get<double>();
    cb.sigma_inc = j.at("scaling").at("sigma_inc").get<double>();
    cb.tag = j.at("digitizer_tag").get<std::string>();
    for (const auto& c : j.at("centers")) cb.centers.push_back({c.at(0).get<double>(), c.at(1).get<double>()});
    cb.symbols = j.at("symbols").get<std::vector<std::string>>();
    cb.mean_lengths = j.at("mean_lengths").get<std::vector<double>>();
    cb.validate();
    return cb;
}

std::string model_json(const Model& m) {
    nlohmann::json j = codebook_json(m.cb);
    j["version"] = 1;
    j["seed"] = m.seed;
    j["tol"] = m.tol;
    return j.dump(2) + "\n";
}

Model model_from(const std::string& text) {
    nlohmann::json j;
    try {
        j = nlohmann::json::parse(text);
    } catch (const nlohmann::json::parse_error& e) {
        throw DataError(std::string("model is not valid JSON: ") + e.what());
    }
    if (!j.contains("version") || !j.at("version").is_number_integer() ||
        j.at("version").get<int>() != 1)
        throw DataError("unsupported model version (expected 1)");
    Model m;
    try {
        m.cb = codebook_from(j);
        m.seed = j.value("seed", uint64_t{0});
        m.tol = j.value("tol", 0.0);
    } catch (const nlohmann::json::exception& e) {
        throw DataError(std::string("model: ") + e.what());
    }
    return m;
}

std::string symbolic_json(const Symbolic& r, const Model& m) {
    nlohmann::json j;
    j["version"] = 1;
    j["model"] = nlohmann::json::parse(model_json(m));
    j["layout"] = layout_name(r.layout);
    auto& arr = j["series"] = nlohmann::json::array();
    for (const auto& s : r.series) {
        nlohmann::json e;
        e["id"] = s.id;
        e["anchor"] = s.anchor;
        e["length"] = s.source_length;
        e["labels"] = s.labels;
        arr.push_back(std::move(e));
    }
    return j.dump(2) + "\n";
}

Symbolic symbolic_from_json(const std::string& text) {
    nlohmann::json j;
    try {
        j = nlohmann::json::parse(text);
    } catch (const nlohmann::json::parse_error& e) {
        throw DataError(std::string("symbolic result is not valid JSON: ") + e.what());
    }
    try {
        if (!j.contains("version") || j.at("version").get<int>() != 1)
            throw DataError("unsupported symbolic result version");
        Symbolic r;
        r.cb = codebook_from(j.at("model"));
        r.layout = layout_from(j.at("layout").get<std::string>());
        for (const auto& e : j.at("series")) {
            SymSeries s;
            s.id = e.at("id").get<std::string>();
            s.anchor = e.at("anchor").get<double>();
            s.source_length = e.at("length").get<int64_t>();
            s.labels = e.at("labels").get<std::vector<uint32_t>>();
            for (uint32_t l : s.labels)
                if (l >= r.cb.size())
                    throw DataError("label " + std::to_string(l) + " outside codebook");
            r.series.push_back(std::move(s));
        }
        return r;
    } catch (const nlohmann::json::exception& e) {
        throw DataError(std::string("symbolic result: ") + e.what());
    }
}

std::string symbolic_text(const Symbolic& r) {
    std::ostringstream out;
    out.precision(17);
    for (const auto& s : r.series) {
        out << s.id << '\t' << s.anchor << '\t' << s.source_length << '\t';
        for (size_t i = 0; i < s.labels.size(); ++i) {
            if (i) out << ' ';
            out << r.cb.symbols.at(s.labels[i]);
        }
        out << '\n';
    }
    return out.str();
}

Symbolic symbolic_from_text(const std::string& text, const Codebook& cb) {
    Symbolic r;
    r.cb = cb;
    r.layout = JB_LAYOUT_COLLECTION;  // the text format does not carry the layout
    std::istringstream in(text);
    size_t line_no = 0;
    for (std::string line; std::getline(in, line);) {
        ++line_no;
        line = strip_cr(line);
        if (line.empty()) continue;
        const auto f = split(line, '\t');
        if (f.size() != 4)
            throw DataError("symbols line " + std::to_string(line_no) +
                            ": expected <id>\\t<anchor>\\t<length>\\t<tokens>");
        SymSeries s;
        s.id = f[0];
        s.anchor = parse_cell(f[1], line_no, 2);
        s.source_length = (int64_t)parse_cell(f[2], line_no, 3);
        std::istringstream toks(f[3]);
        for (std::string tok; toks >> tok;) s.labels.push_back((uint32_t)cb.index_of(tok));
        r.series.push_back(std::move(s));
    }
    if (r.series.empty()) throw DataError("empty symbols file");
    return r;
}

std::string csv_rows(const std::vector<Series>& series) {  // save_series_csv_rows io.hpp:146-155
    std::ostringstream out;
    out.precision(17);
    for (const auto& ts : series) {
        for (size_t i = 0; i < ts.values.size(); ++i) {
            if (i) out << ',';
            out << ts.values[i];
        }
        out << '\n';
    }
    return out.str();
}

// ---------------------------------------------------------------------------
// the pipeline through the C ABI

struct Fit {
    Symbolic sym;
    int64_t pieces = 0, total_steps = 0;
    double ms_compress = 0.0, ms_digitize = 0.0;
    std::vector<int64_t> off, len;  // CompressedBatch: per-segment piece offsets, lengths
    std::vector<double> inc;
};

Dataset partitioned(Series ts, int64_t m) {
    Dataset d;
    d.series.push_back(std::move(ts));
    d.layout = JB_LAYOUT_UNIVARIATE_PARTITIONED;
    d.m = m;
    return d;
}

Fit fit_transform(const Dataset& ds, const jb_config& cfg) {
    if (ds.series.empty()) throw DataError("empty dataset");
    std::vector<int64_t> lengths;
    std::vector<double> values;
    for (const auto& s : ds.series) {
        lengths.push_back((int64_t)s.values.size());
        values.insert(values.end(), s.values.begin(), s.values.end());
    }
    const int64_t parts = ds.layout == JB_LAYOUT_UNIVARIATE_PARTITIONED ? ds.m : 1;
    std::vector<int64_t> first(lengths.size() * (size_t)std::max<int64_t>(parts, 1)),
        steps(first.size());
    int64_t nseg = 0;
    check(jb_plan_segments(lengths.data(), (int64_t)lengths.size(), ds.layout, parts,
                           first.data(), steps.data(), &nseg));
    jb_fit* raw = nullptr;
    check(jb_fit_transform(ctx(), values.data(), (int64_t)values.size(), 0, first.data(),
                           steps.data(), nseg, ds.layout, &cfg, &raw));
    std::unique_ptr<jb_fit, void (*)(jb_fit*)> f(raw, jb_fit_free);
    const int64_t N = jb_fit_n_pieces(raw);
    const uint64_t k = jb_fit_k(raw);
    std::vector<int64_t> off(nseg + 1), sl(nseg), plen(std::max<int64_t>(N, 1));
    std::vector<uint32_t> labels(std::max<int64_t>(N, 1));
    std::vector<double> centers(2 * k), ml(k), scaling(3), anchors(nseg), pinc(std::max<int64_t>(N, 1));
    check(jb_fit_copy_pieces(raw, off.data(), plen.data(), pinc.data()));
    check(jb_fit_copy_symbolic(raw, labels.data(), centers.data(), ml.data(), scaling.data(),
                               anchors.data(), sl.data()));
    double ph[8] = {};
    check(jb_fit_stats(raw, nullptr, nullptr, nullptr, nullptr, nullptr, ph));
    Fit out;
    out.pieces = N;
    out.off = off;
    out.len.assign(plen.begin(), plen.begin() + N);
    out.inc.assign(pinc.begin(), pinc.begin() + N);
    for (auto s : steps) out.total_steps += s;
    out.ms_compress = ph[0];
    out.ms_digitize = ph[4] - ph[0];
    Symbolic& r = out.sym;
    r.layout = ds.layout;
    r.cb.scl = scaling[0];
    r.cb.sigma_len = scaling[1];
    r.cb.sigma_inc = scaling[2];
    r.cb.tag = backend_name(cfg.backend);
    for (uint64_t g = 0; g < k; ++g) {
        r.cb.centers.push_back({centers[2 * g], centers[2 * g + 1]});
        r.cb.mean_lengths.push_back(ml[g]);
        r.cb.symbols.push_back(token(g, k));
    }
    for (int64_t s = 0; s < nseg; ++s) {
        SymSeries x;
        // ids as partitional_compress names the segments (compression.hpp:153)
        x.id = ds.layout == JB_LAYOUT_UNIVARIATE_PARTITIONED
                   ? ds.series.front().id + "[" + std::to_string(s) + "]"
                   : ds.series[s].id;
        x.anchor = anchors[s];
        x.source_length = sl[s];
        x.labels.assign(labels.begin() + off[s], labels.begin() + off[s + 1]);
        r.series.push_back(std::move(x));
    }
    return out;
}

std::vector<Series> reconstruct(const Symbolic& r) {  // reconstruct inverse.hpp:127-132
    const uint64_t k = r.cb.size();
    std::vector<double> centers, anchors;
    for (const auto& c : r.cb.centers) {
        centers.push_back(c[0]);
        centers.push_back(c[1]);
    }
    const double scaling[3] = {r.cb.scl, r.cb.sigma_len, r.cb.sigma_inc};
    std::vector<int64_t> off{0}, sl;
    std::vector<uint32_t> labels;
    for (const auto& s : r.series) {
        labels.insert(labels.end(), s.labels.begin(), s.labels.end());
        off.push_back((int64_t)labels.size());
        anchors.push_back(s.anchor);
        sl.push_back(s.source_length);
    }
    const int64_t nseg = (int64_t)r.series.size();
    const int64_t total = jb_reconstruct_size(sl.data(), nseg, r.layout);
    std::vector<double> out(std::max<int64_t>(total, 1));
    check(jb_inverse_transform(ctx(), centers.data(), r.cb.mean_lengths.data(), k, scaling,
                               labels.data(), off.data(), anchors.data(), sl.data(), nseg,
                               r.layout, out.data()));
    out.resize(total);
    std::vector<Series> res;
    if (r.layout == JB_LAYOUT_UNIVARIATE_PARTITIONED) {  // stitched (compression.hpp:198-213)
        std::string id = r.series.front().id;
        const auto b = id.find('[');
        if (b != std::string::npos) id.resize(b);
        res.push_back(Series{id, std::move(out)});
        return res;
    }
    int64_t pos = 0;
    for (const auto& s : r.series) {
        const int64_t n = s.source_length + 1;
        res.push_back(Series{s.id, std::vector<double>(out.begin() + pos, out.begin() + pos + n)});
        pos += n;
    }
    return res;
}

double mse(const std::vector<double>& a, const std::vector<double>& b) {  // metrics.hpp:18-29
    if (a.size() != b.size())
        throw DataError("mse: length mismatch (" + std::to_string(a.size()) + " vs " +
                        std::to_string(b.size()) + ")");
    if (a.empty()) throw DataError("mse: empty series");
    double out = 0.0;
    check(jb_mse(ctx(), a.data(), b.data(), (int64_t)a.size(), 0, &out));  // on the GPU, bit-exact
    return out;
}

// ---------------------------------------------------------------------------
// argument parsing: --name value | --name=value | --flag

struct Args {
    std::map<std::string, std::string> kv;
    std::vector<std::string> flags_seen;
    Args(int argc, char** argv, int from, const std::vector<std::string>& names,
         const std::vector<std::string>& flags) {
        for (int i = from; i < argc; ++i) {
            std::string a = argv[i];
            if (a.rfind("--", 0) != 0) throw UsageError("unexpected argument: " + a);
            std::string name = a, val;
            const auto eq = a.find('=');
            bool has_val = false;
            if (eq != std::string::npos) {
                name = a.substr(0, eq);
                val = a.substr(eq + 1);
                has_val = true;
            }
            const bool is_flag = std::find(flags.begin(), flags.end(), name) != flags.end();
            const bool is_opt = std::find(names.begin(), names.end(), name) != names.end();
            if (!is_flag && !is_opt) throw UsageError("unknown option: " + name);
            if (is_flag) {
                flags_seen.push_back(name);
                continue;
            }
            if (!has_val) {
                if (i + 1 >= argc) throw UsageError(name + " needs a value");
                val = argv[++i];
            }
            kv[name] = val;
        }
    }
    bool has(const std::string& n) const { return kv.count(n) > 0; }
    bool flag(const std::string& n) const {
        return std::find(flags_seen.begin(), flags_seen.end(), n) != flags_seen.end();
    }
    std::string str(const std::string& n, const std::string& d = "") const {
        auto it = kv.find(n);
        return it == kv.end() ? d : it->second;
    }
    template <class T>
    T num(const std::string& n, T d) const {
        auto it = kv.find(n);
        if (it == kv.end()) return d;
        T v{};
        const char* b = it->second.data();
        const char* e = b + it->second.size();
        const auto r = std::from_chars(b, e, v);
        if (r.ec != std::errc{} || r.ptr != e)
            throw UsageError("invalid value for " + n + ": " + it->second);
        return v;
    }
    std::string req(const std::string& n) const {
        if (!has(n)) throw UsageError(n + " is required");
        return kv.at(n);
    }
};

const char* kUsage =
    "jabba_b200 — joint symbolic aggregate approximation of time series (B200)\n"
    "usage: jabba_b200 symbolize --input F [--format csv-rows|csv-cols|ts-lite] [--tol X]\n"
    "                  [--backend vq|svq|ga|ga-auto|ga-hier] [--k N] [--alpha X] [--r X] [--scl X]\n"
    "                  [--eta X] [--partitions M] [--threads T] [--seed S] [--model-out F]\n"
    "                  [--out F] [--json]\n"
    "       jabba_b200 reconstruct --symbols F [--model F] [--out F] [--ref F] [--ref-format FMT]\n"
    "       jabba_b200 inspect --model F\n"
    "       jabba_b200 bench partition-sweep [--n N] [--tol X] [--alpha X] [--partitions 1,2,4]\n"
    "                  [--seed S] [--out F] [--json-out F]\n"
    "       jabba_b200 bench multivariate --input F [--format FMT] [--tol X] [--eta X] [--r X]\n"
    "                  [--scl X] [--seed S] [--out F] [--json-out F]\n";

// ---------------------------------------------------------------------------
// subcommands

int run_symbolize(const Args& a) {
    Dataset ds = load_dataset(a.req("--input"), a.str("--format", "csv-rows"));
    const int partitions = a.num<int>("--partitions", 0);
    if (partitions > 0) {
        if (ds.series.size() != 1)
            throw DataError("--partitions applies to single-series input only");
        ds = partitioned(std::move(ds.series.front()), partitions);
    }
    jb_config cfg;
    jb_config_default(&cfg);
    cfg.tol = a.num<double>("--tol", 0.1);
    cfg.threads = a.num<unsigned>("--threads", 1u);
    cfg.backend = backend_from(a.str("--backend", "ga"));
    cfg.scl = a.num<double>("--scl", 1.0);
    cfg.k = a.num<uint64_t>("--k", 8);
    cfg.r = a.num<double>("--r", 1.0);
    cfg.seed = a.num<uint64_t>("--seed", 0);
    cfg.alpha = a.num<double>("--alpha", 0.5);
    cfg.eta = a.num<double>("--eta", 1.0);
    const Fit f = fit_transform(ds, cfg);
    const Model model{f.sym.cb, cfg.seed, cfg.tol};
    if (a.has("--model-out")) write_file(a.str("--model-out"), model_json(model));
    const std::string payload = a.flag("--json") ? symbolic_json(f.sym, model) : symbolic_text(f.sym);
    if (a.has("--out")) write_file(a.str("--out"), payload);
    else std::cout << payload;
    const int64_t n_samples =
        f.total_steps + (f.sym.layout == JB_LAYOUT_UNIVARIATE_PARTITIONED
                             ? 1
                             : (int64_t)f.sym.series.size());
    std::cerr << "symbolized " << f.sym.series.size() << " segment(s), " << f.pieces
              << " pieces, alphabet " << f.sym.cb.size();
    if ((int64_t)f.sym.cb.size() < n_samples)  // compression_rate digitization.hpp:312-318
        std::cerr << ", tau_c " << 1.0 - (double)f.sym.cb.size() / (double)n_samples;
    std::cerr << "\n";
    return 0;
}

int run_reconstruct(const Args& a) {
    const std::string text = read_file(a.req("--symbols"));
    Symbolic sym;
    if (!text.empty() && (text.front() == '{' || text.front() == '[')) {
        sym = symbolic_from_json(text);
    } else {
        const Model m = model_from(read_file(a.str("--model")));
        sym = symbolic_from_text(text, m.cb);
    }
    const auto rec = reconstruct(sym);
    const std::string csv = csv_rows(rec);
    if (a.has("--out")) write_file(a.str("--out"), csv);
    else std::cout << csv;
    if (a.has("--ref")) {
        const Dataset ref = load_dataset(a.str("--ref"), a.str("--ref-format", "csv-rows"));
        if (ref.series.size() == rec.size()) {
            double acc = 0.0;
            for (size_t i = 0; i < rec.size(); ++i) acc += mse(ref.series[i].values, rec[i].values);
            std::cout << "mse " << acc / (double)rec.size() << "\n";
        } else {
            std::cerr << "warning: --ref has " << ref.series.size() << " series, reconstruction has "
                      << rec.size() << "; skipping MSE\n";
        }
    }
    return 0;
}

int run_inspect(const Args& a) {
    const Model m = model_from(read_file(a.req("--model")));
    const auto& cb = m.cb;
    std::cout << "digitizer: " << cb.tag << "\n"
              << "alphabet:  " << cb.size() << " symbols\n"
              << "scaling:   scl=" << cb.scl << " sigma_len=" << cb.sigma_len
              << " sigma_inc=" << cb.sigma_inc << "\n"
              << "tol:       " << m.tol << "\n"
              << "seed:      " << m.seed << "\n";
    const size_t show = std::min<size_t>(cb.size(), 10);
    for (size_t i = 0; i < show; ++i)
        std::cout << "  " << cb.symbols[i] << " -> center (" << cb.centers[i][0] << ", "
                  << cb.centers[i][1] << "), mean len " << cb.mean_lengths[i] << "\n";
    if (cb.size() > show) std::cout << "  ... " << cb.size() - show << " more\n";
    return 0;
}

// bench partition-sweep (bench.hpp:438-511): joint fits of one Gaussian noise
// series with m partitions; compression / digitization times from the GPU
// fit's phase clocks, MSE of the reconstruction on the GPU (bit-exact),
// scaled-space SSE, tau_c, and the invariants re-checked before reporting.
struct Row {  // BenchRow core.hpp:220-239
    std::string method;
    int partitions = 1, threads = 1;
    size_t symbols = 0;
    double mse = 0, sse = 0, tau_c = 1, t_compress = 0, t_digitize = 0, t_total = 0, speedup = 1;
    double dtw = std::numeric_limits<double>::quiet_NaN();  // NaN: not measured
    void validate() const {
        if (mse < 0 || sse < 0) throw DataError("bench row: negative metric");
        if (!(tau_c > 0.0 && tau_c <= 1.0)) throw DataError("bench row: tau_c outside (0,1]");
        if (!std::isnan(dtw) && dtw < 0) throw DataError("bench row: negative dtw");
    }
};

std::vector<double> gaussian_noise(size_t n, uint64_t seed) {  // bench.hpp:27-36
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> d(0.0, 1.0);
    std::vector<double> v(n);
    for (auto& x : v) x = d(rng);
    return v;
}

std::string rows_csv(const std::vector<Row>& rows) {  // BenchReport::to_csv bench.hpp:198-219
    std::ostringstream out;
    out.precision(10);
    out << "method,partitions,threads,symbols,mse,dtw,sse,tau_c,t_compress,t_digitize,t_total,"
           "speedup\n";
    for (const auto& r : rows)
    {
        out << r.method << ',' << r.partitions << ',' << r.threads << ',' << r.symbols << ','
            << r.mse << ',';
        if (!std::isnan(r.dtw)) out << r.dtw;
        out << ',' << r.sse << ',' << r.tau_c << ',' << r.t_compress << ',' << r.t_digitize
            << ',' << r.t_total << ',' << r.speedup << '\n';
    }
    return out.str();
}

std::string rows_text(const std::vector<Row>& rows) {  // BenchReport::to_text bench.hpp:221-241
    std::ostringstream out;
    out << std::left << std::setw(14) << "method" << std::right << std::setw(6) << "m"
        << std::setw(8) << "thr" << std::setw(9) << "symbols" << std::setw(13) << "mse"
        << std::setw(13) << "dtw" << std::setw(11) << "tau_c" << std::setw(12) << "t_comp"
        << std::setw(12) << "t_digit" << std::setw(9) << "phi" << '\n';
    for (const auto& r : rows) {
        out << std::left << std::setw(14) << r.method << std::right << std::setw(6) << r.partitions
            << std::setw(8) << r.threads << std::setw(9) << r.symbols << std::setw(13)
            << std::setprecision(4) << std::scientific << r.mse;
        if (std::isnan(r.dtw)) out << std::setw(13) << "-";
        else out << std::setw(13) << std::setprecision(4) << std::scientific << r.dtw;
        out << std::setw(11) << std::setprecision(5) << std::fixed << r.tau_c << std::setw(12)
            << std::setprecision(4) << std::fixed << r.t_compress << std::setw(12) << r.t_digitize
            << std::setw(9) << std::setprecision(2) << std::fixed << r.speedup << '\n';
    }
    return out.str();
}

std::string rows_json(const std::vector<Row>& rows) {  // BenchReport::to_json bench.hpp:243-261
    nlohmann::json arr = nlohmann::json::array();
    for (const auto& r : rows) {
        nlohmann::json e;
        e["method"] = r.method;
        e["partitions"] = r.partitions;
        e["threads"] = r.threads;
        e["symbols"] = r.symbols;
        e["mse"] = r.mse;
        if (!std::isnan(r.dtw)) e["dtw"] = r.dtw;
        e["sse"] = r.sse;
        e["tau_c"] = r.tau_c;
        e["t_compress"] = r.t_compress;
        e["t_digitize"] = r.t_digitize;
        e["t_total"] = r.t_total;
        e["speedup"] = r.speedup;
        arr.push_back(std::move(e));
    }
    return arr.dump(2) + "\n";
}

// scaled-space SSE of a fit from its own scaling and labels (bench.hpp:285-296)
double fit_sse(const Fit& f) {
    double acc = 0.0;
    const auto& cb = f.sym.cb;
    for (size_t s = 0; s < f.sym.series.size(); ++s)
        for (int64_t i = f.off[s]; i < f.off[s + 1]; ++i) {
            const double px = cb.scl * (double)f.len[i] / cb.sigma_len, py = f.inc[i] / cb.sigma_inc;
            const auto& c = cb.centers[f.sym.series[s].labels[i - f.off[s]]];
            const double dx = px - c[0], dy = py - c[1];
            acc += dx * dx + dy * dy;
        }
    return acc;
}

// the bench's invariants of one run (bench.hpp:112-152, 460-485): every
// piece within its compression bound (naive restatement), the global bound,
// the pinned endpoints (sum of reconstructed increments), the aggregation
// SSE bound
void check_run(const std::vector<double>& series, const Fit& f, double tol, double alpha) {
    size_t start = 0;
    double orig = 0.0, recon = 0.0;
    const auto& cb = f.sym.cb;
    for (size_t s = 0; s < f.sym.series.size(); ++s) {
        double total_dev = 0.0;
        for (int64_t i = f.off[s]; i < f.off[s + 1]; ++i) {
            const size_t end = start + (size_t)f.len[i];
            const double base = series[start], inc = series[end] - base, len = (double)f.len[i];
            double dev = 0.0;
            for (size_t q = start; q <= end; ++q) {
                const double d = base + inc * ((double)(q - start) / len) - series[q];
                dev += d * d;
            }
            const double bound = (len - 1.0) * tol * tol;
            if (dev > bound + 1e-9 * std::max(1.0, bound))
                throw DataError("bench: compression piece bound violated");
            total_dev += dev;
            orig += f.inc[i];
            recon += cb.centers[f.sym.series[s].labels[i - f.off[s]]][1] * cb.sigma_inc;
            start = end;
        }
        const double n = (double)f.sym.series[s].source_length, N = (double)(f.off[s + 1] - f.off[s]);
        const double global = (n - N) * tol * tol;
        if (total_dev > global + 1e-9 * std::max(1.0, global))
            throw DataError("bench: global compression bound violated");
    }
    if (std::abs(orig - recon) > 1e-9 * std::max({1.0, std::abs(orig), std::abs(recon)}))
        throw DataError("bench: pinned-endpoint identity violated");
    const double bound = alpha * alpha * ((double)f.pieces - (double)cb.size());
    if (fit_sse(f) > bound + 1e-9 * std::max(1.0, bound))
        throw DataError("bench: aggregation SSE bound violated");
}

int run_partition_sweep(const Args& a) {
    const size_t n = a.num<size_t>("--n", 100000);
    const double tol = a.num<double>("--tol", 0.01), alpha = a.num<double>("--alpha", 0.05);
    const uint64_t seed = a.num<uint64_t>("--seed", 42);
    std::vector<int> parts;
    for (const auto& s : split(a.str("--partitions", "1,2,4,8,16,32"), ','))
        if (!s.empty()) parts.push_back(std::stoi(s));
    Series noise{"gaussian-noise", gaussian_noise(n, seed)};
    if (noise.values.size() < 2) throw DataError("partition sweep: series too short");
    std::vector<Row> rows;
    std::map<int, double> tc;
    for (int m : parts) {
        if (m < 1) throw DataError("partition counts must be >= 1");
        jb_config cfg;
        jb_config_default(&cfg);
        cfg.tol = tol;
        cfg.backend = JB_BACKEND_GA;
        cfg.alpha = alpha;
        Fit best;
        std::vector<double> t_c, t_d;
        for (int rep = 0; rep < 3; ++rep) {  // median of 3 (bench.hpp:94-106)
            best = fit_transform(partitioned(noise, m), cfg);
            t_c.push_back(best.ms_compress * 1e-3);
            t_d.push_back(best.ms_digitize * 1e-3);
        }
        std::sort(t_c.begin(), t_c.end());
        std::sort(t_d.begin(), t_d.end());
        // re-validate the run's invariants before reporting it (bench.hpp:460-485)
        check_run(noise.values, best, tol, alpha);
        const auto rec = reconstruct(best.sym);
        Row r;
        r.method = "jabba-ga";
        r.partitions = m;
        r.threads = m;
        r.symbols = best.sym.cb.size();
        r.mse = mse(noise.values, rec.front().values);
        r.sse = fit_sse(best);
        r.tau_c = 1.0 - (double)r.symbols / (double)noise.values.size();
        r.t_compress = t_c[1];
        r.t_digitize = t_d[1];
        r.t_total = r.t_compress + r.t_digitize;
        if (!(r.tau_c > 0.0 && r.tau_c <= 1.0) || r.mse < 0)
            throw DataError("bench row: invalid metrics");
        tc[m] = r.t_compress;
        rows.push_back(r);
    }
    if (tc.count(1))  // Phi(m) on the compression phase (metrics.hpp:139-150)
        for (auto& r : rows) r.speedup = tc[1] / tc[r.partitions];
    std::cout << rows_text(rows);
    if (a.has("--out")) write_file(a.str("--out"), rows_csv(rows));
    if (a.has("--json-out")) write_file(a.str("--json-out"), rows_json(rows));
    return 0;
}

// dtw (metrics.hpp:33-50): O(n m) dynamic programming, on the host
double dtw(const std::vector<double>& x, const std::vector<double>& y) {
    if (x.empty() || y.empty()) throw DataError("dtw: empty series");
    const double inf = std::numeric_limits<double>::infinity();
    std::vector<double> prev(y.size() + 1, inf), cur(y.size() + 1, inf);
    prev[0] = 0.0;
    for (size_t i = 1; i <= x.size(); ++i) {
        cur[0] = inf;
        for (size_t j = 1; j <= y.size(); ++j) {
            const double d = x[i - 1] - y[j - 1];
            cur[j] = d * d + std::min({prev[j], cur[j - 1], prev[j - 1]});
        }
        std::swap(prev, cur);
    }
    return prev[y.size()];
}

// auto_alpha (digitization.hpp:66-75), the same expression with the host libm
double auto_alpha(int64_t n, int64_t N, double tol, double eta) {
    if (N < 1 || n <= N) throw DataError("auto_alpha: requires n > N >= 1");
    if (!(tol > 0.0)) throw DataError("auto_alpha: tol must be > 0");
    if (!(eta > 0.0)) throw DataError("auto_alpha: eta must be > 0");
    const double dn = (double)n, dN = (double)N;
    const double poly = 3.0 * dn * dn * dn * dn + 2.0 - 5.0 * dn * dn;
    const double num = 60.0 * dn * (dn - dN) * tol * tol;
    return std::pow(num / (dN * eta * eta * poly), 0.25);
}

// check_pinned_endpoints (bench.hpp:140-152): the reconstructed increments of
// a joint fit sum to the original ones
void check_pinned(const Fit& f) {
    double orig = 0.0, recon = 0.0;
    const auto& cb = f.sym.cb;
    for (size_t s = 0; s < f.sym.series.size(); ++s) {
        for (int64_t i = f.off[s]; i < f.off[s + 1]; ++i) orig += f.inc[i];
        for (uint32_t l : f.sym.series[s].labels) recon += cb.centers[l][1] * cb.sigma_inc;
    }
    if (std::abs(orig - recon) > 1e-9 * std::max({1.0, std::abs(orig), std::abs(recon)}))
        throw DataError("bench: pinned-endpoint identity violated");
}

// check_compression_bound (bench.hpp:112-138) of segment s of a fit
void check_segment_bound(const std::vector<double>& series, const Fit& f, size_t s, double tol) {
    size_t start = 0;
    double total_dev = 0.0;
    for (int64_t i = f.off[s]; i < f.off[s + 1]; ++i) {
        const size_t end = start + (size_t)f.len[i];
        const double base = series[start], inc = series[end] - base, len = (double)f.len[i];
        double dev = 0.0;
        for (size_t q = start; q <= end; ++q) {
            const double d = base + inc * ((double)(q - start) / len) - series[q];
            dev += d * d;
        }
        const double bound = (len - 1.0) * tol * tol;
        if (dev > bound + 1e-9 * std::max(1.0, bound))
            throw DataError("bench: compression piece bound violated");
        total_dev += dev;
        start = end;
    }
    const double n = (double)f.sym.series[s].source_length, N = (double)(f.off[s + 1] - f.off[s]);
    const double global = (n - N) * tol * tol;
    if (total_dev > global + 1e-9 * std::max(1.0, global))
        throw DataError("bench: global compression bound violated");
}

// bench multivariate (run_multivariate_protocol bench.hpp:297-420): a ga-auto
// joint fit fixes alpha and the symbol budget k_m; a joint sampling-VQ fit
// gets k_m symbols, per-dimension GA fits get alpha, per-dimension full VQ
// fits share k_m. Each method: symbols, MSE (GPU, bit-exact) and DTW (host)
// of the reconstruction per dimension, scaled-space SSE, tau_c; times are
// medians of 3 runs from the GPU fits' phase clocks.
int run_multivariate(const Args& a) {
    Dataset ds = load_dataset(a.req("--input"), a.str("--format", "ts-lite"));
    if (ds.layout == JB_LAYOUT_COLLECTION) {  // promote an equal-length collection (csv-cols)
        for (const auto& x : ds.series)
            if (x.values.size() != ds.series.front().values.size())
                throw DataError("multivariate dataset: dimensions must have equal length");
        ds.layout = JB_LAYOUT_MULTIVARIATE;
        ds.m = (int64_t)ds.series.size();
    }
    if (ds.layout != JB_LAYOUT_MULTIVARIATE)
        throw DataError("multivariate protocol needs a multivariate dataset");
    const size_t d = ds.series.size();
    if (d == 0) throw DataError("empty dataset");
    const double tol = a.num<double>("--tol", 0.01), eta = a.num<double>("--eta", 1.0);
    const double r_opt = a.num<double>("--r", 0.5), scl = a.num<double>("--scl", 1.0);
    const uint64_t seed = a.num<uint64_t>("--seed", 0);
    const uint64_t max_iters = 300;
    int64_t total_samples = 0;
    for (const auto& x : ds.series) total_samples += (int64_t)x.values.size();

    auto base_cfg = [&](int32_t backend) {
        jb_config c;
        jb_config_default(&c);
        c.tol = tol;
        c.backend = backend;
        c.scl = scl;
        return c;
    };
    struct Timed {
        std::vector<Fit> fits;  // one joint fit, or one per dimension
        double t_compress = 0.0, t_digitize = 0.0;
    };
    // median of 3 runs (median_runtime bench.hpp:94-106) of a list of fits
    auto timed = [&](const std::vector<std::pair<Dataset, jb_config>>& runs) {
        Timed t;
        std::vector<double> tc, td;
        for (int rep = 0; rep < 3; ++rep) {
            std::vector<Fit> fits;
            double c = 0.0, g = 0.0;
            for (const auto& [dd, cfg] : runs) {
                fits.push_back(fit_transform(dd, cfg));
                c += fits.back().ms_compress * 1e-3;
                g += fits.back().ms_digitize * 1e-3;
            }
            tc.push_back(c);
            td.push_back(g);
            t.fits = std::move(fits);
        }
        std::sort(tc.begin(), tc.end());
        std::sort(td.begin(), td.end());
        t.t_compress = tc[1];
        t.t_digitize = td[1];
        return t;
    };

    // 1) joint GA with auto alpha fixes the budget
    jb_config ga_cfg = base_cfg(JB_BACKEND_GA_AUTO);
    ga_cfg.eta = eta;
    const Timed joint_ga = timed({{ds, ga_cfg}});
    const Fit& jg = joint_ga.fits.front();
    for (size_t i = 0; i < d; ++i) check_segment_bound(ds.series[i].values, jg, i, tol);
    check_pinned(jg);
    const double alpha = auto_alpha(jg.total_steps, jg.pieces, tol, eta);
    const uint64_t k_m = jg.sym.cb.size();

    // 2) joint VQ (sampling k-means) with the same symbol count; the sample
    // must still hold at least k_m points
    jb_config vq_cfg = base_cfg(JB_BACKEND_SVQ);
    vq_cfg.k = k_m;
    vq_cfg.r = std::min(1.0, std::max(r_opt, ((double)k_m + 1.0) / (double)jg.pieces));
    vq_cfg.seed = seed;
    vq_cfg.max_iters = max_iters;
    const Timed joint_vq = timed({{ds, vq_cfg}});
    check_pinned(joint_vq.fits.front());

    // 3) per-dimension GA with the same alpha; 4) per-dimension VQ sharing
    // k_m (the first k_m % d dimensions get the extra center)
    std::vector<std::pair<Dataset, jb_config>> pga, pvq;
    for (size_t i = 0; i < d; ++i) {
        const Dataset one = collection({ds.series[i]});
        jb_config g = base_cfg(JB_BACKEND_GA);
        g.alpha = alpha;
        pga.emplace_back(one, g);
        jb_config v = base_cfg(JB_BACKEND_VQ);
        uint64_t k = std::max<uint64_t>(1, k_m / d + (i < k_m % d ? 1 : 0));
        k = std::min<uint64_t>(k, (uint64_t)(jg.off[i + 1] - jg.off[i]));
        v.k = k;
        v.seed = seed;
        v.max_iters = max_iters;
        pvq.emplace_back(one, v);
    }
    const Timed per_ga = timed(pga);
    const Timed per_vq = timed(pvq);

    // the compression phase alone: the joint GA runs' compression clocks
    const double t_compress = joint_ga.t_compress;
    std::vector<Row> rows;
    auto evaluate = [&](const std::string& method, const Timed& t) {
        std::vector<std::vector<double>> recons;
        double sse = 0.0;
        size_t symbols = 0;
        for (const auto& f : t.fits) {
            symbols += f.sym.cb.size();
            for (auto& x : reconstruct(f.sym)) recons.push_back(std::move(x.values));
            sse += fit_sse(f);
        }
        Row r;
        r.method = method;
        r.partitions = (int)d;
        r.threads = 1;
        r.symbols = symbols;
        r.t_compress = t_compress;
        r.t_digitize = t.t_digitize;
        r.t_total = r.t_compress + r.t_digitize;
        double mse_acc = 0.0, dtw_acc = 0.0;
        for (size_t i = 0; i < d; ++i) {
            mse_acc += mse(ds.series[i].values, recons[i]);
            dtw_acc += dtw(ds.series[i].values, recons[i]);
        }
        r.mse = mse_acc / (double)d;
        r.dtw = dtw_acc / (double)d;
        r.sse = sse;
        if ((int64_t)symbols >= total_samples) throw DataError("bench: alphabet larger than the dataset");
        r.tau_c = 1.0 - (double)symbols / (double)total_samples;
        r.validate();
        rows.push_back(r);
    };
    evaluate("abba-vq", per_vq);
    evaluate("fabba-ga", per_ga);
    evaluate("jabba-vq", joint_vq);
    evaluate("jabba-ga", joint_ga);
    std::cout << rows_text(rows);
    if (a.has("--out")) write_file(a.str("--out"), rows_csv(rows));
    if (a.has("--json-out")) write_file(a.str("--json-out"), rows_json(rows));
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        if (argc < 2) throw UsageError("a subcommand is required");
        const std::string cmd = argv[1];
        if (cmd == "-h" || cmd == "--help") {
            std::cout << kUsage;
            return 0;
        }
        if (cmd == "symbolize")
            return run_symbolize(Args(argc, argv, 2,
                                      {"--input", "--format", "--tol", "--backend", "--k", "--alpha",
                                       "--r", "--scl", "--eta", "--partitions", "--threads",
                                       "--seed", "--model-out", "--out"},
                                      {"--json"}));
        if (cmd == "reconstruct")
            return run_reconstruct(Args(argc, argv, 2,
                                        {"--model", "--symbols", "--out", "--ref", "--ref-format"},
                                        {}));
        if (cmd == "inspect") return run_inspect(Args(argc, argv, 2, {"--model"}, {}));
        if (cmd == "bench") {
            const std::string proto = argc >= 3 ? argv[2] : "";
            if (proto == "partition-sweep")
                return run_partition_sweep(Args(argc, argv, 3,
                                                {"--n", "--tol", "--alpha", "--partitions",
                                                 "--seed", "--out", "--json-out"},
                                                {}));
            if (proto == "multivariate")
                return run_multivariate(Args(argc, argv, 3,
                                             {"--input", "--format", "--tol", "--eta", "--r",
                                              "--scl", "--seed", "--out", "--json-out"},
                                             {}));
            throw UsageError("bench needs a protocol: partition-sweep | multivariate");
        }
        throw UsageError("unknown subcommand: " + cmd);
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << "\n" << kUsage;
        return 2;
    } catch (const DataError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
