// ref_cli.cpp — TEST INFRASTRUCTURE ONLY. The reference CLI's symbolize /
// reconstruct / inspect pipelines (proj/tools/jabba_cli.cpp:51-148) driven
// through the UNMODIFIED reference headers, with a hand-written flag parser
// because CLI11 is absent offline. tests/test_cli.py runs it next to the
// product CLI (paper_2401_00109_b200/jabba_b200) on the same files.
#include <cstdint>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>

#include "jabba/bench.hpp"
#include "jabba/jabba.hpp"

namespace {

std::map<std::string, std::string> parse(int argc, char** argv, bool& json) {
    std::map<std::string, std::string> kv;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        if (a == "--json") {
            json = true;
        } else if (i + 1 < argc) {
            kv[a] = argv[++i];
        }
    }
    return kv;
}

std::string get(const std::map<std::string, std::string>& kv, const std::string& k,
                const std::string& d) {
    const auto it = kv.find(k);
    return it == kv.end() ? d : it->second;
}

void put(const std::string& path, const std::string& s) {
    std::ofstream out(path);
    out << s;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string cmd = argv[1];
    bool json = false;
    const auto kv = parse(argc, argv, json);
    try {
        if (cmd == "symbolize") {
            jabba::Dataset ds = jabba::load_dataset(
                get(kv, "--input", ""), jabba::data_format_from_string(get(kv, "--format", "csv-rows")));
            const int m = std::stoi(get(kv, "--partitions", "0"));
            if (m > 0) ds = jabba::Dataset::partitioned(ds.series.front(), (std::size_t)m);
            jabba::JabbaConfig cfg;
            cfg.compression.tol = std::stod(get(kv, "--tol", "0.1"));
            cfg.digitize.backend = jabba::backend_from_string(get(kv, "--backend", "ga"));
            cfg.digitize.scl = std::stod(get(kv, "--scl", "1"));
            cfg.digitize.vq.k = std::stoull(get(kv, "--k", "8"));
            cfg.digitize.vq.r = std::stod(get(kv, "--r", "1"));
            cfg.digitize.vq.seed = std::stoull(get(kv, "--seed", "0"));
            cfg.digitize.ga.alpha = std::stod(get(kv, "--alpha", "0.5"));
            cfg.digitize.auto_digitize.eta = std::stod(get(kv, "--eta", "1"));
            const jabba::JabbaFit fit = jabba::jabba_fit(ds, cfg);
            const jabba::Model model{fit.symbolic.codebook, cfg.digitize.vq.seed,
                                     cfg.compression.tol};
            if (kv.count("--model-out")) jabba::save_model(kv.at("--model-out"), model);
            const std::string out = json ? jabba::symbolic_to_json(fit.symbolic, model)
                                         : jabba::symbolic_to_text(fit.symbolic);
            if (kv.count("--out")) put(kv.at("--out"), out);
            else std::cout << out;
            return 0;
        }
        if (cmd == "bench-multivariate") {  // run_multivariate_protocol (bench.hpp:297-420)
            jabba::Dataset ds = jabba::load_dataset(
                get(kv, "--input", ""), jabba::data_format_from_string(get(kv, "--format", "ts-lite")));
            if (ds.layout == jabba::Layout::collection)
                ds = jabba::Dataset::multivariate(std::move(ds.series));
            jabba::MultivariateOptions opt;
            opt.eta = std::stod(get(kv, "--eta", "1"));
            opt.sampling_r = std::stod(get(kv, "--r", "0.5"));
            opt.scl = std::stod(get(kv, "--scl", "1"));
            opt.seed = std::stoull(get(kv, "--seed", "0"));
            const jabba::BenchReport report =
                jabba::run_multivariate_protocol(ds, std::stod(get(kv, "--tol", "0.01")), opt);
            if (kv.count("--json-out")) put(kv.at("--json-out"), report.to_json());
            std::cout << report.to_text();
            return 0;
        }
        if (cmd == "reconstruct") {
            std::ifstream in(get(kv, "--symbols", ""));
            std::stringstream ss;
            ss << in.rdbuf();
            const std::string text = ss.str();
            jabba::SymbolicResult sym;
            if (!text.empty() && (text.front() == '{' || text.front() == '[')) {
                sym = jabba::symbolic_from_json(text).first;
            } else {
                const jabba::Model model = jabba::load_model(get(kv, "--model", ""));
                sym = jabba::symbolic_from_text(text, model.codebook);
            }
            std::ostringstream out;
            jabba::save_series_csv_rows(out, jabba::reconstruct(sym));
            if (kv.count("--out")) put(kv.at("--out"), out.str());
            else std::cout << out.str();
            return 0;
        }
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
    return 2;
}
