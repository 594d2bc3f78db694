"""Generate tests/golden/io/: model JSON, symbolic-result JSON and the
tab-separated symbols text written by the UNMODIFIED reference (io.hpp
model_to_json / symbolic_to_json / symbolic_to_text after jabba_fit) for a
few seeded inputs. Needs /root/reference (this container only); the files are
committed and tests/test_io_persistence.py compares the Python mirror
(paper_2401_00109_b200/io.py) against them byte for byte.

    python tests/golden/make_io_golden.py
"""
import os
import subprocess
import tempfile

REF = "/root/reference/proj/include"
JSON_INC = ("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/"
            "thirdparty/nlohmann")
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io")

SRC = r"""
#include <cstdio>
#include <fstream>
#include <random>
#include "jabba/jabba.hpp"
using namespace jabba;

static TimeSeries walk(std::uint64_t seed, std::size_t n, const std::string& id) {
    std::mt19937_64 g(seed);
    std::normal_distribution<double> nd(0.0, 1.0);
    TimeSeries ts;
    ts.id = id;
    double x = 0.0;
    for (std::size_t t = 0; t < n; ++t) { ts.values.push_back(x); x += nd(g); }
    return ts;
}

static void emit(const std::string& dir, const std::string& name, const Dataset& ds,
                 JabbaConfig cfg) {
    const JabbaFit fit = jabba_fit(ds, cfg);
    Model m;
    m.codebook = fit.symbolic.codebook;
    m.seed = cfg.digitize.vq.seed;
    m.tol = cfg.compression.tol;
    std::ofstream(dir + "/" + name + ".model.json") << model_to_json(m);
    std::ofstream(dir + "/" + name + ".symbolic.json") << symbolic_to_json(fit.symbolic, m);
    std::ofstream(dir + "/" + name + ".symbols.txt") << symbolic_to_text(fit.symbolic);
}

int main(int argc, char** argv) {
    const std::string dir = argv[1];
    {   // sampled k-means on a partitioned walk: 1-char tokens incl. escapes
        JabbaConfig cfg;
        cfg.compression.tol = 0.05;
        cfg.digitize.backend = Backend::sampling_vq;
        cfg.digitize.vq.k = 90; cfg.digitize.vq.r = 0.6; cfg.digitize.vq.seed = 7;
        emit(dir, "walk_svq_k90", Dataset::partitioned(walk(11, 6000, "w"), 3), cfg);
    }
    {   // greedy aggregation on a collection
        JabbaConfig cfg;
        cfg.compression.tol = 0.2;
        cfg.digitize.backend = Backend::ga;
        cfg.digitize.ga.alpha = 0.3;
        std::vector<TimeSeries> ms = {walk(1, 900, "a"), walk(2, 700, "b"), walk(3, 800, "c")};
        emit(dir, "collection_ga", Dataset::collection(ms), cfg);
    }
    {   // more than 94 symbols: "#rank" tokens; vq
        JabbaConfig cfg;
        cfg.compression.tol = 0.01;
        cfg.digitize.backend = Backend::vq;
        cfg.digitize.vq.k = 120; cfg.digitize.vq.seed = 3;
        emit(dir, "walk_vq_k120", Dataset::partitioned(walk(5, 4000, "v"), 1), cfg);
    }
    return 0;
}
"""


def main():
    os.makedirs(OUT, exist_ok=True)
    with tempfile.TemporaryDirectory() as t:
        c, exe = os.path.join(t, "g.cpp"), os.path.join(t, "g")
        with open(c, "w") as f:
            f.write(SRC)
        subprocess.run(["g++", "-std=c++20", "-O2", f"-I{REF}", f"-I{JSON_INC}", "-o", exe, c,
                        "-lpthread"], check=True)
        subprocess.run([exe, OUT], check=True)
    print("\n".join(sorted(os.listdir(OUT))))


if __name__ == "__main__":
    main()
