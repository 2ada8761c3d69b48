// Runs the reference's experiment layer (run_compare / run_stepsize_sweep and their CSV / ME
// writers, proj/src/experiment.cpp) on a config file.  Built twice by tests/cpp/Makefile:
// against the reference library (compare_ref) and against the B200 library (compare_b200,
// experiment.cpp compiled unchanged against tests/cpp/compat), so the two output
// directories can be compared byte for byte (tests/test_gpu_dropin.py).
//
// usage: compare_* CONFIG OUTDIR [sweep DT1,DT2,...]
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "spde2d/experiment.hpp"

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s CONFIG OUTDIR [sweep DT1,DT2,...]\n", argv[0]);
        return 2;
    }
    std::ifstream in(argv[1]);
    std::stringstream text;
    text << in.rdbuf();
    try {
        spde2d::ExperimentConfig cfg = spde2d::parse_config_text(text.str());
        cfg.out = argv[2];
        if (argc >= 5 && std::string(argv[3]) == "sweep") {
            std::vector<double> dts;
            std::stringstream list(argv[4]);
            for (std::string tok; std::getline(list, tok, ',');) dts.push_back(std::strtod(tok.c_str(), nullptr));
            spde2d::run_stepsize_sweep(cfg, dts);
        } else {
            spde2d::run_compare(cfg);
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
