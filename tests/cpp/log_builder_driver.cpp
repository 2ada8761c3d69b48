// MagnusLogBuilder parity driver (host only): builds the union pattern of a CommutatorSet and
// fills it for a few functionals at every order the builder allows, then writes the raw
// row_ptr / col_idx / values bytes to the file given as argv[1].  Compiled once against the
// reference library and once against the B200 library's host half (tests/cpp/Makefile);
// tests/test_host.py compares the two files byte for byte.
#include <cmath>
#include <cstdio>
#include <vector>

#include "spde2d/magnus.hpp"
#include "spde2d/operators.hpp"

using namespace spde2d;

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    std::FILE* out = std::fopen(argv[1], "wb");
    if (!out) return 2;
    const double fs[3][5] = {{0.1, -0.56, -0.0169, -0.00126, 0.0054},
                             {0.01, 0.0, 0.0, 0.0, 0.0},
                             {0.05, 0.031, 1.3e-3, -2.5e-5, 4.0e-5}};
    for (int fam = 0; fam < 3; ++fam) {
        for (std::size_t d : {7, 16, 33}) {
            const GridSpec g{build_grid(-4.0, 4.0, d), build_grid(-4.0, 4.0, d + (fam == 2 ? 3 : 0))};
            CoefficientFamily family = fam == 0 ? CoefficientFamily::langevin_constant(1.1, 0.3)
                                     : fam == 1 ? CoefficientFamily::langevin_variable(1.1, 0.3)
                                                : CoefficientFamily::custom(CoefficientEvaluators{
                                                      [](double x, double v) { return 0.2 * std::cos(x + v); },
                                                      [](double, double v) { return -v; },
                                                      [](double x, double) { return 0.3 * std::sin(x); },
                                                      [](double, double v) { return 0.05 * (1.0 + v * v / 16.0); },
                                                      [](double x, double v) { return 0.02 * std::sin(x * v); },
                                                      [](double x, double) { return 1.1 + 0.1 * std::cos(x); },
                                                      [](double, double v) { return 0.1 * std::cos(v); },
                                                      [](double x, double) { return 0.05 * std::sin(x); },
                                                      [](double x, double) { return 0.3 + 0.01 * x * x; }});
            const CoefficientFields f = sample_coefficients(family, g);
            const CommutatorSet comms = precompute_commutators(assemble_diffusion(f, g), assemble_drift(f, g), 3);
            for (int bo = 1; bo <= 3; ++bo) {
                const MagnusLogBuilder b(comms, bo);
                const std::size_t head[2] = {b.dim(), b.nnz()};
                std::fwrite(head, sizeof(head), 1, out);
                std::vector<double> vals;
                for (int o = 1; o <= bo; ++o)
                    for (const auto& q : fs) {
                        const ItoFunctionals itf{q[0], q[1], q[2], q[3], q[4]};
                        b.fill(o, itf, vals);
                        const SparseView v = b.view_with(vals);
                        std::fwrite(v.row_ptr.data(), sizeof(std::size_t), v.row_ptr.size(), out);
                        std::fwrite(v.col_idx.data(), sizeof(std::int32_t), v.col_idx.size(), out);
                        std::fwrite(v.values.data(), sizeof(double), v.values.size(), out);
                    }
            }
        }
    }
    std::fclose(out);
    return 0;
}
