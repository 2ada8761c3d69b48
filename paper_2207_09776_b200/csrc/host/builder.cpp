// Host-kept half of the drop-in: grid, CSR algebra, coefficient sampling,
// operator assembly, commutators and the xoshiro Brownian batch.
//
// These stay on the CPU (north star: "the host stays C++ and keeps ... grid and
// coefficient setup, the FD operator builder").  Their outputs are what the GPU
// consumes, and parity demands the operator VALUES be bitwise the reference's,
// so every floating-point expression below performs the same roundings in the
// same order as the reference routine cited beside it (compiled with
// -ffp-contract=off, no FMA).  The sparse layer (CsrBuilder, merge_rows, the
// MagnusLogBuilder union) is structured our own way; the coefficient families,
// assemble_*, precompute_commutators, the xoshiro256++/splitmix64 stream and the
// path functionals necessarily follow the reference's term order and error
// messages closely, since both are part of the bitwise / API contract.
#include <algorithm>
#include <cmath>
#include <limits>
#include <numbers>
#include <ostream>
#include <cstdio>
#include <string>

#include "spde2d_b200.hpp"

namespace spde2d {

// ---- grid.cpp:8-40 ------------------------------------------------------------
Grid1D build_grid(double a, double b, std::size_t n) {
    if (!(b > a)) throw ConfigError("build_grid: need b > a");
    if (n == 0) throw ConfigError("build_grid: need at least one interior node");
    Grid1D g;
    g.a = a;
    g.b = b;
    g.n = n;
    g.delta = (b - a) / static_cast<double>(n + 1);
    return g;
}

bool Field::all_zero() const {
    for (double x : v_)
        if (x != 0.0) return false;
    return true;
}

std::vector<double> vectorize(const Field& f) { return {f.data().begin(), f.data().end()}; }

Field devectorize(std::span<const double> vec, std::size_t nx, std::size_t nv) {
    if (vec.size() != nx * nv) throw DimensionError("devectorize: length mismatch");
    Field f(nx, nv);
    std::copy(vec.begin(), vec.end(), f.data().begin());
    return f;
}

// ---- sparse.cpp:25-363 ----------------------------------------------------------
SparseMatrix::SparseMatrix(std::size_t rows, std::size_t cols, std::vector<std::size_t> rp,
                           std::vector<std::int32_t> ci, std::vector<double> v)
    : rows_(rows), cols_(cols), rp_(std::move(rp)), ci_(std::move(ci)), val_(std::move(v)) {}

namespace {

// Incremental CSR writer: append entries row by row, dropping exact zeros
// (the reference prunes every exact zero it produces).
struct CsrBuilder {
    std::size_t rows, cols;
    std::vector<std::size_t> rp;
    std::vector<std::int32_t> ci;
    std::vector<double> v;
    CsrBuilder(std::size_t r, std::size_t c, std::size_t reserve = 0) : rows(r), cols(c) {
        rp.reserve(r + 1);
        rp.push_back(0);
        ci.reserve(reserve);
        v.reserve(reserve);
    }
    void put(std::size_t col, double val) {
        if (val != 0.0) {
            ci.push_back(static_cast<std::int32_t>(col));
            v.push_back(val);
        }
    }
    void end_row() { rp.push_back(ci.size()); }
    SparseMatrix done() { return SparseMatrix(rows, cols, std::move(rp), std::move(ci), std::move(v)); }
};

void same_shape(const SparseMatrix& a, const SparseMatrix& b, const char* what) {
    if (a.rows() != b.rows() || a.cols() != b.cols())
        throw DimensionError(std::string(what) + ": shape mismatch");
}

// Row-wise merge of two sorted CSR rows; absent entries enter as 0.0 (sparse.cpp:297-338).
template <class Op>
SparseMatrix merge_rows(const SparseMatrix& a, const SparseMatrix& b, Op op) {
    CsrBuilder out(a.rows(), a.cols(), a.nnz() + b.nnz());
    const auto arp = a.row_ptr(), brp = b.row_ptr();
    const auto aci = a.col_idx(), bci = b.col_idx();
    const auto av = a.values(), bv = b.values();
    for (std::size_t r = 0; r < a.rows(); ++r) {
        std::size_t p = arp[r], q = brp[r];
        const std::size_t pe = arp[r + 1], qe = brp[r + 1];
        while (p < pe || q < qe) {
            const bool take_a = q >= qe || (p < pe && aci[p] < bci[q]);
            const bool take_b = p >= pe || (q < qe && bci[q] < aci[p]);
            if (take_a) {
                out.put(aci[p], op(av[p], 0.0));
                ++p;
            } else if (take_b) {
                out.put(bci[q], op(0.0, bv[q]));
                ++q;
            } else {
                out.put(aci[p], op(av[p], bv[q]));
                ++p;
                ++q;
            }
        }
        out.end_row();
    }
    return out.done();
}

} // namespace

SparseMatrix SparseMatrix::from_triplets(std::size_t rows, std::size_t cols,
                                         std::vector<Triplet> t) {
    std::sort(t.begin(), t.end(), [](const Triplet& x, const Triplet& y) {
        return x.row != y.row ? x.row < y.row : x.col < y.col;
    });
    CsrBuilder out(rows, cols, t.size());
    std::size_t i = 0;
    for (std::size_t r = 0; r < rows; ++r) {
        while (i < t.size() && t[i].row == r) {
            const std::size_t c = t[i].col;
            if (c >= cols) throw DimensionError("from_triplets: column out of range");
            double s = t[i++].value;
            while (i < t.size() && t[i].row == r && t[i].col == c) s += t[i++].value;
            out.put(c, s);
        }
        out.end_row();
    }
    if (i != t.size()) throw DimensionError("from_triplets: row out of range");
    return out.done();
}

SparseMatrix SparseMatrix::identity(std::size_t n) {
    CsrBuilder out(n, n, n);
    for (std::size_t r = 0; r < n; ++r) {
        out.put(r, 1.0);
        out.end_row();
    }
    return out.done();
}

SparseMatrix SparseMatrix::zero(std::size_t rows, std::size_t cols) {
    return SparseMatrix(rows, cols, std::vector<std::size_t>(rows + 1, 0), {}, {});
}

std::size_t SparseMatrix::nonzero_diagonals() const {
    if (rows_ == 0 && cols_ == 0) return 0;
    std::vector<std::int64_t> offs;
    offs.reserve(val_.size());
    for (std::size_t r = 0; r < rows_; ++r)
        for (std::size_t k = rp_[r]; k < rp_[r + 1]; ++k)
            offs.push_back(static_cast<std::int64_t>(ci_[k]) - static_cast<std::int64_t>(r));
    std::sort(offs.begin(), offs.end());
    return static_cast<std::size_t>(std::unique(offs.begin(), offs.end()) - offs.begin());
}

SparseMatrix tridiag(std::size_t n, double lo, double mid, double hi, double scale) {
    if (n == 0) throw ConfigError("tridiag: n must be positive");
    const double w[3] = {lo * scale, mid * scale, hi * scale}; // sparse.cpp:100-102
    CsrBuilder out(n, n, 3 * n);
    for (std::size_t r = 0; r < n; ++r) {
        if (r > 0) out.put(r - 1, w[0]);
        out.put(r, w[1]);
        if (r + 1 < n) out.put(r + 1, w[2]);
        out.end_row();
    }
    return out.done();
}

SparseMatrix kron(const SparseMatrix& a, const SparseMatrix& b) {
    const std::size_t rows = a.rows() * b.rows(), cols = a.cols() * b.cols();
    if ((a.rows() && rows / a.rows() != b.rows()) || (a.cols() && cols / a.cols() != b.cols()))
        throw DimensionError("kron: dimension overflow");
    if (cols > static_cast<std::size_t>(std::numeric_limits<std::int32_t>::max()))
        throw DimensionError("kron: column dimension exceeds index range");
    CsrBuilder out(rows, cols, a.nnz() * b.nnz());
    const auto arp = a.row_ptr(), brp = b.row_ptr();
    const auto aci = a.col_idx(), bci = b.col_idx();
    const auto av = a.values(), bv = b.values();
    for (std::size_t ra = 0; ra < a.rows(); ++ra)
        for (std::size_t rb = 0; rb < b.rows(); ++rb) {
            for (std::size_t p = arp[ra]; p < arp[ra + 1]; ++p) {
                const std::size_t base = static_cast<std::size_t>(aci[p]) * b.cols();
                for (std::size_t q = brp[rb]; q < brp[rb + 1]; ++q)
                    out.put(base + static_cast<std::size_t>(bci[q]), av[p] * bv[q]);
            }
            out.end_row();
        }
    return out.done();
}

SparseMatrix diag_of(std::span<const double> v) {
    CsrBuilder out(v.size(), v.size(), v.size());
    for (std::size_t r = 0; r < v.size(); ++r) {
        out.put(r, v[r]);
        out.end_row();
    }
    return out.done();
}

SparseMatrix spmm(const SparseMatrix& a, const SparseMatrix& b) {
    if (a.cols() != b.rows()) throw DimensionError("spmm: inner dimensions disagree");
    const auto arp = a.row_ptr(), brp = b.row_ptr();
    const auto aci = a.col_idx(), bci = b.col_idx();
    const auto av = a.values(), bv = b.values();
    std::vector<double> acc(b.cols(), 0.0);
    std::vector<std::int32_t> stamp(b.cols(), -1); // row that last touched a column
    std::vector<std::int32_t> cols;
    CsrBuilder out(a.rows(), b.cols());
    for (std::size_t r = 0; r < a.rows(); ++r) {
        cols.clear();
        // accumulate in (a-entry, b-entry) order, sparse.cpp:210-222
        for (std::size_t p = arp[r]; p < arp[r + 1]; ++p) {
            const std::size_t k = static_cast<std::size_t>(aci[p]);
            for (std::size_t q = brp[k]; q < brp[k + 1]; ++q) {
                const std::int32_t c = bci[q];
                if (stamp[c] != static_cast<std::int32_t>(r)) {
                    stamp[c] = static_cast<std::int32_t>(r);
                    acc[c] = 0.0;
                    cols.push_back(c);
                }
                acc[c] += av[p] * bv[q];
            }
        }
        std::sort(cols.begin(), cols.end());
        for (std::int32_t c : cols) out.put(static_cast<std::size_t>(c), acc[c]);
        out.end_row();
    }
    return out.done();
}

void spmv(const SparseView& a, std::span<const double> x, std::span<double> y) {
    if (x.size() != a.cols || y.size() != a.rows) throw DimensionError("spmv: length mismatch");
    for (std::size_t r = 0; r < a.rows; ++r) {
        double s = 0.0;
        for (std::size_t k = a.row_ptr[r]; k < a.row_ptr[r + 1]; ++k)
            s += a.values[k] * x[static_cast<std::size_t>(a.col_idx[k])];
        y[r] = s;
    }
}

std::vector<double> spmv(const SparseMatrix& a, std::span<const double> x) {
    std::vector<double> y(a.rows());
    spmv(a.view(), x, y);
    return y;
}

SparseMatrix sparse_add(const SparseMatrix& a, const SparseMatrix& b) {
    same_shape(a, b, "sparse_add");
    return merge_rows(a, b, [](double x, double y) { return x + y; });
}

SparseMatrix sparse_sub(const SparseMatrix& a, const SparseMatrix& b) {
    same_shape(a, b, "sparse_sub");
    return merge_rows(a, b, [](double x, double y) { return x - y; });
}

SparseMatrix sparse_scale(const SparseMatrix& a, double s) {
    CsrBuilder out(a.rows(), a.cols(), a.nnz());
    const auto rp = a.row_ptr();
    const auto ci = a.col_idx();
    const auto v = a.values();
    for (std::size_t r = 0; r < a.rows(); ++r) {
        for (std::size_t k = rp[r]; k < rp[r + 1]; ++k) out.put(ci[k], v[k] * s);
        out.end_row();
    }
    return out.done();
}

SparseMatrix commutator(const SparseMatrix& a, const SparseMatrix& b) {
    if (a.rows() != a.cols() || b.rows() != b.cols())
        throw DimensionError("commutator: matrices must be square");
    same_shape(a, b, "commutator");
    return sparse_sub(spmm(a, b), spmm(b, a));
}

double one_norm(const SparseView& m) {
    std::vector<double> colsum(m.cols, 0.0);
    for (std::size_t k = 0; k < m.values.size(); ++k)
        colsum[static_cast<std::size_t>(m.col_idx[k])] += std::abs(m.values[k]);
    double best = 0.0;
    for (double s : colsum) best = std::max(best, s);
    return best;
}

// ---- operators.cpp:8-208 ------------------------------------------------------
void CoefficientFields::refresh_zero_flags() {
    zero_h = h.all_zero();
    zero_fx = fx.all_zero();
    zero_fv = fv.all_zero();
    zero_gxx = gxx.all_zero();
    zero_gxv = gxv.all_zero();
    zero_gvv = gvv.all_zero();
    zero_sig = sig.all_zero();
    zero_sigx = sigx.all_zero();
    zero_sigv = sigv.all_zero();
}

namespace {
void check_langevin(const char* name, double a, double sigma) {
    if (!(a > 0.0) || sigma < 0.0 || !(a - sigma * sigma > 0.0))
        throw ConfigError(std::string(name) + " requires a > 0 and a - sigma^2 > 0");
}
} // namespace

CoefficientFamily CoefficientFamily::langevin_constant(double a, double sigma) {
    check_langevin("langevin-constant", a, sigma);
    CoefficientEvaluators e;
    e.fx = [](double, double v) { return -v; };
    e.gvv = [a](double, double) { return a; };
    e.sigv = [sigma](double, double) { return sigma; };
    return CoefficientFamily(FamilyTag::LangevinConstant, a, sigma, std::move(e));
}

CoefficientFamily CoefficientFamily::langevin_variable(double a, double sigma) {
    check_langevin("langevin-variable", a, sigma);
    CoefficientEvaluators e;
    e.fx = [](double, double v) { return -v; };
    e.gvv = [a](double x, double) { return a * (1.0 + 1.0 / (x * x + 1.0)); };
    e.sigv = [sigma](double x, double) { return sigma * std::sqrt(1.0 + 1.0 / (x * x + 1.0)); };
    return CoefficientFamily(FamilyTag::LangevinVariable, a, sigma, std::move(e));
}

CoefficientFamily CoefficientFamily::custom(CoefficientEvaluators evals) {
    return CoefficientFamily(FamilyTag::Custom, 0.0, 0.0, std::move(evals));
}

CoefficientFields sample_coefficients(const CoefficientFamily& family, const GridSpec& grid) {
    const auto& e = family.evaluators();
    auto sample = [&](const CoefficientEvaluators::Fn& fn) {
        Field f(grid.x.n, grid.v.n);
        if (!fn) return f;
        for (std::size_t j = 0; j < grid.v.n; ++j)
            for (std::size_t i = 0; i < grid.x.n; ++i) f(i, j) = fn(grid.x.node(i), grid.v.node(j));
        return f;
    };
    CoefficientFields f;
    f.h = sample(e.h);
    f.fx = sample(e.fx);
    f.fv = sample(e.fv);
    f.gxx = sample(e.gxx);
    f.gxv = sample(e.gxv);
    f.gvv = sample(e.gvv);
    f.sig = sample(e.sig);
    f.sigx = sample(e.sigx);
    f.sigv = sample(e.sigv);
    f.refresh_zero_flags();
    if (family.tag() != FamilyTag::Custom) {
        for (std::size_t k = 0; k < f.gvv.size(); ++k) {
            const double s = f.sigv.data()[k];
            if (!(f.gvv.data()[k] - s * s > 0.0))
                throw ConfigError("coefficient positivity violated: g^vv - (sigma^v)^2 <= 0");
        }
    }
    return f;
}

namespace {

void check_fields(const CoefficientFields& f, const GridSpec& g) {
    for (const Field* x : {&f.h, &f.fx, &f.fv, &f.gxx, &f.gxv, &f.gvv, &f.sig, &f.sigx, &f.sigv})
        if (x->nx() != g.x.n || x->nv() != g.v.n)
            throw DimensionError("coefficient field shape does not match the grid");
}

// diag(vec z) * k as a row scaling (operators.cpp:105-130).
SparseMatrix scale_rows(const Field& z, const SparseMatrix& k) {
    CsrBuilder out(k.rows(), k.cols(), k.nnz());
    const auto rp = k.row_ptr();
    const auto ci = k.col_idx();
    const auto v = k.values();
    const auto zv = z.data();
    for (std::size_t r = 0; r < k.rows(); ++r) {
        if (zv[r] != 0.0)
            for (std::size_t e = rp[r]; e < rp[r + 1]; ++e) out.put(ci[e], zv[r] * v[e]);
        out.end_row();
    }
    return out.done();
}

SparseMatrix d1(std::size_t n, double delta) { return tridiag(n, -1.0, 0.0, 1.0, 1.0 / (2.0 * delta)); }
SparseMatrix d2(std::size_t n, double delta) {
    return tridiag(n, 1.0, -2.0, 1.0, 1.0 / (delta * delta));
}

} // namespace

SparseMatrix assemble_drift(const CoefficientFields& f, const GridSpec& g) {
    check_fields(f, g);
    const std::size_t nx = g.x.n, nv = g.v.n;
    const SparseMatrix ix = SparseMatrix::identity(nx), iv = SparseMatrix::identity(nv);
    SparseMatrix b = SparseMatrix::zero(nx * nv, nx * nv);
    // term order and the late 1/2 scaling follow operators.cpp:141-167
    if (!f.zero_h) b = sparse_add(b, diag_of(f.h.data()));
    if (!f.zero_fx) b = sparse_add(b, scale_rows(f.fx, kron(iv, d1(nx, g.x.delta))));
    if (!f.zero_fv) b = sparse_add(b, scale_rows(f.fv, kron(d1(nv, g.v.delta), ix)));
    if (!f.zero_gxx)
        b = sparse_add(b, sparse_scale(scale_rows(f.gxx, kron(iv, d2(nx, g.x.delta))), 0.5));
    if (!f.zero_gxv)
        b = sparse_add(b, scale_rows(f.gxv, kron(d1(nv, g.v.delta), d1(nx, g.x.delta))));
    if (!f.zero_gvv)
        b = sparse_add(b, sparse_scale(scale_rows(f.gvv, kron(d2(nv, g.v.delta), ix)), 0.5));
    return b;
}

SparseMatrix assemble_diffusion(const CoefficientFields& f, const GridSpec& g) {
    check_fields(f, g);
    const std::size_t nx = g.x.n, nv = g.v.n;
    SparseMatrix a = SparseMatrix::zero(nx * nv, nx * nv);
    if (!f.zero_sig) a = sparse_add(a, diag_of(f.sig.data()));
    if (!f.zero_sigx)
        a = sparse_add(a, scale_rows(f.sigx, kron(SparseMatrix::identity(nv), d1(nx, g.x.delta))));
    if (!f.zero_sigv)
        a = sparse_add(a, scale_rows(f.sigv, kron(d1(nv, g.v.delta), SparseMatrix::identity(nx))));
    return a;
}

CommutatorSet precompute_commutators(const SparseMatrix& a, const SparseMatrix& b, int order) {
    if (order < 1 || order > 3) throw ConfigError("commutator order must be in {1, 2, 3}");
    CommutatorSet s;
    s.order = order;
    s.A = a;
    s.B = b;
    if (order >= 2) {
        s.A2 = spmm(a, a);
        s.BA = commutator(b, a); // [B,A] = BA - AB (operators.cpp:201)
    }
    if (order >= 3) {
        s.BAA = commutator(s.BA, a);
        s.BAB = commutator(s.BA, b);
    }
    return s;
}

// ---- stochastics.cpp:13-141 ----------------------------------------------------
namespace {
std::uint64_t splitmix(std::uint64_t& x) {
    std::uint64_t z = (x += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
inline std::uint64_t rotl64(std::uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

std::size_t exact_ratio(double total, double step, const char* what) {
    if (!(step > 0.0)) throw ConfigError(std::string(what) + ": step must be positive");
    if (!(total > 0.0)) throw ConfigError(std::string(what) + ": horizon must be positive");
    const auto k = static_cast<std::int64_t>(std::llround(total / step));
    if (k < 1 || std::abs(total - static_cast<double>(k) * step) >
                     1e-12 * std::max(1.0, std::abs(total)))
        throw ConfigError(std::string(what) + ": horizon is not an integer multiple of the step");
    return static_cast<std::size_t>(k);
}
} // namespace

NormalStream::NormalStream(std::uint64_t seed, std::uint64_t trajectory) {
    std::uint64_t mix = seed;
    (void)splitmix(mix);
    mix ^= (trajectory + 1) * 0xD1B54A32D192ED03ULL;
    for (auto& s : s_) s = splitmix(mix);
}

std::uint64_t NormalStream::next_u64() {
    const std::uint64_t out = rotl64(s_[0] + s_[3], 23) + s_[0];
    const std::uint64_t t = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= t;
    s_[3] = rotl64(s_[3], 45);
    return out;
}

double NormalStream::next() {
    if (has_cached_) {
        has_cached_ = false;
        return cached_;
    }
    const double u1 = (static_cast<double>(next_u64() >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = static_cast<double>(next_u64() >> 11) * 0x1.0p-53;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double ang = 2.0 * std::numbers::pi * u2;
    cached_ = r * std::sin(ang);
    has_cached_ = true;
    return r * std::cos(ang);
}

// ---- text output used by the reference's experiment layer ---------------------------
// dump_path (stochastics.cpp:229-237): one "t value" line per Lebesgue index.
void dump_path(const BrownianBatch& batch, std::size_t m, std::ostream& os) {
    if (m >= batch.M) throw ConfigError("dump_path: trajectory index out of range");
    char line[96];
    for (std::size_t k = 0; k <= batch.steps; ++k) {
        std::snprintf(line, sizeof line, "%.12g %.17g\n", static_cast<double>(k) * batch.dt_leb, batch.values[m][k]);
        os << line;
    }
}

// write_triplets (sparse.cpp:352-363): "row col value" per stored entry, CSR order.
void write_triplets(const SparseMatrix& m, std::ostream& os) {
    const auto rp = m.row_ptr();
    const auto ci = m.col_idx();
    const auto v = m.values();
    char line[96];
    for (std::size_t r = 0; r < m.rows(); ++r)
        for (std::size_t q = rp[r]; q < rp[r + 1]; ++q) {
            std::snprintf(line, sizeof line, "%zu %d %.17g\n", r, ci[q], v[q]);
            os << line;
        }
}

BrownianBatch simulate_brownian(double T, double dt_leb, std::size_t M, std::uint64_t seed) {
    if (M == 0) throw ConfigError("simulate_brownian: need at least one trajectory");
    BrownianBatch b;
    b.T = T;
    b.dt_leb = dt_leb;
    b.M = M;
    b.seed = seed;
    b.steps = exact_ratio(T, dt_leb, "simulate_brownian");
    const double scale = std::sqrt(dt_leb);
    b.increments.assign(M, std::vector<double>(b.steps));
    b.values.assign(M, std::vector<double>(b.steps + 1));
    for (std::size_t m = 0; m < M; ++m) {
        NormalStream rng(seed, m);
        auto& inc = b.increments[m];
        auto& val = b.values[m];
        val[0] = 0.0;
        for (std::size_t k = 0; k < b.steps; ++k) {
            inc[k] = scale * rng.next();
            val[k + 1] = val[k] + inc[k];
        }
    }
    return b;
}

std::size_t BrownianBatch::index_of(double t) const {
    const auto k = static_cast<std::int64_t>(std::llround(t / dt_leb));
    if (k < 0 || static_cast<std::size_t>(k) > steps ||
        std::abs(t - static_cast<double>(k) * dt_leb) > 1e-12 * std::max(1.0, std::abs(t)))
        throw ConfigError("time " + std::to_string(t) + " is not on the Lebesgue grid");
    return static_cast<std::size_t>(k);
}

PathSegment window(const BrownianBatch& batch, double t0, double t1, std::size_t m) {
    if (m >= batch.M) throw ConfigError("window: trajectory index out of range");
    const std::size_t k0 = batch.index_of(t0), k1 = batch.index_of(t1);
    if (k0 >= k1) throw ConfigError("window: need t0 < t1 on the grid");
    return PathSegment{&batch.values[m], k0, k1, batch.dt_leb};
}

ItoFunctionals lebesgue_functionals(const PathSegment& seg) {
    if (seg.steps() == 0) throw ConfigError("lebesgue_functionals: empty segment");
    const auto& p = *seg.path;
    const double base = p[seg.k0], dt = seg.dt_leb;
    double iw = 0.0, isw = 0.0, iw2 = 0.0;
    for (std::size_t j = 0; j < seg.steps(); ++j) {
        const double w = p[seg.k0 + j] - base;
        const double s = static_cast<double>(j) * dt;
        iw += w;
        isw += s * w;
        iw2 += w * w;
    }
    ItoFunctionals f;
    f.h = seg.length();
    f.W = seg.terminal();
    f.IW = iw * dt;
    f.IsW = isw * dt;
    f.IW2 = iw2 * dt;
    return f;
}

// ---- Ito identity residuals (stochastics.cpp:143-227), test oracles ---------------
namespace {
double pw(double x, int k) {
    double r = 1.0;
    for (int i = 0; i < k; ++i) r *= x;
    return r;
}
} // namespace

double ito_identity_residual(ItoIdentity id, const ItoExponents& e, const PathSegment& seg) {
    if (e.p < 0 || e.p1 < 0 || e.p2 < 0 || e.q < 0 || e.q1 < 0 || e.q2 < 0)
        throw ConfigError("ito_identity_residual: exponents must be non-negative");
    const std::size_t n = seg.steps();
    if (n == 0) throw ConfigError("ito_identity_residual: empty segment");
    const auto& p = *seg.path;
    const double base = p[seg.k0], dt = seg.dt_leb, t = seg.length(), wt = seg.terminal();
    auto W = [&](std::size_t j) { return p[seg.k0 + j] - base; };
    auto dW = [&](std::size_t j) { return p[seg.k0 + j + 1] - p[seg.k0 + j]; };
    if (id == ItoIdentity::A) {
        // int s^p W^q dW = (t^p W_t^{q+1} - int [q(q+1)/2 s^p W^{q-1} + p W^{q+1} s^{p-1}] ds)/(q+1)
        double lhs = 0.0, rem = 0.0;
        const double cq = 0.5 * e.q * (e.q + 1);
        for (std::size_t j = 0; j < n; ++j) {
            const double s = static_cast<double>(j) * dt, w = W(j);
            lhs += pw(s, e.p) * pw(w, e.q) * dW(j);
            double g = 0.0;
            if (e.q > 0) g += cq * pw(s, e.p) * pw(w, e.q - 1);
            if (e.p > 0) g += e.p * pw(w, e.q + 1) * pw(s, e.p - 1);
            rem += g;
        }
        return lhs - (pw(t, e.p) * pw(wt, e.q + 1) - rem * dt) / (e.q + 1);
    }
    if (id == ItoIdentity::B) {
        // int s^{p1} (int r^{p2} W^q dr) ds = (t^{1+p1} int s^{p2} W^q - int s^{1+p1+p2} W^q)/(1+p1)
        double lhs = 0.0, inner = 0.0, i1 = 0.0, i2 = 0.0;
        for (std::size_t j = 0; j < n; ++j) {
            const double s = static_cast<double>(j) * dt, w = W(j);
            lhs += pw(s, e.p1) * inner;
            inner += pw(s, e.p2) * pw(w, e.q) * dt;
            i1 += pw(s, e.p2) * pw(w, e.q);
            i2 += pw(s, 1 + e.p1 + e.p2) * pw(w, e.q);
        }
        lhs *= dt;
        return lhs - (pw(t, 1 + e.p1) * i1 * dt - i2 * dt) / (1 + e.p1);
    }
    // C: int s^{p1} W^{q1} (int r^{p2} W^{q2} dr) dW with three Lebesgue remainders
    double lhs = 0.0, inner = 0.0, i1 = 0.0, i2 = 0.0, i3 = 0.0, i4 = 0.0;
    const double cq = 0.5 * e.q1 * (e.q1 + 1);
    for (std::size_t j = 0; j < n; ++j) {
        const double s = static_cast<double>(j) * dt, w = W(j);
        lhs += pw(s, e.p1) * pw(w, e.q1) * inner * dW(j);
        i1 += pw(s, e.p2) * pw(w, e.q2);
        i2 += pw(s, e.p1 + e.p2) * pw(w, e.q1 + e.q2 + 1);
        if (e.q1 > 0) i3 += pw(s, e.p1) * pw(w, e.q1 - 1) * inner;
        if (e.p1 > 0) i4 += pw(s, e.p1 - 1) * pw(w, e.q1 + 1) * inner;
        inner += pw(s, e.p2) * pw(w, e.q2) * dt;
    }
    double rhs = pw(t, e.p1) * pw(wt, e.q1 + 1) * i1 * dt - i2 * dt;
    if (e.q1 > 0) rhs -= cq * i3 * dt;
    if (e.p1 > 0) rhs -= e.p1 * i4 * dt;
    return lhs - rhs / (e.q1 + 1);
}

// ---- magnus_log (magnus.cpp:26-40, 63-82): the logarithm as an explicit CSR ------------
SparseMatrix magnus_log(int order, const CommutatorSet& comms, const ItoFunctionals& f) {
    if (order < 1 || order > 3) throw ConfigError("magnus_log: order must be in {1, 2, 3}");
    if (order > comms.order) throw ConfigError("magnus_log: commutator set does not cover this order");
    const double h = f.h;
    SparseMatrix y = sparse_add(sparse_scale(comms.B, h), sparse_scale(comms.A, f.W));
    if (order >= 2) {
        y = sparse_add(y, sparse_scale(comms.A2, -0.5 * h));
        y = sparse_add(y, sparse_scale(comms.BA, f.IW - 0.5 * h * f.W));
    }
    if (order >= 3) {
        y = sparse_add(y, sparse_scale(comms.BAA, 0.5 * f.IW2 - 0.5 * f.W * f.IW + h * f.W * f.W / 12.0));
        y = sparse_add(y, sparse_scale(comms.BAB, f.IsW - 0.5 * h * f.IW - h * h * f.W / 12.0));
    }
    return y;
}

// ---- MagnusLogBuilder (magnus.hpp:61-86, magnus.cpp:88-164) ------------------------------
namespace {
int first_order_of(int slot) { return slot < 2 ? 1 : (slot < 4 ? 2 : 3); }

// log_coefficients (magnus.cpp:26-40): weights of B, A, A2, [B,A], [[B,A],A], [[B,A],B]
void log_weights(int order, const ItoFunctionals& f, double c[6]) {
    const double h = f.h;
    c[0] = h;
    c[1] = f.W;
    c[2] = order >= 2 ? -0.5 * h : 0.0;
    c[3] = order >= 2 ? f.IW - 0.5 * h * f.W : 0.0;
    c[4] = order >= 3 ? 0.5 * f.IW2 - 0.5 * f.W * f.IW + h * f.W * f.W / 12.0 : 0.0;
    c[5] = order >= 3 ? f.IsW - 0.5 * h * f.IW - h * h * f.W / 12.0 : 0.0;
}
} // namespace

MagnusLogBuilder::MagnusLogBuilder(const CommutatorSet& comms, int order) : order_(order) {
    if (order < 1 || order > 3 || order > comms.order) throw ConfigError("MagnusLogBuilder: unsupported order");
    rows_ = comms.B.rows();
    const SparseMatrix* by_slot[6] = {&comms.B, &comms.A, &comms.A2, &comms.BA, &comms.BAA, &comms.BAB};
    for (int slot = 0; slot < 6; ++slot) {
        if (first_order_of(slot) > order) continue;
        if (by_slot[slot]->rows() != rows_) throw DimensionError("MagnusLogBuilder: source dimension mismatch");
        Part p;
        p.slot = slot;
        p.matrix = by_slot[slot];
        p.to_union.resize(p.matrix->nnz());
        parts_.push_back(std::move(p));
    }
    // per row: every (column, part, entry) of the participating sources, ordered by column;
    // each distinct column is one union entry, and every source entry learns its position
    struct Hit {
        std::int32_t col;
        std::uint32_t part;
        std::size_t entry;
    };
    std::vector<Hit> hits;
    row_start_.assign(rows_ + 1, 0);
    for (std::size_t r = 0; r < rows_; ++r) {
        hits.clear();
        for (std::uint32_t q = 0; q < parts_.size(); ++q) {
            const auto rp = parts_[q].matrix->row_ptr();
            const auto ci = parts_[q].matrix->col_idx();
            for (std::size_t k = rp[r]; k < rp[r + 1]; ++k) hits.push_back(Hit{ci[k], q, k});
        }
        std::sort(hits.begin(), hits.end(), [](const Hit& a, const Hit& b) { return a.col < b.col; });
        for (std::size_t h = 0; h < hits.size(); ++h) {
            if (h == 0 || hits[h].col != hits[h - 1].col) cols_.push_back(hits[h].col);
            parts_[hits[h].part].to_union[hits[h].entry] = cols_.size() - 1;
        }
        row_start_[r + 1] = cols_.size();
    }
}

void MagnusLogBuilder::fill(int order, const ItoFunctionals& f, std::vector<double>& values) const {
    if (order < 1 || order > order_) throw ConfigError("MagnusLogBuilder::fill: order exceeds builder order");
    double c[6];
    log_weights(order, f, c);
    values.assign(cols_.size(), 0.0);
    for (const Part& p : parts_) { // slot order: every union entry folds its sources in that order
        if (first_order_of(p.slot) > order) continue;
        const double coef = c[p.slot];
        if (coef == 0.0) continue;
        const auto w = p.matrix->values();
        for (std::size_t k = 0; k < w.size(); ++k) values[p.to_union[k]] += coef * w[k];
    }
}

SparseView MagnusLogBuilder::view_with(std::span<const double> values) const {
    return SparseView{rows_, rows_, row_start_, cols_, values};
}

// ---- EulerStencils::from_grid (euler.cpp:18-26) ----------------------------------------
EulerStencils EulerStencils::from_grid(const GridSpec& grid) {
    const double dx = grid.x.delta, dv = grid.v.delta;
    EulerStencils st;
    st.inv2dx = 1.0 / (2.0 * dx);
    st.invdx2 = 1.0 / (dx * dx);
    st.inv2dv = 1.0 / (2.0 * dv);
    st.invdv2 = 1.0 / (dv * dv);
    st.inv4dxdv = 1.0 / (4.0 * dx * dv);
    return st;
}

// ---- gamma0 (exact_langevin.cpp:20-27) --------------------------------------------
double gamma0(double t, double x, double v, const LangevinParams& p) {
    if (!(p.a > 0.0) || p.sigma < 0.0 || !(p.gap() > 0.0))
        throw ConfigError("exact Langevin solution needs a > 0 and a - sigma^2 > 0");
    if (!(t > 0.0)) throw ConfigError("gamma0: t must be positive");
    const double c = p.gap();
    const double quad = v * v / t - 3.0 * v * x / (t * t) + 3.0 * x * x / (t * t * t);
    return std::numbers::sqrt3 / (std::numbers::pi * t * t * c) * std::exp(-(2.0 / c) * quad);
}

std::size_t SolutionEnsemble::blowup_count() const {
    return static_cast<std::size_t>(std::count(status.begin(), status.end(), TrajectoryStatus::BlownUp));
}

// ---- exact_langevin.cpp:29-39 / analysis.cpp:9-31 (host-side setup pieces) ----------
Field gaussian_datum(const GridSpec& g) {
    Field f(g.x.n, g.v.n);
    for (std::size_t j = 0; j < g.v.n; ++j) {
        const double v = g.v.node(j);
        for (std::size_t i = 0; i < g.x.n; ++i) {
            const double x = g.x.node(i);
            f(i, j) = std::exp(-(x * x + v * v) / 2.0);
        }
    }
    return f;
}

CentralRegion central_region(std::size_t d, int kappa) {
    if (d < 2) throw ConfigError("central_region: need d >= 2");
    if (kappa < 0) throw ConfigError("central_region: kappa must be non-negative");
    if (kappa >= 63 || (std::size_t{1} << kappa) > d)
        throw ConfigError("central_region: empty region, kappa too large");
    const double half = static_cast<double>(d) / 2.0;
    const double width = static_cast<double>(d) / std::pow(2.0, kappa + 1);
    const auto lo1 = static_cast<std::int64_t>(std::floor(half - width));
    const auto hi1 = static_cast<std::int64_t>(std::floor(half + width));
    CentralRegion r;
    r.d = d;
    r.kappa = kappa;
    r.lo = static_cast<std::size_t>(std::max<std::int64_t>(lo1 - 1, 0));
    r.hi = static_cast<std::size_t>(std::min<std::int64_t>(hi1 - 1, static_cast<std::int64_t>(d) - 1));
    if (r.hi < r.lo) throw ConfigError("central_region: empty region");
    return r;
}

double avg_mean_abs_error(const Field& me) {
    double s = 0.0;
    for (double v : me.data()) s += v;
    return me.size() ? s / static_cast<double>(me.size()) : 0.0;
}

} // namespace spde2d
