// Shared by the Magnus pass-engine translation units (magnus.cu, term_nt*.cu).
#pragma once

#include <algorithm>
#include <cstdint>
#include <initializer_list>
#include <utility>

#include "s2b_internal.cuh"

namespace s2b {
namespace mg {

constexpr int kMaxTerms = 55;   // sparse.cpp:435
constexpr int kStripRows = 128; // output rows per work item (term_tma_kernel; 32 measured 10% slower)
constexpr int kStages = 8;      // TMA ring depth (power of two)

__host__ __device__ constexpr int box_bit(int dx, int dv) { return (dv + kBoxR) * kBoxW + (dx + kBoxR); }

__device__ __forceinline__ int xclass(int i, int nx) {
    return i == 0 ? 0 : (i == 1 ? 1 : (i == nx - 2 ? 3 : (i == nx - 1 ? 4 : 2)));
}

// |v| as bits, cleared on the high word (one integer LOP3: the 64-bit mask form is otherwise
// recognised as fabs and issued as a DADD on the fp64 pipe)
__device__ __forceinline__ unsigned long long abs_bits(double v) {
    const unsigned hi = static_cast<unsigned>(__double2hiint(v)) & 0x7fffffffu;
    const unsigned lo = static_cast<unsigned>(__double2loint(v));
    return (static_cast<unsigned long long>(hi) << 32) | lo;
}
constexpr unsigned long long kInfBits = 0x7FF0000000000000ULL;

__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) {
    return a > b ? a : b;
}

__device__ __forceinline__ unsigned long long warp_umax(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = umax64(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

struct OpView {
    const int* pair_begin; // kBoxBits + 1
    const int* pair_slot;
    const double* w;
    int nx, nv;
    int compressed;
    const double* wpm = nullptr; // uncompressed weights point-major [row][x][npairs | 1] (term_var)
};

struct TermArgs {
    OpView op;
    const double* ctab; // [M][nwin][6]
    int nwin;
    const int* act;
    const int* cnt; // cnt[0] = live paths this pass
    const int* win;
    const int* k;
    const int* nseg;
    const int* par;
    double* T0;
    double* T1;
    double* S0;
    double* S1;
    unsigned long long* tn;
    unsigned long long* sn;
    int nstrips;
    int strip_rows; // output rows per work item of term_tma_kernel (kStripRows; S2B_STRIP overrides)
    int sync_g;     // term_tma_kernel: one CTA barrier per sync_g ring steps (1, 2, 4; S2B_TMA_SYNC)
    int8_t e2bit[kBoxBits];
    // entry-major weights of the kernel's mask: wt[(j * NYE + q) * kPairSlots + k] is the
    // k-th source weight (slot order) of Y entry q = cls * NBM + e at row j, zero-padded;
    // eslot[q * kPairSlots + k] is its CommutatorSet slot, -1 for padding.
    const double* wt;
    const int* eslot;
};
constexpr int kPairSlots = 6;
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// Variants taking precomputed shared-window addresses (no per-call address conversion).
__device__ __forceinline__ void mbar_expect_tx_u(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_u(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_u(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_row_u(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tma_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <uint64_t MASK>
struct MaskInfo {
    static constexpr int count() {
        int n = 0;
        for (int b = 0; b < kBoxBits; ++b) n += (MASK >> b) & 1;
        return n;
    }
    static constexpr int rank(int bit) {
        int n = 0;
        for (int b = 0; b < bit; ++b) n += (MASK >> b) & 1;
        return n;
    }
    static constexpr bool has(int dx, int dv) { return (MASK >> box_bit(dx, dv)) & 1; }
    static constexpr int bit_of(int e) { // the e-th set bit
        for (int b = 0; b < kBoxBits; ++b)
            if ((MASK >> b) & 1) {
                if (e == 0) return b;
                --e;
            }
        return -1;
    }
};

// One work item = (live path, strip of kStripRows output rows).  Threads own two adjacent
// x-points (i = 2t, 2t+1).  Rows stream through a kStages-deep TMA ring (stage s carries
// input row j0-KRV+s and accum row j0-2KRV+s); each thread keeps a (2KRV+1)-row register
// window of its x-neighbourhood.  The Y values of the next output row (5 x-classes x the
// mask's stencil points) are folded from the compressed weights one step ahead, by the
// threads that own those entries, into a double-buffered shared row.  Warps without an
// x-boundary point read one Y set for both of their points.
constexpr uint64_t mask_of(std::initializer_list<std::pair<int, int>> pts) {
    uint64_t m = 0;
    for (auto [dx, dv] : pts) m |= 1ULL << box_bit(dx, dv);
    return m;
}
constexpr uint64_t box_mask(int rx, int rv) {
    uint64_t m = 0;
    for (int dv = -rv; dv <= rv; ++dv)
        for (int dx = -rx; dx <= rx; ++dx) m |= 1ULL << box_bit(dx, dv);
    return m;
}
// Union stencils of the Langevin families: orders 1, 2, 3.
constexpr uint64_t kMask5 = mask_of({{0, 0}, {-1, 0}, {1, 0}, {0, -1}, {0, 1}});
constexpr uint64_t kMask11 = kMask5 | mask_of({{0, -2}, {0, 2}, {-1, -1}, {1, -1}, {-1, 1}, {1, 1}});
constexpr uint64_t kMask19 =
    kMask11 | mask_of({{-1, -2}, {1, -2}, {-1, 2}, {1, 2}, {-2, -1}, {2, -1}, {-2, 1}, {2, 1}});
constexpr uint64_t kBox22 = box_mask(2, 2);
constexpr uint64_t kBox23 = box_mask(2, 3);
constexpr uint64_t kBox33 = box_mask(3, 3);

// bm: stencil entries (mask rank e) whose Y may differ on an x-boundary class at an in-grid
// offset; the boundary warp loads those per lane and broadcasts the interior value for the
// rest (bm == 0: boundary points use the interior Y outright).
struct Variant {
    uint64_t mask;
    int rx, rv;
    uint32_t bm;
};
constexpr uint32_t kBmAll = 0xFFFFFFFFu;
// constant Langevin order 3: only (dx, dv) = (0, -1), (0, +1) differ at i = 0 and nx-1
constexpr uint32_t kBm19c = (1u << MaskInfo<kMask19>::rank(box_bit(0, -1))) |
                            (1u << MaskInfo<kMask19>::rank(box_bit(0, 1)));
constexpr Variant kVariants[] = {
    {0, 0, 0, 0},             // 0: generic
    {kMask5, 1, 1, kBmAll},   // 1
    {kMask11, 1, 2, kBmAll},  // 2
    {kMask19, 2, 2, kBmAll},  // 3
    {kBox22, 2, 2, kBmAll},   // 4
    {kBox23, 2, 3, kBmAll},   // 5
    {kBox33, 3, 3, kBmAll},   // 6
    {kMask5, 1, 1, 0},        // 7: Langevin order 1
    {kMask11, 1, 2, 0},       // 8: Langevin order 2
    {kMask19, 2, 2, kBm19c},  // 9: Langevin order 3 (constant coefficients)
};
constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);

// Block-size classes: (max threads, min resident blocks) -> register budget.
int tma_popcount(int variant);
constexpr size_t kTermSmem = 226 * 1024; // dynamic shared memory of term_tma_kernel (opt-in maximum less its static part)
size_t tma_smem_fixed(int variant, size_t nx);
size_t tma_strip_cap(int variant, size_t nx);
// term_tma_kernel launchers, one translation unit per block-size class
void launch_term_nt128(s2b_context* ctx, int variant, const TermArgs& a, int nt, size_t smem, size_t work);
void launch_term_nt256(s2b_context* ctx, int variant, const TermArgs& a, int nt, size_t smem, size_t work);
void launch_term_nt512(s2b_context* ctx, int variant, const TermArgs& a, int nt, size_t smem, size_t work);

// Two Taylor terms per pass (term2_kernel.cuh): the extra state of the two-term engine
struct Term2Args {
    double* S2;              // third accumulator buffer
    int* tpar;               // per path: which T buffer holds t_{k-1}
    unsigned long long* tn2; // running max |t_{k+1}| (bits)
    unsigned long long* sn2; // running max |s_{k+1}| (bits)
};
void launch_term2_nt128(s2b_context* ctx, int variant, const TermArgs& a, const Term2Args& b, int nt, size_t smem,
                        size_t work);
void launch_term2_nt256(s2b_context* ctx, int variant, const TermArgs& a, const Term2Args& b, int nt, size_t smem,
                        size_t work);
void launch_term2_nt512(s2b_context* ctx, int variant, const TermArgs& a, const Term2Args& b, int nt, size_t smem,
                        size_t work);

// Streaming term kernel for uncompressed (x-dependent) weights with a Langevin union mask
// (term_var.cu); S2B_TERMVAR=0 falls back to term_generic_k_kernel.
bool term_var_supported(const s2b_operator* op);
void launch_term_var(s2b_context* ctx, const s2b_operator* op, const TermArgs& a, size_t live_max);

// Cluster-resident engine (cluster_magnus.cu): one 8-CTA cluster per path, all Taylor terms
// of windows [win0, win1) on chip.
struct ClusterArgs {
    const double* wt;  // entry-major weights of the variant (as TermArgs::wt)
    const int* eslot;
    int nx, nv;
    const double* ctab; // [M][nwin][6]
    const int* stab;    // [M][nwin]
    int nwin, win0, win1, dt_steps;
    double* S0;
    double* S1;
    int* par;
    int* status;
    int* win;
    int* rec_next;
    long long* terms;
    long long* windows;
    long long* segments;
    double* const* rec; // R-1 record buffers
    uint8_t* rec_status;
    const long long* rec_steps;
    int R;
    double tol, cap;
    int M;
    int* work; // path counter (zeroed before the launch)
    double* sx; // accumulator scratch of the in-place engine: [slots][CL][nx][rows] (x-major)
    int sx_slots;
    int nz; // the datum holds no -0.0 (shortened stencil folds are then bit-identical)
};
// Several sessions (e.g. a step-size sweep on shared paths) in ONE persistent launch: the
// clusters draw virtual path ids from one counter (a[0].work); ids [prefix[s], prefix[s+1])
// belong to session s.  The x-march engines support n > 1; the row-band one n == 1.
constexpr int kMaxBatch = 8;
struct ClusterBatch {
    ClusterArgs a[kMaxBatch];
    int prefix[kMaxBatch + 1];
    int n;
    int total;
};
bool cluster_engine_supported(int variant, int nx, int nv);
bool cluster_batch_supported(int variant, int nx, int nv); // n > 1 allowed
void launch_cluster_magnus(s2b_context* ctx, int variant, const ClusterBatch& b);
// x-march variant of the cluster engine (cluster_xm.cu); S2B_XM=0 disables it
bool cluster_xm_supported(int variant, int nx, int nv);
void launch_cluster_xm(s2b_context* ctx, int variant, const ClusterBatch& b);
// in-place x-march with the accumulator in L2 (cluster_xmi.cu): 16-CTA clusters at 512^2;
// S2B_XMI=0 disables it.  sx_doubles: scratch the session must pass in ClusterArgs::sx.
bool cluster_xmi_supported(int variant, int nx, int nv);
size_t cluster_xmi_scratch(int nx, int nv, int* slots);
void launch_cluster_xmi(s2b_context* ctx, int variant, const ClusterBatch& b);

// Streaming x-march engine (term_xs.cu): the compressed Langevin stencils on grids no cluster
// holds (nx >= 256, multiples of 128 x 32).  While it runs, a session's term and accumulator
// vectors are x-major ([path][x][v]); S2B_XS=0 disables it.
bool term_xs_supported(const s2b_operator* op);
size_t term_xs_y_doubles(const s2b_operator* op, size_t M);
void launch_term_xs(s2b_context* ctx, const s2b_operator* op, const TermArgs& a, const int* seg, double* Yg,
                    int4* meta4, size_t M, bool nz);
void xs_transpose_paths(s2b_context* ctx, const double* S0, const double* S1, double* T0, double* T1,
                        const int* par, size_t M, int R, int C);
void xs_transpose_paths_inplace(s2b_context* ctx, double* S0, double* S1, const int* par, size_t p_lo, size_t M,
                                int d);
bool term_xs_slice_supported(const s2b_operator* op);
void xs_records(s2b_context* ctx, const int* cnt, const int4* recq, const double* S0, const double* S1,
                const double* S2, double* const* rec, int nx, int nv, size_t M);
// two Taylor terms per pass (term_xs2_kernel, term2's buffer protocol; default, S2B_XS2=0 disables)
bool term_xs2_enabled();
void launch_term_xs2(s2b_context* ctx, const s2b_operator* op, const TermArgs& a, const Term2Args& b, const int* seg,
                     double* Yg, int4* meta4, size_t M, bool nz);

} // namespace mg
} // namespace s2b
