// term2_kernel instantiations (the Langevin stencils, variants 7-9) for blocks of up to 128 threads.
#include "term2_kernel.cuh"

namespace s2b {
namespace mg {

void launch_term2_nt128(s2b_context* ctx, int variant, const TermArgs& a, const Term2Args& b, int nt, size_t smem,
                        size_t work) {
    switch (variant) {
    case 7: launch_term2_nt<7, 128>(ctx, a, b, nt, smem, work); return;
    case 8: launch_term2_nt<8, 128>(ctx, a, b, nt, smem, work); return;
    case 9: launch_term2_nt<9, 128>(ctx, a, b, nt, smem, work); return;
    }
    fail(S2B_ERR_RUNTIME, "term2 kernel: unknown variant");
}

} // namespace mg
} // namespace s2b
