// term_tma_kernel instantiations for blocks of up to 128 threads.
#include "term_kernel.cuh"

namespace s2b {
namespace mg {

void launch_term_nt128(s2b_context* ctx, int variant, const TermArgs& a, int nt, size_t smem, size_t work) {
    switch (variant) {
    case 1: launch_term_nt<1, 128>(ctx, a, nt, smem, work); return;
    case 2: launch_term_nt<2, 128>(ctx, a, nt, smem, work); return;
    case 3: launch_term_nt<3, 128>(ctx, a, nt, smem, work); return;
    case 4: launch_term_nt<4, 128>(ctx, a, nt, smem, work); return;
    case 5: launch_term_nt<5, 128>(ctx, a, nt, smem, work); return;
    case 6: launch_term_nt<6, 128>(ctx, a, nt, smem, work); return;
    case 7: launch_term_nt<7, 128>(ctx, a, nt, smem, work); return;
    case 8: launch_term_nt<8, 128>(ctx, a, nt, smem, work); return;
    case 9: launch_term_nt<9, 128>(ctx, a, nt, smem, work); return;
    }
    fail(S2B_ERR_RUNTIME, "term kernel: unknown variant");
}

} // namespace mg
} // namespace s2b
