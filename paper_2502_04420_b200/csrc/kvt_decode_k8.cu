// Instances of the decode kernel for key bits = 8 (split across files for parallel compilation).
#include "kvt_decode.cuh"
#include "kvt_decode_mma.cuh"

namespace kvt {
namespace dec {

using KFn = void (*)(DecodeArgs);

template <int VB, bool KPC>
static KFn pick_gm(int GM) {
    return GM == 4 ? decode_kernel<8, VB, KPC, 4> : decode_kernel<8, VB, KPC, 8>;
}

template <bool KPC>
static KFn pick_vb(int VB, int GM) {
    switch (VB) {
        case 2: return pick_gm<2, KPC>(GM);
        case 4: return pick_gm<4, KPC>(GM);
        case 8: return pick_gm<8, KPC>(GM);
        default: return pick_gm<16, KPC>(GM);
    }
}

KFn get_decode_k8(int VB, bool KPC, int GM) {
    return KPC ? pick_vb<true>(VB, GM) : pick_vb<false>(VB, GM);
}

// tensor-core instances (G = 32 tile records): returns the kernel and its dynamic shared memory.
// KPT (per-token keys): q needs no hi/lo split, so with g <= 4 the 8 columns hold the 4 heads twice (the
// lanes tig and tig ^ 2 then see the same heads, as after the KIVI hi/lo fold).
template <int VB, bool P>
static KFn mma_pick(int GM, bool kpt, size_t* smem) {
    if (kpt && GM == 4) { *smem = mma::Geo<8, VB, 4>::SMEM; return mma::decode_mma_kernel<8, VB, 4, true, P>; }
    if (kpt) { *smem = mma::Geo<8, VB, 8>::SMEM; return mma::decode_mma_kernel<8, VB, 8, true, P>; }
    if (GM == 4) { *smem = mma::Geo<8, VB, 4>::SMEM; return mma::decode_mma_kernel<8, VB, 4, false, P>; }
    *smem = mma::Geo<8, VB, 8>::SMEM;
    return mma::decode_mma_kernel<8, VB, 8, false, P>;
}

template <bool P>
static KFn mma_pick_vb(int VB, int GM, bool kpt, size_t* smem) {
    switch (VB) {
        case 2: return mma_pick<2, P>(GM, kpt, smem);
        case 4: return mma_pick<4, P>(GM, kpt, smem);
        default: return mma_pick<8, P>(GM, kpt, smem);
    }
}

KFn get_decode_mma_k8(int VB, int GM, bool kpt, bool paged, size_t* smem) {
    return paged ? mma_pick_vb<true>(VB, GM, kpt, smem) : mma_pick_vb<false>(VB, GM, kpt, smem);
}

}  // namespace dec
}  // namespace kvt
