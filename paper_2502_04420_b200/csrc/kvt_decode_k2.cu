// Instances of the decode kernel for key bits = 2 (split across files for parallel compilation).
#include "kvt_decode.cuh"
#include "kvt_decode_mma.cuh"

namespace kvt {
namespace dec {

using KFn = void (*)(DecodeArgs);

template <int VB, bool KPC>
static KFn pick_gm(int GM) {
    return GM == 4 ? decode_kernel<2, VB, KPC, 4> : decode_kernel<2, VB, KPC, 8>;
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

KFn get_decode_k2(int VB, bool KPC, int GM) {
    return KPC ? pick_vb<true>(VB, GM) : pick_vb<false>(VB, GM);
}

// tensor-core KIVI instances (G = 32): returns the kernel and its dynamic shared memory
KFn get_decode_mma_k2(int VB, int GM, size_t* smem) {
    switch (VB) {
        case 2: *smem = GM == 4 ? mma::Geo<2, 2, 4>::SMEM : mma::Geo<2, 2, 8>::SMEM; return GM == 4 ? mma::decode_mma_kernel<2, 2, 4> : mma::decode_mma_kernel<2, 2, 8>;
        case 4: *smem = GM == 4 ? mma::Geo<2, 4, 4>::SMEM : mma::Geo<2, 4, 8>::SMEM; return GM == 4 ? mma::decode_mma_kernel<2, 4, 4> : mma::decode_mma_kernel<2, 4, 8>;
        default: *smem = GM == 4 ? mma::Geo<2, 8, 4>::SMEM : mma::Geo<2, 8, 8>::SMEM; return GM == 4 ? mma::decode_mma_kernel<2, 8, 4> : mma::decode_mma_kernel<2, 8, 8>;
    }
}

}  // namespace dec
}  // namespace kvt
