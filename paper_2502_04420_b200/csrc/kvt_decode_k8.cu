// Instances of the decode kernel for key bits = 8 (split across files for parallel compilation).
#include "kvt_decode.cuh"

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

}  // namespace dec
}  // namespace kvt
