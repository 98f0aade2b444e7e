// Instances of the decode kernel for key bits = 16 (split across files for parallel compilation).
#include "kvt_decode.cuh"

namespace kvt {
namespace dec {

using KFn = void (*)(DecodeArgs);

template <int VB, bool KPC>
static KFn pick_gm(int GM) {
    return GM == 4 ? decode_kernel<16, VB, KPC, 4> : decode_kernel<16, VB, KPC, 8>;
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

KFn get_decode_k16(int VB, bool KPC, int GM) {
    (void)KPC;  // a bf16 key is never per-channel
    return pick_vb<false>(VB, GM);
}

}  // namespace dec
}  // namespace kvt
