// Tuning variants of the fused Adam kernel, second half (variants 34 and up)
// and the n-source forms (tfg_adam_fused_multi_variant): a separate
// translation unit so the tuning library's two halves compile in parallel.
#include "adam_variants.cuh"

namespace tfb {

// Variants 68-71: the staged kernel with larger CTAs (NT threads): bigger
// tiles (4 x NT params, i.e. larger bulk copies) at full occupancy.
template <int S, int M, int NT>
cudaError_t launch_staged_nt(const AdamLaunch& a, cudaStream_t stream) {
    AdamLaunch b = a;
    b.grads_verified = true;
    return launch_staged<S, M, 1, 1, 0, 0, NT>(b, stream);
}

cudaError_t launch_adam_fused_variant_hi(const AdamLaunch& a, int variant, cudaStream_t stream) {
    switch (variant) {
        case 68: return launch_staged_nt<2, 3, 320>(a, stream);
        case 69: return launch_staged_nt<2, 2, 384>(a, stream);
        case 70: return launch_staged_nt<2, 2, 512>(a, stream);
        case 71: return launch_staged_nt<3, 2, 512>(a, stream);
        case 34: return launch_variant<34>(a, stream);
        case 35: return launch_variant<35>(a, stream);
        case 36: return launch_variant<36>(a, stream);
        case 37: return launch_variant<37>(a, stream);
        case 38: return launch_variant<38>(a, stream);
        case 39: return launch_variant<39>(a, stream);
        case 40: return launch_variant<40>(a, stream);
        case 41: return launch_variant<41>(a, stream);
        case 42: return launch_variant<42>(a, stream);
        case 43: return launch_variant<43>(a, stream);
        case 44: return launch_variant<44>(a, stream);
        case 45: return launch_variant<45>(a, stream);
        case 46: return launch_variant<46>(a, stream);
        case 47: return launch_variant<47>(a, stream);
        case 48: return launch_variant<48>(a, stream);
        case 49: return launch_variant<49>(a, stream);
        case 50: return launch_variant<50>(a, stream);
        case 51: return launch_variant<51>(a, stream);
        case 52: return launch_variant<52>(a, stream);
        case 53: return launch_variant<53>(a, stream);
        case 54: return launch_variant<54>(a, stream);
        case 55: return launch_variant<55>(a, stream);
        case 56: return launch_variant<56>(a, stream);
        case 57: return launch_variant<57>(a, stream);
        case 58: return launch_variant<58>(a, stream);
        case 59: return launch_variant<59>(a, stream);
        case 60: return launch_variant<60>(a, stream);
        case 61: return launch_variant<61>(a, stream);
        case 62: return launch_variant<62>(a, stream);
        case 63: return launch_variant<63>(a, stream);
        case 64: return launch_variant<64>(a, stream);
        case 65: return launch_variant<65>(a, stream);
        case 66: return launch_variant<66>(a, stream);
        case 67: return launch_variant<67>(a, stream);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_adam_fused_multi_variant(const AdamLaunch& a, int variant, cudaStream_t stream) {
    if (a.n == 0) return cudaSuccess;
    if (variant == 1) return launch_dtypes<Cfg<1, true, 4>>(a, stream);
    // 0: the staged n-source kernel (2, 4, 8 sources; anything else the register form)
    cudaError_t e = cudaErrorNotSupported;
    if (a.n_peers == 2) e = launch_staged<2, 4, 1, 1, 0, 2>(a, stream);
    if (a.n_peers == 4) e = launch_staged<2, 4, 1, 1, 0, 4>(a, stream);
    if (a.n_peers == 8) e = launch_staged<2, 3, 1, 1, 0, 8>(a, stream);
    return e == cudaErrorNotSupported ? launch_dtypes<Cfg<1, true, 4>>(a, stream) : e;
}

}  // namespace tfb
