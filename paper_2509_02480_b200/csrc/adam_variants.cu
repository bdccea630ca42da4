// Tuning variants of the fused Adam kernel, first half (variants 1-33) and the
// dispatch; the kernels themselves are in adam_variants.cuh, variants 34 and
// up in adam_variants_hi.cu. See adam_variants.cuh for what each one is.
#include "adam_variants.cuh"

namespace tfb {

// Self-test of adam_element_fast2's error bound: the step D' it computes
// against the exact chain's D on random (m, v, t) spanning many exponents;
// the largest |D'/D - 1| observed (as -log2) and how many elements would
// take the exact fallback for p = RN(±u), u in [0.01, 1).
__global__ void fast_step_selftest_kernel(uint64_t n, uint64_t seed, double lr, double beta1, double beta2,
                                          double eps, unsigned long long* worst_bits,
                                          unsigned long long* fallbacks) {
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    double worst = 0.0;
    unsigned fb = 0;
    for (uint64_t i = tid; i < n; i += nthreads) {
        const uint64_t r1 = splitmix64(seed ^ (2 * i)), r2 = splitmix64(seed ^ (2 * i + 1));
        const int t = 1 + static_cast<int>(r1 % 20000);
        const double bc1 = 1.0 - pow(beta1, static_cast<double>(t));
        const double bc2 = 1.0 - pow(beta2, static_cast<double>(t));
        const double ib1 = 1.0 / bc1, ib2 = 1.0 / bc2;
        const double m = ldexp(static_cast<double>(static_cast<float>((r1 >> 11) * 0x1.0p-53 - 0.5)),
                               -static_cast<int>((r1 >> 40) % 40));
        const double v = ldexp(static_cast<double>(static_cast<float>((r2 >> 11) * 0x1.0p-53)),
                               -static_cast<int>((r2 >> 40) % 80));
        const double vh = v * ib2;
        if (!(vh > 0.0)) continue;
        double y, r;
        asm("rsqrt.approx.f64 %0, %1;" : "=d"(y) : "d"(vh));
        y = fma(0.5 * y, fma(-(vh * y), y, 1.0), y);
        const double den = fma(vh, y, eps);
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
        r = fma(r, fma(-den, r, 1.0), r);
        const double step = (m * (lr * ib1)) * r;
        const double mhat = div_by_const(m, bc1, ib1);
        const double vhat = div_by_const(v, bc2, ib2);
        const double exact = __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), eps));
        if (exact != 0.0) worst = fmax(worst, fabs(step / exact - 1.0));
        float pf = static_cast<float>((2.0 * ((r2 >> 11) & 1) - 1.0) * (0.01 + 0.99 * ((r2 >> 12) % 1000003) / 1000003.0));
        float mf = static_cast<float>(m), vf = static_cast<float>(v), pf2 = pf, mf2 = mf, vf2 = vf;
        AdamConsts c{lr, beta1, beta2, 1.0 - beta1, 1.0 - beta2, eps, 0.0, bc1, bc2, ib1, ib2};
        adam_element<false, true>(pf, mf, vf, 0.0f, c);
        adam_element_fast2<false, 30>(pf2, mf2, vf2, 0.0f, c);
        if (__float_as_uint(pf) != __float_as_uint(pf2) || __float_as_uint(mf) != __float_as_uint(mf2) ||
            __float_as_uint(vf) != __float_as_uint(vf2))
            atomicAdd(fallbacks + 1, 1ull);  // a bit mismatch: must stay 0
        (void)fb;
    }
    atomicMax(worst_bits, static_cast<unsigned long long>(__double_as_longlong(worst)));
}

cudaError_t launch_fast_rn_selftest(uint64_t n, uint64_t seed, unsigned long long* bad, cudaStream_t stream) {
    fast_rn_selftest_kernel<<<grid_for(n, 4), kThreads, 0, stream>>>(n, seed, bad);
    return cudaGetLastError();
}

cudaError_t launch_fast_step_selftest(uint64_t n, uint64_t seed, unsigned long long* out, cudaStream_t stream) {
    fast_step_selftest_kernel<<<grid_for(n, 4), kThreads, 0, stream>>>(n, seed, 1e-3, 0.9, 0.999, 1e-8, out, out);
    return cudaGetLastError();
}

cudaError_t launch_adam_fused_variant(const AdamLaunch& a, int variant, cudaStream_t stream) {
    if (a.n == 0) return cudaSuccess;
    if (variant == 0) return launch_adam_fused(a, stream);
    if (a.grad_kind != kF16 || a.out_kind != kF16 || a.n_peers > 0) return cudaErrorInvalidValue;
    switch (variant) {
        case 1: return launch_variant<1>(a, stream);
        case 2: return launch_variant<2>(a, stream);
        case 3: return launch_variant<3>(a, stream);
        case 4: return launch_variant<4>(a, stream);
        case 5: return launch_variant<5>(a, stream);
        case 6: return launch_variant<6>(a, stream);
        case 7: return launch_variant<7>(a, stream);
        case 8: return launch_variant<8>(a, stream);
        case 9: return launch_variant<9>(a, stream);
        case 10: return launch_variant<10>(a, stream);
        case 11: return launch_variant<11>(a, stream);
        case 12: return launch_variant<12>(a, stream);
        case 13: return launch_variant<13>(a, stream);
        case 14: return launch_variant<14>(a, stream);
        case 15: return launch_variant<15>(a, stream);
        case 16: return launch_variant<16>(a, stream);
        case 17: return launch_variant<17>(a, stream);
        case 18: return launch_variant<18>(a, stream);
        case 19: return launch_variant<19>(a, stream);
        case 20: return launch_variant<20>(a, stream);
        case 21: return launch_variant<21>(a, stream);
        case 22: return launch_variant<22>(a, stream);
        case 23: return launch_variant<23>(a, stream);
        case 24: return launch_variant<24>(a, stream);
        case 25: return launch_variant<25>(a, stream);
        case 26: return launch_variant<26>(a, stream);
        case 27: return launch_variant<27>(a, stream);
        case 28: return launch_variant<28>(a, stream);
        case 29: return launch_variant<29>(a, stream);
        case 30: return launch_variant<30>(a, stream);
        case 31: return launch_variant<31>(a, stream);
        case 32: return launch_variant<32>(a, stream);
        case 33: return launch_variant<33>(a, stream);
        default: return launch_adam_fused_variant_hi(a, variant, stream);
    }
}

int adam_variant_count() { return 72; }

}  // namespace tfb
