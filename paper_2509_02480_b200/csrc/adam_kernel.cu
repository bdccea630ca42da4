// The hot kernel of the update phase: fused upscale -> Adam -> downscale.
//
// One HBM pass per subgroup replaces upscale_f16_to_f32 -> adam_step ->
// downscale_f32_to_f16 (reference scheduler.hpp:467, 479, 490): read P, m, v
// (fp32) and the 16-bit gradient, widen, bias-corrected Adam/AdamW in binary64
// (bit-exact with optimizer.hpp:91-108), write P, m, v and the 16-bit working
// params, and count non-finite gradients and narrowing overflows.
// 28 algorithmic bytes per parameter; the kernel is HBM-bound when the
// binary64 element math (~45 FP64 + ~12 XU instructions per element) and
// the memory latency are both hidden — hence the variants below, which trade
// per-thread unroll (independent loads in flight) against occupancy.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"
#include "launch_util.cuh"
#include "numerics.cuh"

namespace tfb {

using namespace detail;

namespace {

// VEC = true: P, m, v 16-byte aligned and g, p16 8-byte aligned; the body
// walks quads (float4 / 4 x 16-bit) and the n % 4 tail is scalar.
// VEC = false: scalar everywhere (e.g. a contiguous P||m||v with P % 4 != 0).
template <int GK, int OK, bool WD, bool VEC, int UNROLL, bool DIVC, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    adam_fused_kernel(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                      const uint16_t* __restrict__ g, uint16_t* __restrict__ p16, uint64_t n,
                      AdamConsts c, unsigned long long* __restrict__ counters) {
    unsigned nonfinite = 0, overflow = 0;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;

    if constexpr (VEC) {
        const uint64_t nq = n / 4;
        float4* p4 = reinterpret_cast<float4*>(p);
        float4* m4 = reinterpret_cast<float4*>(m);
        float4* v4 = reinterpret_cast<float4*>(v);
        for (uint64_t base = tid; base < nq; base += nthreads * UNROLL) {
            float4 rp[UNROLL], rm[UNROLL], rv[UNROLL];
            U16x4 rg[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {  // all loads first: UNROLL quads in flight
                const uint64_t q = base + static_cast<uint64_t>(u) * nthreads;
                if (q < nq) {
                    rp[u] = __ldcs(p4 + q);
                    rm[u] = __ldcs(m4 + q);
                    rv[u] = __ldcs(v4 + q);
                    rg[u] = load_u16x4(g + 4 * q);
                }
            }
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const uint64_t q = base + static_cast<uint64_t>(u) * nthreads;
                if (q < nq) {
                    nonfinite += nonfinite16<GK>(rg[u].x) + nonfinite16<GK>(rg[u].y) +
                                 nonfinite16<GK>(rg[u].z) + nonfinite16<GK>(rg[u].w);
                    adam_element<WD, DIVC>(rp[u].x, rm[u].x, rv[u].x, widen16<GK>(rg[u].x), c);
                    adam_element<WD, DIVC>(rp[u].y, rm[u].y, rv[u].y, widen16<GK>(rg[u].y), c);
                    adam_element<WD, DIVC>(rp[u].z, rm[u].z, rv[u].z, widen16<GK>(rg[u].z), c);
                    adam_element<WD, DIVC>(rp[u].w, rm[u].w, rv[u].w, widen16<GK>(rg[u].w), c);
                    U16x4 h;
                    h.x = narrow16<OK>(rp[u].x);
                    h.y = narrow16<OK>(rp[u].y);
                    h.z = narrow16<OK>(rp[u].z);
                    h.w = narrow16<OK>(rp[u].w);
                    overflow += is_inf16<OK>(h.x) + is_inf16<OK>(h.y) + is_inf16<OK>(h.z) + is_inf16<OK>(h.w);
                    __stcs(p4 + q, rp[u]);
                    __stcs(m4 + q, rm[u]);
                    __stcs(v4 + q, rv[u]);
                    store_u16x4(p16 + 4 * q, h);
                }
            }
        }
        const uint64_t i = nq * 4 + tid;  // scalar tail: n % 4 elements
        if (i < n) {
            float pf = p[i], mf = m[i], vf = v[i];
            const uint16_t gh = g[i];
            nonfinite += nonfinite16<GK>(gh);
            adam_element<WD, DIVC>(pf, mf, vf, widen16<GK>(gh), c);
            const uint16_t h = narrow16<OK>(pf);
            overflow += is_inf16<OK>(h);
            p[i] = pf;
            m[i] = mf;
            v[i] = vf;
            p16[i] = h;
        }
    } else {
        for (uint64_t i = tid; i < n; i += nthreads) {
            float pf = __ldcs(p + i), mf = __ldcs(m + i), vf = __ldcs(v + i);
            const uint16_t gh = __ldcs(g + i);
            nonfinite += nonfinite16<GK>(gh);
            adam_element<WD, DIVC>(pf, mf, vf, widen16<GK>(gh), c);
            const uint16_t h = narrow16<OK>(pf);
            overflow += is_inf16<OK>(h);
            __stcs(p + i, pf);
            __stcs(m + i, mf);
            __stcs(v + i, vf);
            p16[i] = h;
        }
    }
    if (counters != nullptr) {
        warp_count_add(counters + 0, nonfinite);
        warp_count_add(counters + 1, overflow);
    }
}

template <int UNROLL, bool DIVC, int MINB>
struct Cfg {
    static constexpr int kUnroll = UNROLL;
    static constexpr bool kDivc = DIVC;
    static constexpr int kMinBlocks = MINB;
};

bool is_vec(const AdamLaunch& a) {
    return ((reinterpret_cast<uintptr_t>(a.p) | reinterpret_cast<uintptr_t>(a.m) | reinterpret_cast<uintptr_t>(a.v)) &
            15u) == 0 &&
           ((reinterpret_cast<uintptr_t>(a.g) | reinterpret_cast<uintptr_t>(a.p16)) & 7u) == 0;
}

template <int GK, int OK, bool WD, class C>
cudaError_t launch_cfg(const AdamLaunch& a, cudaStream_t stream) {
    constexpr int U = C::kUnroll;
    constexpr int B = C::kMinBlocks;
    if (is_vec(a)) {
        const unsigned grid = grid_for((a.n / 4 + U - 1) / U, B);
        adam_fused_kernel<GK, OK, WD, true, U, C::kDivc, B>
            <<<grid, kThreads, 0, stream>>>(a.p, a.m, a.v, a.g, a.p16, a.n, a.c, a.counters);
    } else {
        const unsigned grid = grid_for(a.n, B);
        adam_fused_kernel<GK, OK, WD, false, 1, C::kDivc, B>
            <<<grid, kThreads, 0, stream>>>(a.p, a.m, a.v, a.g, a.p16, a.n, a.c, a.counters);
    }
    return cudaGetLastError();
}

template <int GK, int OK, class C>
cudaError_t launch_wd(const AdamLaunch& a, cudaStream_t stream) {
    return a.c.lr_wd != 0.0 ? launch_cfg<GK, OK, true, C>(a, stream) : launch_cfg<GK, OK, false, C>(a, stream);
}

template <class C>
cudaError_t launch_dtypes(const AdamLaunch& a, cudaStream_t stream) {
    if (a.grad_kind == kF16 && a.out_kind == kF16) return launch_wd<kF16, kF16, C>(a, stream);
    if (a.grad_kind == kF16 && a.out_kind == kBF16) return launch_wd<kF16, kBF16, C>(a, stream);
    if (a.grad_kind == kBF16 && a.out_kind == kF16) return launch_wd<kBF16, kF16, C>(a, stream);
    return launch_wd<kBF16, kBF16, C>(a, stream);
}

// Shipped configuration: one quad per thread per iteration, constant-divisor
// quotients, <= 64 registers for 4 resident CTAs (32 warps) per SM. The
// 2026-10-17 sweep (profiles/kernel_sweep_r1.json) measured it at 474 us per
// 100M-param launch, 5.90 TB/s algorithmic = 0.92 of the measured HBM copy
// peak, against 1045 us for the register-heavy unroll-2 form (variant 1).
using VariantDefault = Cfg<1, true, 4>;
// Tuning variants (F16 gradients and params only), for the kernel sweep.
template <int V>
cudaError_t launch_variant(const AdamLaunch& a, cudaStream_t stream) {
    if constexpr (V == 1) return launch_wd<kF16, kF16, Cfg<2, false, 1>>(a, stream);
    if constexpr (V == 2) return launch_wd<kF16, kF16, Cfg<1, false, 4>>(a, stream);
    if constexpr (V == 3) return launch_wd<kF16, kF16, Cfg<2, false, 3>>(a, stream);
    if constexpr (V == 4) return launch_wd<kF16, kF16, Cfg<1, true, 4>>(a, stream);
    if constexpr (V == 5) return launch_wd<kF16, kF16, Cfg<2, true, 3>>(a, stream);
    if constexpr (V == 6) return launch_wd<kF16, kF16, Cfg<2, true, 2>>(a, stream);
    if constexpr (V == 7) return launch_wd<kF16, kF16, Cfg<1, true, 3>>(a, stream);
    if constexpr (V == 8) return launch_wd<kF16, kF16, Cfg<4, true, 2>>(a, stream);
    if constexpr (V == 9) return launch_wd<kF16, kF16, Cfg<1, true, 5>>(a, stream);
    if constexpr (V == 10) return launch_wd<kF16, kF16, Cfg<2, true, 4>>(a, stream);
    if constexpr (V == 11) return launch_wd<kF16, kF16, Cfg<1, true, 6>>(a, stream);
    return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// Self-test of div_by_const against div.rn.f64: numerators with random 52-bit
// significands over a wide exponent range plus structured near-boundary cases.
__global__ void divtest_kernel(double b, double y, uint64_t n, uint64_t seed, int exp_lo, int exp_span,
                               unsigned long long* mismatches, double* first_bad) {
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    unsigned bad = 0;
    for (uint64_t i = tid; i < n; i += nthreads) {
        const uint64_t r = splitmix64(seed ^ (i * 0x9E3779B97F4A7C15ULL));
        uint64_t mant = r & 0xFFFFFFFFFFFFFULL;
        const int sel = static_cast<int>((r >> 52) & 7u);
        if (sel == 0) mant |= 0xFFFFFFFFFF000ULL;  // near the top of the binade
        if (sel == 1) mant &= 0x0000000000FFFULL;  // near a power of two
        const int e = exp_lo + static_cast<int>((r >> 55) % static_cast<uint64_t>(exp_span));
        double a = __longlong_as_double(static_cast<long long>((static_cast<uint64_t>(e + 1023) << 52) | mant));
        if (r >> 63) a = -a;
        if (sel == 2) a = __dmul_rn(b, static_cast<double>(static_cast<int>(r & 0xFFFF)));  // exact multiples
        const double want = __ddiv_rn(a, b);
        const double got = div_by_const(a, b, y);
        if (__double_as_longlong(want) != __double_as_longlong(got)) {
            ++bad;
            *first_bad = a;
        }
    }
    warp_count_add(mismatches, bad);
}

}  // namespace

cudaError_t launch_adam_fused(const AdamLaunch& a, cudaStream_t stream) {
    if (a.n == 0) return cudaSuccess;
    return launch_dtypes<VariantDefault>(a, stream);
}

cudaError_t launch_adam_fused_variant(const AdamLaunch& a, int variant, cudaStream_t stream) {
    if (a.n == 0) return cudaSuccess;
    if (variant == 0) return launch_adam_fused(a, stream);
    if (a.grad_kind != kF16 || a.out_kind != kF16) return cudaErrorInvalidValue;
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
        default: return cudaErrorInvalidValue;
    }
}

int adam_variant_count() { return 12; }

cudaError_t launch_divtest(double b, double y, uint64_t n, uint64_t seed, int exp_lo, int exp_span,
                           unsigned long long* mismatches, double* first_bad, cudaStream_t stream) {
    divtest_kernel<<<grid_for(n, 8), kThreads, 0, stream>>>(b, y, n, seed, exp_lo, exp_span, mismatches, first_bad);
    return cudaGetLastError();
}

}  // namespace tfb
