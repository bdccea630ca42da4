// The hot kernel of the update phase: fused upscale -> Adam -> downscale,
// launched in its shipped configuration (adam_fused.cuh holds the template;
// the measured alternatives live in adam_variants.cu).
//
// 28 algorithmic bytes per parameter; the kernel is HBM-bound when the
// binary64 element math (~45 FP64 + ~12 XU instructions per element) and
// the memory latency are both hidden.
#include <cuda_runtime.h>

#include <cstdint>

#include "adam_fused.cuh"

namespace tfb {
namespace {

// Shipped configuration. One 16-bit gradient source in place (the engine's
// pipeline, the device-resident bench leg, the operator API): the staged
// kernel, 2 shared-memory stages of 2048 params (56 KiB) per CTA, 2 CTAs of
// 512 threads per SM (32 warps, 64 registers), f16 gradients widened straight
// to binary64, no second non-finite count behind a whole-phase check. Under
// the bench's sustained, power-capped load it holds 0.909-0.929 of the HBM
// copy peak on three boxes against 0.893-0.894 for the 256-thread / 4-CTA
// shape (tuning variants 70 vs 55, profiles/sustained_sweep_r2_nt_box*.json)
// and 0.84-0.85 for the register kernel; launched cool, 456 us per 100M
// params = 0.937, the best of every measured form (profiles/kernel_sweep_r2.json).
// Everything else (summed or fp32 gradients, separate outputs, misaligned or
// sub-tile launches, a launch's n % 1024 tail): the register kernel, one quad
// per thread per iteration, constant-divisor quotients, <= 64 registers for 4
// resident CTAs (32 warps) per SM (0.93-0.95 of the copy peak launched cool,
// profiles/kernel_sweep_r1.json).
using VariantDefault = Cfg<1, true, 4>;
constexpr int kStages = 2;
constexpr int kStagedCtasPerSm = 2;
constexpr int kStagedThreads = 512;
// Tuning variants (F16 gradients and params only), for the kernel sweep.

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

// Whether every gradient source is memory of the current device. Bulk copies
// (cp.async.bulk) from a peer's NVLink-mapped memory are not exercised on the
// one-GPU boxes this was measured on, so peer sources keep the register
// form's per-thread loads, which the multi-GPU tests cover.
static bool sources_on_this_device(const AdamLaunch& a) {
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    for (int s = 0; s < a.n_peers; ++s) {
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, a.peers[s]) != cudaSuccess) {
            (void)cudaGetLastError();
            return false;
        }
        if (at.type != cudaMemoryTypeDevice || at.device != dev) return false;
    }
    return true;
}

cudaError_t launch_adam_fused(const AdamLaunch& a, cudaStream_t stream) {
    if (a.n == 0) return cudaSuccess;
    cudaError_t e = cudaErrorNotSupported;
    // n summed gradient sources. With the sources in local HBM under
    // sustained load (profiles/multi_sustained_r2.json) the staged form wins
    // at 8 sources (0.920-0.965 vs 0.876-0.892 of the copy peak) and the
    // register form at 2 and 4, whose extra loads per thread already keep
    // enough bytes in flight.
    switch (a.n_peers) {
        case 0: e = launch_staged<kStages, kStagedCtasPerSm, 1, 1, 0, 0, kStagedThreads>(a, stream); break;
        case 8:  // 56 KiB per CTA: 3 fit an SM
            if (sources_on_this_device(a)) e = launch_staged<kStages, 3, 1, 1, 0, 8>(a, stream);
            break;
        default: break;
    }
    if (e != cudaErrorNotSupported) return e;
    return launch_dtypes<VariantDefault>(a, stream);
}

cudaError_t launch_divtest(double b, double y, uint64_t n, uint64_t seed, int exp_lo, int exp_span,
                           unsigned long long* mismatches, double* first_bad, cudaStream_t stream) {
    divtest_kernel<<<grid_for(n, 8), kThreads, 0, stream>>>(b, y, n, seed, exp_lo, exp_span, mismatches, first_bad);
    return cudaGetLastError();
}

}  // namespace tfb
