// Host-side launchers for the sm_100a kernels (kernels.cu). Plain C++ so the
// engine and the C-ABI layer compile with g++ and only link against them.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "types.hpp"

namespace tfb {

// Maximum gradient sources of one fused launch (the data-parallel peers whose
// contributions the fused reduce + update sums).
constexpr int kMaxGradSources = 8;

struct AdamLaunch {
    float* p = nullptr;  // fp32 master params, in place
    float* m = nullptr;  // fp32 first moment, in place
    float* v = nullptr;  // fp32 second moment, in place
    const void* g = nullptr;  // gradient: 16-bit (grad_kind F16/BF16) or fp32 (grad_kind F32)
    // n_peers > 0: the gradient is the fp32 sum over these 16-bit sources (in
    // order), rounded once to grad_kind; g is ignored.
    const void* peers[kMaxGradSources] = {};
    int n_peers = 0;
    uint16_t* p16 = nullptr;  // 16-bit working params out (out_kind)
    // Optional separate destinations of the updated state (null = in place),
    // e.g. mapped pinned host memory: the D2H write-back fused into the kernel.
    float* p_out = nullptr;
    float* m_out = nullptr;
    float* v_out = nullptr;
    uint64_t n = 0;
    int grad_kind = 0;
    int out_kind = 0;
    AdamConsts c{};
    // [0] += non-finite gradient count, [1] += narrowing overflows (+-Inf
    // outputs). May be null.
    unsigned long long* counters = nullptr;
    // Device-side gate (may be null): when *gate != 0 at kernel start the
    // launch writes nothing. A whole-phase non-finite count accumulated into
    // it on the same stream rejects every later update of the phase without
    // a host round trip between the check and the updates.
    const unsigned long long* gate = nullptr;
    // The gradients were counted finite by a whole-phase check before this
    // launch (a host verdict, or the gate above): the kernel does not count
    // them again, counters[0] is left alone.
    bool grads_verified = false;
};

cudaError_t launch_adam_fused(const AdamLaunch& a, cudaStream_t stream);
// Tuning variants of the fused kernel (0 = default; F16/F16 only otherwise).
cudaError_t launch_adam_fused_variant(const AdamLaunch& a, int variant, cudaStream_t stream);
// The n-source launch in form `variant` (0 = shipped dispatch, 1 = register kernel).
cudaError_t launch_adam_fused_multi_variant(const AdamLaunch& a, int variant, cudaStream_t stream);
int adam_variant_count();
// Self-test of the second verified fast path: out[0] = largest |D'/D - 1| (double bits), out[1] += bit mismatches.
cudaError_t launch_fast_step_selftest(uint64_t n, uint64_t seed, unsigned long long* out, cudaStream_t stream);
// Self-test of the in-range sqrt / division (variant 47) against __dsqrt_rn / __ddiv_rn: *bad += mismatches.
cudaError_t launch_fast_rn_selftest(uint64_t n, uint64_t seed, unsigned long long* bad, cudaStream_t stream);
// Self-test: div_by_const(a, b, y) vs div.rn.f64 on generated numerators.
cudaError_t launch_divtest(double b, double y, uint64_t n, uint64_t seed, int exp_lo, int exp_span,
                           unsigned long long* mismatches, double* first_bad, cudaStream_t stream);
cudaError_t launch_synthetic_grads(uint16_t* out, uint64_t n, int kind, uint64_t prefix,
                                   bool accumulate, cudaStream_t stream);
cudaError_t launch_synthetic_state(float* p, float* m, float* v, uint64_t n, uint64_t prefix,
                                   cudaStream_t stream);
cudaError_t launch_widen16(const uint16_t* src, float* dst, uint64_t n, int kind,
                           unsigned long long* nonfinite_out, cudaStream_t stream);
cudaError_t launch_narrow16(const float* src, uint16_t* dst, uint64_t n, int kind,
                            unsigned long long* overflow_out, cudaStream_t stream);
cudaError_t launch_spin_ns(uint64_t ns, cudaStream_t stream);
// One-value conversions on the host (the kernels' codec, numerics.cuh).
float widen16_scalar(uint16_t h, int kind);
uint16_t narrow16_scalar(float f, int kind);
cudaError_t launch_count_nonfinite16(const uint16_t* src, uint64_t n, int kind,
                                     unsigned long long* out, cudaStream_t stream);
// Non-finite count of the fp32 sum (in order, rounded once to kind) of nsrc
// 16-bit sources: the pre-check of the fused multi-source update.
// The fp32 sum (in order, rounded once to kind) of nsrc 16-bit sources into
// dst (null: count only), *out += non-finite results: the engine's reduction
// of bound gradient sources at the phase check.
cudaError_t launch_reduce_sum16(const void* const* srcs, int nsrc, uint64_t n, int kind, uint16_t* dst,
                                unsigned long long* out, cudaStream_t stream);
cudaError_t launch_count_nonfinite_sum16(const void* const* srcs, int nsrc, uint64_t n, int kind,
                                         unsigned long long* out, cudaStream_t stream);

}  // namespace tfb
