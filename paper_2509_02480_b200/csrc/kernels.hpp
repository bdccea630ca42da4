// Host-side launchers for the sm_100a kernels (kernels.cu). Plain C++ so the
// engine and the C-ABI layer compile with g++ and only link against them.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "types.hpp"

namespace tfb {


// Resident CTAs per SM the fused kernel grid is sized for (grid = SMs x this).
constexpr int kAdamCtasPerSm = 4;

struct AdamLaunch {
    float* p = nullptr;  // fp32 master params, in place
    float* m = nullptr;  // fp32 first moment, in place
    float* v = nullptr;  // fp32 second moment, in place
    const uint16_t* g = nullptr;  // 16-bit gradient (grad_kind)
    uint16_t* p16 = nullptr;      // 16-bit working params out (out_kind)
    uint64_t n = 0;
    int grad_kind = 0;
    int out_kind = 0;
    AdamConsts c{};
    // [0] += non-finite gradient count, [1] += narrowing overflows (+-Inf
    // outputs). May be null.
    unsigned long long* counters = nullptr;
};

cudaError_t launch_adam_fused(const AdamLaunch& a, cudaStream_t stream);
cudaError_t launch_synthetic_grads(uint16_t* out, uint64_t n, int kind, uint64_t prefix,
                                   bool accumulate, cudaStream_t stream);
cudaError_t launch_synthetic_state(float* p, float* m, float* v, uint64_t n, uint64_t prefix,
                                   cudaStream_t stream);
cudaError_t launch_widen16(const uint16_t* src, float* dst, uint64_t n, int kind,
                           unsigned long long* nonfinite_out, cudaStream_t stream);
cudaError_t launch_narrow16(const float* src, uint16_t* dst, uint64_t n, int kind,
                            unsigned long long* overflow_out, cudaStream_t stream);
cudaError_t launch_spin_ns(uint64_t ns, cudaStream_t stream);
cudaError_t launch_count_nonfinite16(const uint16_t* src, uint64_t n, int kind,
                                     unsigned long long* out, cudaStream_t stream);

}  // namespace tfb
