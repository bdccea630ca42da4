// sm_100a kernels of the update phase.
//
//  * adam_fused      — the hot kernel. One HBM pass per subgroup: read P,m,v
//                      (fp32) + the 16-bit gradient, widen, bias-corrected
//                      Adam/AdamW in binary64, write P,m,v + the 16-bit working
//                      params, and count non-finite gradients and narrowing
//                      overflows. Replaces upscale_f16_to_f32 -> adam_step ->
//                      downscale_f32_to_f16 (reference scheduler.hpp:467,479,490).
//  * synthetic_grads — SyntheticGradSource::fill + GradBufferF16::accumulate
//                      (scheduler.hpp:85-102, precision.hpp:66-75) on device.
//  * synthetic_state — synthetic_param_init + zero moments (scheduler.hpp:104-110,352).
//  * widen16 / narrow16 / count_nonfinite16 — the standalone precision
//                      operators (precision.hpp:17-43).
//
// Element-wise work: no tensor cores. Each thread streams 128-bit vectors
// (float4 of P, m, v; 4 x 16-bit of g and of the working params) with
// evict-first cache hints; the grid is a multiple of the SM count and
// grid-strides, so every SM keeps several quads in flight per thread.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels.hpp"
#include "launch_util.cuh"
#include "numerics.cuh"

namespace tfb {

using namespace detail;

namespace {

// ---------------------------------------------------------------------------
// Synthetic gradients. prefix = splitmix64 chain over (seed, sg, iteration,
// step) folded on the host; element i is splitmix64(prefix ^ i) mapped to
// [-0.25, 0.25), rounded double->float->16-bit. accumulate: the running
// buffer is widened, added in f32 and narrowed back (precision.hpp:66-75).
template <int K>
__global__ void __launch_bounds__(kThreads)
    synthetic_grads_kernel(uint16_t* __restrict__ out, uint64_t n, uint64_t prefix, int accumulate) {
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = tid; i < n; i += nthreads) {
        // The reference generator rounds the sample double -> float -> binary16;
        // the bf16 variant narrows the same float to bf16 instead.
        const uint16_t s = narrow16<K>(unit_to_float(splitmix64(prefix ^ i), 0.5));
        out[i] = accumulate ? narrow16<K>(__fadd_rn(widen16<K>(out[i]), widen16<K>(s))) : s;
    }
}

// synthetic_param_init(seed, sg, i) into P, zeros into m and v.
__global__ void __launch_bounds__(kThreads)
    synthetic_state_kernel(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                           uint64_t n, uint64_t prefix) {
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = tid; i < n; i += nthreads) {
        p[i] = unit_to_float(splitmix64(prefix ^ i), 0.2);
        m[i] = 0.0f;
        v[i] = 0.0f;
    }
}

template <int K>
__global__ void __launch_bounds__(kThreads)
    widen_kernel(const uint16_t* __restrict__ src, float* __restrict__ dst, uint64_t n,
                 unsigned long long* __restrict__ nonfinite_out) {
    unsigned bad = 0;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = tid; i < n; i += nthreads) {
        const uint16_t h = src[i];
        bad += nonfinite16<K>(h);
        dst[i] = widen16<K>(h);
    }
    if (nonfinite_out != nullptr) warp_count_add(nonfinite_out, bad);
}

template <int K>
__global__ void __launch_bounds__(kThreads)
    narrow_kernel(const float* __restrict__ src, uint16_t* __restrict__ dst, uint64_t n,
                  unsigned long long* __restrict__ overflow_out) {
    unsigned over = 0;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = tid; i < n; i += nthreads) {
        const uint16_t h = narrow16<K>(src[i]);
        over += is_inf16<K>(h);
        dst[i] = h;
    }
    if (overflow_out != nullptr) warp_count_add(overflow_out, over);
}

template <int K>
__global__ void __launch_bounds__(kThreads)
    count_nonfinite_kernel(const uint16_t* __restrict__ src, uint64_t n,
                           unsigned long long* __restrict__ out) {
    unsigned bad = 0;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t nq = n / 8;
    const uint4* s8 = reinterpret_cast<const uint4*>(src);
    const bool vec = (reinterpret_cast<uintptr_t>(src) & 15u) == 0;
    if (vec) {
        // 4 independent 16-byte loads in flight per thread before any is
        // counted: a read-only stream needs the bytes in flight, not the ALU.
        constexpr int U = 4;
        uint64_t q = tid;
        for (; q + (U - 1) * nthreads < nq; q += U * nthreads) {
            uint4 r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) r[u] = __ldcs(s8 + q + u * nthreads);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t w[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    bad += nonfinite16<K>(static_cast<uint16_t>(w[k] & 0xFFFFu)) +
                           nonfinite16<K>(static_cast<uint16_t>(w[k] >> 16));
            }
        }
        for (; q < nq; q += nthreads) {
            const uint4 r = __ldcs(s8 + q);
            const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
            for (int k = 0; k < 4; ++k)
                bad += nonfinite16<K>(static_cast<uint16_t>(w[k] & 0xFFFFu)) +
                       nonfinite16<K>(static_cast<uint16_t>(w[k] >> 16));
        }
        for (uint64_t i = nq * 8 + tid; i < n; i += nthreads) bad += nonfinite16<K>(src[i]);
    } else {
        for (uint64_t i = tid; i < n; i += nthreads) bad += nonfinite16<K>(src[i]);
    }
    warp_count_add(out, bad);
}

// Busy-waits `ns` nanoseconds of device time (synthetic per-subgroup update
// cost, the reference's update_pad_ns knob; scheduler.hpp:480-481).
__global__ void spin_kernel(uint64_t ns) {
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 >= ns) break;
        __nanosleep(1000);
    }
}

}  // namespace

// Scalar codecs on the host, the kernels' own __host__ __device__ code.
float widen16_scalar(uint16_t h, int kind) { return kind == kF16 ? widen16<kF16>(h) : widen16<kBF16>(h); }
uint16_t narrow16_scalar(float f, int kind) { return kind == kF16 ? narrow16<kF16>(f) : narrow16<kBF16>(f); }

cudaError_t launch_spin_ns(uint64_t ns, cudaStream_t stream) {
    if (ns == 0) return cudaSuccess;
    spin_kernel<<<1, 1, 0, stream>>>(ns);
    return cudaGetLastError();
}

cudaError_t launch_synthetic_grads(uint16_t* out, uint64_t n, int kind, uint64_t prefix,
                                   bool accumulate, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    const unsigned grid = grid_for(n, 8);
    if (kind == kF16)
        synthetic_grads_kernel<kF16><<<grid, kThreads, 0, stream>>>(out, n, prefix, accumulate ? 1 : 0);
    else
        synthetic_grads_kernel<kBF16><<<grid, kThreads, 0, stream>>>(out, n, prefix, accumulate ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_synthetic_state(float* p, float* m, float* v, uint64_t n, uint64_t prefix,
                                   cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    synthetic_state_kernel<<<grid_for(n, 8), kThreads, 0, stream>>>(p, m, v, n, prefix);
    return cudaGetLastError();
}

cudaError_t launch_widen16(const uint16_t* src, float* dst, uint64_t n, int kind,
                           unsigned long long* nonfinite_out, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    if (kind == kF16)
        widen_kernel<kF16><<<grid_for(n, 8), kThreads, 0, stream>>>(src, dst, n, nonfinite_out);
    else
        widen_kernel<kBF16><<<grid_for(n, 8), kThreads, 0, stream>>>(src, dst, n, nonfinite_out);
    return cudaGetLastError();
}

cudaError_t launch_narrow16(const float* src, uint16_t* dst, uint64_t n, int kind,
                            unsigned long long* overflow_out, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    if (kind == kF16)
        narrow_kernel<kF16><<<grid_for(n, 8), kThreads, 0, stream>>>(src, dst, n, overflow_out);
    else
        narrow_kernel<kBF16><<<grid_for(n, 8), kThreads, 0, stream>>>(src, dst, n, overflow_out);
    return cudaGetLastError();
}

cudaError_t launch_count_nonfinite16(const uint16_t* src, uint64_t n, int kind,
                                     unsigned long long* out, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    const unsigned grid = grid_for((n + 7) / 8, 8);
    if (kind == kF16)
        count_nonfinite_kernel<kF16><<<grid, kThreads, 0, stream>>>(src, n, out);
    else
        count_nonfinite_kernel<kBF16><<<grid, kThreads, 0, stream>>>(src, n, out);
    return cudaGetLastError();
}

namespace {

struct SumSources {
    const uint16_t* src[kMaxGradSources];
    int n;
};

// The reduction of several 16-bit sources (a data-parallel gradient's
// contributions, peers' through NVLink-mapped pointers): the fp32 sum in
// source order, rounded once to K — exactly what the fused multi-source
// update computes in-kernel — written to dst (may be null: count only) with
// the non-finite count of the rounded values. Quads of 8-byte loads from every
// source issued before the sum; NS sources fixed at compile time.
template <int K, int NS>
__global__ void __launch_bounds__(kThreads)
    reduce_sum16_kernel(SumSources s, uint64_t n, uint16_t* __restrict__ dst, unsigned long long* __restrict__ out) {
    unsigned bad = 0;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t nq = n / 4;
    for (uint64_t q = tid; q < nq; q += nthreads) {
        U16x4 x[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) x[k] = load_u16x4(s.src[k] + 4 * q);
        float4 acc = make_float4(-0.f, -0.f, -0.f, -0.f);  // -0 + x == x for every x: the sum starts at source 0
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            acc.x = __fadd_rn(acc.x, widen16<K>(x[k].x));
            acc.y = __fadd_rn(acc.y, widen16<K>(x[k].y));
            acc.z = __fadd_rn(acc.z, widen16<K>(x[k].z));
            acc.w = __fadd_rn(acc.w, widen16<K>(x[k].w));
        }
        U16x4 h;
        h.x = narrow16<K>(acc.x);
        h.y = narrow16<K>(acc.y);
        h.z = narrow16<K>(acc.z);
        h.w = narrow16<K>(acc.w);
        bad += nonfinite16<K>(h.x) + nonfinite16<K>(h.y) + nonfinite16<K>(h.z) + nonfinite16<K>(h.w);
        if (dst != nullptr) store_u16x4(dst + 4 * q, h);
    }
    for (uint64_t i = nq * 4 + tid; i < n; i += nthreads) {  // n % 4 tail
        float acc = -0.f;
#pragma unroll
        for (int k = 0; k < NS; ++k) acc = __fadd_rn(acc, widen16<K>(s.src[k][i]));
        const uint16_t h = narrow16<K>(acc);
        bad += nonfinite16<K>(h);
        if (dst != nullptr) dst[i] = h;
    }
    warp_count_add(out, bad);
}

// Scalar form for sources or destinations not 8-byte aligned.
template <int K>
__global__ void __launch_bounds__(kThreads)
    reduce_sum16_scalar_kernel(SumSources s, uint64_t n, uint16_t* __restrict__ dst,
                               unsigned long long* __restrict__ out) {
    unsigned bad = 0;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = tid; i < n; i += nthreads) {
        float acc = -0.f;
#pragma unroll
        for (int k = 0; k < kMaxGradSources; ++k)
            if (k < s.n) acc = __fadd_rn(acc, widen16<K>(__ldcs(s.src[k] + i)));
        const uint16_t h = narrow16<K>(acc);
        bad += nonfinite16<K>(h);
        if (dst != nullptr) dst[i] = h;
    }
    warp_count_add(out, bad);
}

template <int K, int NS>
void launch_reduce_ns(const SumSources& s, uint64_t n, uint16_t* dst, unsigned long long* out, cudaStream_t st) {
    reduce_sum16_kernel<K, NS><<<grid_for((n + 3) / 4, 8), kThreads, 0, st>>>(s, n, dst, out);
}

template <int K>
void launch_reduce(const SumSources& s, uint64_t n, uint16_t* dst, unsigned long long* out, cudaStream_t st,
                   bool vec) {
    if (!vec) {
        reduce_sum16_scalar_kernel<K><<<grid_for(n, 8), kThreads, 0, st>>>(s, n, dst, out);
        return;
    }
    switch (s.n) {
        case 1: return launch_reduce_ns<K, 1>(s, n, dst, out, st);
        case 2: return launch_reduce_ns<K, 2>(s, n, dst, out, st);
        case 3: return launch_reduce_ns<K, 3>(s, n, dst, out, st);
        case 4: return launch_reduce_ns<K, 4>(s, n, dst, out, st);
        case 5: return launch_reduce_ns<K, 5>(s, n, dst, out, st);
        case 6: return launch_reduce_ns<K, 6>(s, n, dst, out, st);
        case 7: return launch_reduce_ns<K, 7>(s, n, dst, out, st);
        default: return launch_reduce_ns<K, 8>(s, n, dst, out, st);
    }
}

}  // namespace

cudaError_t launch_reduce_sum16(const void* const* srcs, int nsrc, uint64_t n, int kind, uint16_t* dst,
                                unsigned long long* out, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    if (nsrc < 1 || nsrc > kMaxGradSources) return cudaErrorInvalidValue;
    SumSources s{};
    uintptr_t align = reinterpret_cast<uintptr_t>(dst);
    for (int k = 0; k < nsrc; ++k) {
        s.src[k] = static_cast<const uint16_t*>(srcs[k]);
        align |= reinterpret_cast<uintptr_t>(srcs[k]);
    }
    s.n = nsrc;
    const bool vec = (align & 7u) == 0;
    if (kind == kF16)
        launch_reduce<kF16>(s, n, dst, out, stream, vec);
    else
        launch_reduce<kBF16>(s, n, dst, out, stream, vec);
    return cudaGetLastError();
}

cudaError_t launch_count_nonfinite_sum16(const void* const* srcs, int nsrc, uint64_t n, int kind,
                                         unsigned long long* out, cudaStream_t stream) {
    return launch_reduce_sum16(srcs, nsrc, n, kind, nullptr, out, stream);
}

}  // namespace tfb
