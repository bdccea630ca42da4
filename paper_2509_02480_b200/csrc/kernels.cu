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
#include "numerics.cuh"

namespace tfb {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void warp_count_add(unsigned long long* dst, unsigned local) {
    const unsigned total = __reduce_add_sync(0xFFFFFFFFu, local);
    if (total != 0 && (threadIdx.x & 31) == 0) atomicAdd(dst, static_cast<unsigned long long>(total));
}

struct alignas(8) U16x4 {
    uint16_t x, y, z, w;
};

__device__ __forceinline__ U16x4 load_u16x4(const uint16_t* p) {
    const uint2 r = __ldcs(reinterpret_cast<const uint2*>(p));
    U16x4 o;
    o.x = static_cast<uint16_t>(r.x & 0xFFFFu);
    o.y = static_cast<uint16_t>(r.x >> 16);
    o.z = static_cast<uint16_t>(r.y & 0xFFFFu);
    o.w = static_cast<uint16_t>(r.y >> 16);
    return o;
}

__device__ __forceinline__ void store_u16x4(uint16_t* p, U16x4 v) {
    uint2 r;
    r.x = static_cast<uint32_t>(v.x) | (static_cast<uint32_t>(v.y) << 16);
    r.y = static_cast<uint32_t>(v.z) | (static_cast<uint32_t>(v.w) << 16);
    __stcs(reinterpret_cast<uint2*>(p), r);
}

// ---------------------------------------------------------------------------
// Fused Adam. VEC = true: all five streams are 16-byte (P,m,v) / 8-byte (g,
// p16) aligned and the body walks quads; the n % 4 tail is handled scalar by
// the first threads. VEC = false: scalar everywhere (ragged contiguous P||m||v
// views with P % 4 != 0).
template <int GK, int OK, bool WD, bool VEC, int UNROLL>
__global__ void __launch_bounds__(kThreads)
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
            for (int u = 0; u < UNROLL; ++u) {
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
                    adam_element<WD>(rp[u].x, rm[u].x, rv[u].x, widen16<GK>(rg[u].x), c);
                    adam_element<WD>(rp[u].y, rm[u].y, rv[u].y, widen16<GK>(rg[u].y), c);
                    adam_element<WD>(rp[u].z, rm[u].z, rv[u].z, widen16<GK>(rg[u].z), c);
                    adam_element<WD>(rp[u].w, rm[u].w, rv[u].w, widen16<GK>(rg[u].w), c);
                    U16x4 h;
                    h.x = narrow16<OK>(rp[u].x);
                    h.y = narrow16<OK>(rp[u].y);
                    h.z = narrow16<OK>(rp[u].z);
                    h.w = narrow16<OK>(rp[u].w);
                    overflow += is_inf16<OK>(h.x) + is_inf16<OK>(h.y) + is_inf16<OK>(h.z) +
                                is_inf16<OK>(h.w);
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
            adam_element<WD>(pf, mf, vf, widen16<GK>(gh), c);
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
            adam_element<WD>(pf, mf, vf, widen16<GK>(gh), c);
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
        for (uint64_t q = tid; q < nq; q += nthreads) {
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

int g_num_sms = 0;

int num_sms() {
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        int sms = 0;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
            sms = 148;
        g_num_sms = sms;
    }
    return g_num_sms;
}

// Grid sized to whole waves of the SM count, capped by the work.
unsigned grid_for(uint64_t work_items, int ctas_per_sm) {
    const uint64_t need = (work_items + kThreads - 1) / kThreads;
    const uint64_t cap = static_cast<uint64_t>(num_sms()) * static_cast<uint64_t>(ctas_per_sm);
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min(need, cap)));
}

template <int GK, int OK, bool WD>
cudaError_t launch_adam_typed(const AdamLaunch& a, cudaStream_t stream) {
    constexpr int kUnroll = 2;
    const bool vec = ((reinterpret_cast<uintptr_t>(a.p) | reinterpret_cast<uintptr_t>(a.m) |
                       reinterpret_cast<uintptr_t>(a.v)) & 15u) == 0 &&
                     ((reinterpret_cast<uintptr_t>(a.g) | reinterpret_cast<uintptr_t>(a.p16)) & 7u) == 0;
    if (vec) {
        const unsigned grid = grid_for((a.n / 4 + kUnroll - 1) / kUnroll, kAdamCtasPerSm);
        adam_fused_kernel<GK, OK, WD, true, kUnroll><<<grid, kThreads, 0, stream>>>(
            a.p, a.m, a.v, a.g, a.p16, a.n, a.c, a.counters);
    } else {
        const unsigned grid = grid_for(a.n, kAdamCtasPerSm);
        adam_fused_kernel<GK, OK, WD, false, 1><<<grid, kThreads, 0, stream>>>(
            a.p, a.m, a.v, a.g, a.p16, a.n, a.c, a.counters);
    }
    return cudaGetLastError();
}

template <int GK, int OK>
cudaError_t launch_adam_wd(const AdamLaunch& a, cudaStream_t stream) {
    return a.c.lr_wd != 0.0 ? launch_adam_typed<GK, OK, true>(a, stream)
                            : launch_adam_typed<GK, OK, false>(a, stream);
}

}  // namespace

cudaError_t launch_spin_ns(uint64_t ns, cudaStream_t stream) {
    if (ns == 0) return cudaSuccess;
    spin_kernel<<<1, 1, 0, stream>>>(ns);
    return cudaGetLastError();
}

cudaError_t launch_adam_fused(const AdamLaunch& a, cudaStream_t stream) {
    if (a.n == 0) return cudaSuccess;
    if (a.grad_kind == kF16 && a.out_kind == kF16) return launch_adam_wd<kF16, kF16>(a, stream);
    if (a.grad_kind == kF16 && a.out_kind == kBF16) return launch_adam_wd<kF16, kBF16>(a, stream);
    if (a.grad_kind == kBF16 && a.out_kind == kF16) return launch_adam_wd<kBF16, kF16>(a, stream);
    return launch_adam_wd<kBF16, kBF16>(a, stream);
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

}  // namespace tfb
