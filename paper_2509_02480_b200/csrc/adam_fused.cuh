// The fused update-phase kernel as a template, shared by the shipped launch
// path (adam_kernel.cu) and the tuning variants (adam_variants.cu).
//
// One HBM pass per subgroup replaces upscale_f16_to_f32 -> adam_step ->
// downscale_f32_to_f16 (reference scheduler.hpp:467, 479, 490): read P, m, v
// (fp32) and the 16-bit gradient, widen, bias-corrected Adam/AdamW in binary64
// (bit-exact with optimizer.hpp:91-108), write P, m, v and the 16-bit working
// params, and count non-finite gradients and narrowing overflows.
// 28 algorithmic bytes per parameter. Everything here has internal linkage
// (anonymous namespace): each including translation unit instantiates its own.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "kernels.hpp"
#include "launch_util.cuh"
#include "numerics.cuh"
#include "tma.cuh"

namespace tfb {
namespace {

using namespace detail;

// Gradient sources of one launch. GMODE 0: one 16-bit buffer (GK = F16 or
// BF16). GMODE 1: one fp32 buffer (GK = F32; the ZeRO-3 baseline flow that
// fetches fp32 gradients from storage). GMODE 2: the sum of n 16-bit buffers,
// e.g. the same subgroup's gradient contributions in every data-parallel
// peer's memory over NVLink: summed in fp32 in source order, rounded once to
// GK — the reduce-scatter fused into the update. NS > 0 fixes n at compile
// time (the 2/4/8-rank cases: unrolled loads, no per-source predicates);
// NS = 0 reads gs.n at run time.
struct GradSources {
    const void* src[kMaxGradSources];
    int n;
};

__device__ __forceinline__ uint2 pack_u16x4(const U16x4& h) {
    return make_uint2(static_cast<uint32_t>(h.x) | (static_cast<uint32_t>(h.y) << 16),
                      static_cast<uint32_t>(h.z) | (static_cast<uint32_t>(h.w) << 16));
}

// In-order fp32 sum of NS quads already loaded, rounded once to GK (the same
// rule as sum_quad16).
template <int GK, int NS>
__device__ __forceinline__ U16x4 sum16x4(const U16x4 (&x)[NS]) {
    float4 acc = make_float4(-0.f, -0.f, -0.f, -0.f);
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        acc.x = __fadd_rn(acc.x, widen16<GK>(x[s].x));
        acc.y = __fadd_rn(acc.y, widen16<GK>(x[s].y));
        acc.z = __fadd_rn(acc.z, widen16<GK>(x[s].z));
        acc.w = __fadd_rn(acc.w, widen16<GK>(x[s].w));
    }
    U16x4 h;
    h.x = narrow16<GK>(acc.x);
    h.y = narrow16<GK>(acc.y);
    h.z = narrow16<GK>(acc.z);
    h.w = narrow16<GK>(acc.w);
    return h;
}

// In-order fp32 sum of one quad over the sources, rounded once to GK.
template <int GK, int NS>
__device__ __forceinline__ U16x4 sum_quad16(const GradSources& gs, uint64_t q) {
    float4 acc = make_float4(-0.f, -0.f, -0.f, -0.f);  // -0 + x == x for every x: the sum starts at source 0
    auto add = [&](const U16x4& x) {
        acc.x = __fadd_rn(acc.x, widen16<GK>(x.x));
        acc.y = __fadd_rn(acc.y, widen16<GK>(x.y));
        acc.z = __fadd_rn(acc.z, widen16<GK>(x.z));
        acc.w = __fadd_rn(acc.w, widen16<GK>(x.w));
    };
    if constexpr (NS > 0) {
        U16x4 x[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s)  // all loads first: NS independent streams in flight
            x[s] = load_u16x4(reinterpret_cast<const uint16_t*>(gs.src[s]) + 4 * q);
#pragma unroll
        for (int s = 0; s < NS; ++s) add(x[s]);
    } else {
#pragma unroll
        for (int s = 0; s < kMaxGradSources; ++s)
            if (s < gs.n) add(load_u16x4(reinterpret_cast<const uint16_t*>(gs.src[s]) + 4 * q));
    }
    U16x4 h;
    h.x = narrow16<GK>(acc.x);
    h.y = narrow16<GK>(acc.y);
    h.z = narrow16<GK>(acc.z);
    h.w = narrow16<GK>(acc.w);
    return h;
}

// Register form of one gradient quad: 16-bit sources stay packed (2
// registers; a summed quad is held already rounded) and are widened at use;
// fp32 sources (GMODE 1) hold floats.
template <int GK, int GMODE, int NS>
struct GradReg {
    U16x4 h;
    template <bool COUNT = true>
    __device__ __forceinline__ void load(const GradSources& gs, uint64_t q, unsigned& nonfinite) {
        if constexpr (GMODE == 0)
            h = load_u16x4(reinterpret_cast<const uint16_t*>(gs.src[0]) + 4 * q);
        else
            h = sum_quad16<GK, NS>(gs, q);
        if constexpr (COUNT)
            nonfinite += nonfinite16<GK>(h.x) + nonfinite16<GK>(h.y) + nonfinite16<GK>(h.z) + nonfinite16<GK>(h.w);
    }
    __device__ __forceinline__ float get(int k) const {
        return widen16<GK>(k == 0 ? h.x : k == 1 ? h.y : k == 2 ? h.z : h.w);
    }
    // f16 straight to binary64 (one cvt.f64.f16 instead of widen + cvt.f64.f32)
    __device__ __forceinline__ double get64(int k) const {
        static_assert(GK == kF16, "get64: f16 gradients");
        const uint16_t x = k == 0 ? h.x : k == 1 ? h.y : k == 2 ? h.z : h.w;
        double d;
        asm("cvt.f64.f16 %0, %1;" : "=d"(d) : "h"(x));
        return d;
    }
};

template <int GK, int NS>
struct GradReg<GK, 1, NS> {
    float4 f;
    template <bool COUNT = true>
    __device__ __forceinline__ void load(const GradSources& gs, uint64_t q, unsigned& nonfinite) {
        f = __ldcs(reinterpret_cast<const float4*>(gs.src[0]) + q);
        nonfinite += !isfinite(f.x) + !isfinite(f.y) + !isfinite(f.z) + !isfinite(f.w);
    }
    __device__ __forceinline__ float get(int k) const { return k == 0 ? f.x : k == 1 ? f.y : k == 2 ? f.z : f.w; }
};

template <int GK, int GMODE>
__device__ __forceinline__ float load_grad1(const GradSources& gs, uint64_t i, unsigned& nonfinite) {
    if constexpr (GMODE == 1) {
        const float f = __ldcs(reinterpret_cast<const float*>(gs.src[0]) + i);
        nonfinite += !isfinite(f);
        return f;
    } else {
        uint16_t h;
        if constexpr (GMODE == 0) {
            h = __ldcs(reinterpret_cast<const uint16_t*>(gs.src[0]) + i);
        } else {
            float acc = -0.f;
#pragma unroll
            for (int s = 0; s < kMaxGradSources; ++s)
                if (s < gs.n) acc = __fadd_rn(acc, widen16<GK>(__ldcs(reinterpret_cast<const uint16_t*>(gs.src[s]) + i)));
            h = narrow16<GK>(acc);
        }
        nonfinite += nonfinite16<GK>(h);
        return widen16<GK>(h);
    }
}

// Where one launch reads and writes the fp32 state. In place (in == out) for
// the device ring and the HBM-resident path; out may instead be mapped pinned
// host memory, which fuses the D2H write-back into the kernel's epilogue.
struct StateIO {
    const float* p;
    const float* m;
    const float* v;
    float* po;
    float* mo;
    float* vo;
};

// VEC = true: P, m, v 16-byte aligned and the gradient / p16 streams 8-byte
// (16-bit) or 16-byte (fp32) aligned; the body walks quads (float4 / 4 x
// 16-bit) and the n % 4 tail is scalar. VEC = false: scalar everywhere (e.g.
// a contiguous P||m||v with P % 4 != 0). Loads and stores are explicit
// evict-first intrinsics, issued in program order per element, so in-place
// aliasing of in and out is well defined.
// DIVC selects the element math: 0 = div.rn quotients, 1 = constant-divisor
// quotients, 2 = verified fast path (numerics.cuh adam_element_fast), 3 =
// constant-divisor quotients with the quad's elements walked one at a time.
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// State-stream load / store forms (PF < 0, tuning variants 48-50): -1 keeps
// evict-first and asks L2 for 256-byte fetches (ld.global.cs.L2::256B), -2
// the same without evict-first (L1::no_allocate), -3 plain cached accesses.
// Otherwise evict-first __ldcs / __stcs (the shipped form).
template <int PF>
__device__ __forceinline__ float4 ld_state(const float4* p) {
    float4 r;
    if constexpr (PF == -1) {
        asm volatile("ld.global.cs.L2::256B.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    } else if constexpr (PF == -2) {
        asm volatile("ld.global.L1::no_allocate.L2::256B.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    } else if constexpr (PF == -3) {
        r = *p;
    } else {
        r = __ldcs(p);
    }
    return r;
}

template <int PF>
__device__ __forceinline__ void st_state(float4* p, float4 v) {
    if constexpr (PF == -3) *p = v;
    else __stcs(p, v);
}

// PF > 0: one thread per CTA asks the TMA unit to pull the CTA's chunk PF
// grid-stride iterations ahead into L2 (cp.async.bulk.prefetch), so more bytes
// are in flight than the registers of 32 warps per SM can hold.
// OPT (vector body, one 16-bit gradient source): bit 0 skips the per-element
// non-finite count of the gradient (the launch is behind a whole-phase check
// that found none: a device gate or a host verdict); bit 1 widens f16
// gradients straight to binary64.
constexpr int kOptVerified = 1;
constexpr int kOptF64Widen = 2;

template <int GK, int GMODE, int OK, bool WD, bool VEC, int UNROLL, int DIVC, int MINB, int NS = 0, int PF = 0,
          int OPT = 0>
__global__ void __launch_bounds__(kThreads, MINB)
    adam_fused_kernel(const StateIO io, const GradSources gs, uint16_t* __restrict__ p16, uint64_t n, AdamConsts c,
                      unsigned long long* __restrict__ counters, const unsigned long long* __restrict__ gate) {
    if (gate != nullptr && *gate != 0) return;  // the phase was rejected on this stream: no writes
    unsigned nonfinite = 0, overflow = 0;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;

    if constexpr (VEC) {
        const uint64_t nq = n / 4;
        const float4* p4 = reinterpret_cast<const float4*>(io.p);
        const float4* m4 = reinterpret_cast<const float4*>(io.m);
        const float4* v4 = reinterpret_cast<const float4*>(io.v);
        float4* po4 = reinterpret_cast<float4*>(io.po);
        float4* mo4 = reinterpret_cast<float4*>(io.mo);
        float4* vo4 = reinterpret_cast<float4*>(io.vo);
        for (uint64_t base = tid; base < nq; base += nthreads * UNROLL) {
            if constexpr (PF > 0) {
                if (threadIdx.x == 0) {
                    const uint64_t cq = base + static_cast<uint64_t>(PF) * UNROLL * nthreads;
                    if (cq < nq) {
                        const uint64_t nqc = min(static_cast<uint64_t>(blockDim.x) * UNROLL, nq - cq);
                        prefetch_l2(p4 + cq, static_cast<uint32_t>(16 * nqc));
                        prefetch_l2(m4 + cq, static_cast<uint32_t>(16 * nqc));
                        prefetch_l2(v4 + cq, static_cast<uint32_t>(16 * nqc));
                        if constexpr (GMODE == 0) {
                            const uint16_t* g = reinterpret_cast<const uint16_t*>(gs.src[0]) + 4 * cq;
                            const uint32_t gb = static_cast<uint32_t>(8 * nqc) & ~15u;
                            if ((reinterpret_cast<uintptr_t>(g) & 15u) == 0 && gb > 0) prefetch_l2(g, gb);
                        }
                    }
                }
            }
            float4 rp[UNROLL], rm[UNROLL], rv[UNROLL];
            GradReg<GK, GMODE, NS> rg[UNROLL];
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {  // all loads first: UNROLL quads in flight
                const uint64_t q = base + static_cast<uint64_t>(u) * nthreads;
                if (q < nq) {
                    rp[u] = ld_state<PF>(p4 + q);
                    rm[u] = ld_state<PF>(m4 + q);
                    rv[u] = ld_state<PF>(v4 + q);
                    rg[u].template load<(OPT & kOptVerified) == 0>(gs, q, nonfinite);
                }
            }
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const uint64_t q = base + static_cast<uint64_t>(u) * nthreads;
                if (q < nq) {
                    if constexpr (DIVC == 3) {
                        // one element at a time (no cross-element ILP, fewer
                        // live registers): rotate the quad through .x
                        float g4[4] = {rg[u].get(0), rg[u].get(1), rg[u].get(2), rg[u].get(3)};
                        float gx = g4[0], gy = g4[1], gz = g4[2], gw = g4[3];
#pragma unroll 1
                        for (int k = 0; k < 4; ++k) {
                            adam_math<WD, 1>(rp[u].x, rm[u].x, rv[u].x, gx, c);
                            const float tp = rp[u].x, tm = rm[u].x, tv = rv[u].x, tg = gx;
                            rp[u].x = rp[u].y; rp[u].y = rp[u].z; rp[u].z = rp[u].w; rp[u].w = tp;
                            rm[u].x = rm[u].y; rm[u].y = rm[u].z; rm[u].z = rm[u].w; rm[u].w = tm;
                            rv[u].x = rv[u].y; rv[u].y = rv[u].z; rv[u].z = rv[u].w; rv[u].w = tv;
                            gx = gy; gy = gz; gz = gw; gw = tg;
                        }
                    } else if constexpr ((OPT & kOptF64Widen) != 0) {
                        adam_math<WD, DIVC>(rp[u].x, rm[u].x, rv[u].x, rg[u].get64(0), c);
                        adam_math<WD, DIVC>(rp[u].y, rm[u].y, rv[u].y, rg[u].get64(1), c);
                        adam_math<WD, DIVC>(rp[u].z, rm[u].z, rv[u].z, rg[u].get64(2), c);
                        adam_math<WD, DIVC>(rp[u].w, rm[u].w, rv[u].w, rg[u].get64(3), c);
                    } else {
                        adam_math<WD, DIVC>(rp[u].x, rm[u].x, rv[u].x, rg[u].get(0), c);
                        adam_math<WD, DIVC>(rp[u].y, rm[u].y, rv[u].y, rg[u].get(1), c);
                        adam_math<WD, DIVC>(rp[u].z, rm[u].z, rv[u].z, rg[u].get(2), c);
                        adam_math<WD, DIVC>(rp[u].w, rm[u].w, rv[u].w, rg[u].get(3), c);
                    }
                    const uint2 h = narrow16_quad<OK>(rp[u], overflow);
                    st_state<PF>(po4 + q, rp[u]);
                    st_state<PF>(mo4 + q, rm[u]);
                    st_state<PF>(vo4 + q, rv[u]);
                    __stcs(reinterpret_cast<uint2*>(p16) + q, h);
                }
            }
        }
        const uint64_t i = nq * 4 + tid;  // scalar tail: n % 4 elements
        if (i < n) {
            float pf = __ldcs(io.p + i), mf = __ldcs(io.m + i), vf = __ldcs(io.v + i);
            const float gf = load_grad1<GK, GMODE>(gs, i, nonfinite);
            adam_math<WD, DIVC == 3 ? 1 : DIVC>(pf, mf, vf, gf, c);
            const uint16_t h = narrow16<OK>(pf);
            overflow += is_inf16<OK>(h);
            __stcs(io.po + i, pf);
            __stcs(io.mo + i, mf);
            __stcs(io.vo + i, vf);
            p16[i] = h;
        }
    } else {
        for (uint64_t i = tid; i < n; i += nthreads) {
            float pf = __ldcs(io.p + i), mf = __ldcs(io.m + i), vf = __ldcs(io.v + i);
            const float gf = load_grad1<GK, GMODE>(gs, i, nonfinite);
            adam_math<WD, DIVC == 3 ? 1 : DIVC>(pf, mf, vf, gf, c);
            const uint16_t h = narrow16<OK>(pf);
            overflow += is_inf16<OK>(h);
            __stcs(io.po + i, pf);
            __stcs(io.mo + i, mf);
            __stcs(io.vo + i, vf);
            p16[i] = h;
        }
    }
    if (counters != nullptr) {
        warp_count_add(counters + 0, nonfinite);
        warp_count_add(counters + 1, overflow);
    }
}

// One quad of the staged kernel: widen, update, narrow, store at quad index
// qi of the tile at (p, m, v, p16).
template <int GK, int OK, bool WD, bool CNT, int MATH>
__device__ __forceinline__ void staged_quad(float4 rp, float4 rm, float4 rv, uint2 graw, const AdamConsts& c,
                                            unsigned& nonfinite, unsigned& overflow, float* p, float* m, float* v,
                                            uint16_t* p16, int qi) {
    GradReg<GK, 0, 0> rg;
    rg.h.x = static_cast<uint16_t>(graw.x & 0xFFFFu);
    rg.h.y = static_cast<uint16_t>(graw.x >> 16);
    rg.h.z = static_cast<uint16_t>(graw.y & 0xFFFFu);
    rg.h.w = static_cast<uint16_t>(graw.y >> 16);
    if constexpr (CNT)
        nonfinite += nonfinite16<GK>(rg.h.x) + nonfinite16<GK>(rg.h.y) + nonfinite16<GK>(rg.h.z) +
                     nonfinite16<GK>(rg.h.w);
    if constexpr (GK == kF16) {
        adam_math<WD, MATH>(rp.x, rm.x, rv.x, rg.get64(0), c);
        adam_math<WD, MATH>(rp.y, rm.y, rv.y, rg.get64(1), c);
        adam_math<WD, MATH>(rp.z, rm.z, rv.z, rg.get64(2), c);
        adam_math<WD, MATH>(rp.w, rm.w, rv.w, rg.get64(3), c);
    } else {
        adam_math<WD, MATH>(rp.x, rm.x, rv.x, rg.get(0), c);
        adam_math<WD, MATH>(rp.y, rm.y, rv.y, rg.get(1), c);
        adam_math<WD, MATH>(rp.z, rm.z, rv.z, rg.get(2), c);
        adam_math<WD, MATH>(rp.w, rm.w, rv.w, rg.get(3), c);
    }
    const uint2 h = narrow16_quad<OK>(rp, overflow);
    __stcs(reinterpret_cast<float4*>(p) + qi, rp);
    __stcs(reinterpret_cast<float4*>(m) + qi, rm);
    __stcs(reinterpret_cast<float4*>(v) + qi, rv);
    __stcs(reinterpret_cast<uint2*>(p16) + qi, h);
}

// ---------------------------------------------------------------------------
// Staged form (the shipped path for one 16-bit gradient source): one elected
// thread per CTA keeps S-1 tiles of P, m, v and g in flight into a ring of
// shared-memory stages with 1D bulk copies (cp.async.bulk on the TMA unit,
// completion on an mbarrier per stage); every warp computes its quads of the
// current tile from shared memory and stores the results straight to global
// memory. The bytes in flight per SM (MINB CTAs x (S-1) x 14 B x T) do not
// depend on how long the binary64 chain of the current quad takes, so the
// kernel keeps HBM busy when the power cap lowers the SM clock (the register
// kernel's loads are only in flight between two quads' math). Tile T =
// 4 x NT params (one quad per thread: 2048 at the shipped NT = 512); one CTA
// barrier per tile retires a stage
// before it is refilled. The same element math, bit for bit.
// NS > 0: the gradient is the in-order fp32 sum of NS 16-bit sources (the
// peers' contributions, NVLink-mapped), each staged by its own bulk copy per
// tile and summed from shared memory, rounded once to GK (sum_quad16's rule).
template <int GK, int OK, bool WD, int S, bool CNT, int MINB, int MATH = 1, int Q = 1, int PFL2 = 0, int NS = 0,
          int NT = kThreads>
__global__ void __launch_bounds__(NT, MINB)
    adam_staged_kernel(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v, const GradSources gs,
                       uint16_t* __restrict__ p16, uint64_t n, AdamConsts c,
                       unsigned long long* __restrict__ counters, const unsigned long long* __restrict__ gate) {
    if (gate != nullptr && *gate != 0) return;  // the phase was rejected on this stream: no writes
    constexpr int T = 4 * NT * Q;  // Q quads per thread per tile
    constexpr int G = NS > 0 ? NS : 1;   // gradient tiles per stage
    const uint16_t* __restrict__ g = static_cast<const uint16_t*>(gs.src[0]);
    const uint64_t ntiles = n / T;
    extern __shared__ __align__(128) unsigned char smem[];
    float* sp = reinterpret_cast<float*>(smem);
    float* sm = sp + S * T;
    float* sv = sm + S * T;
    uint16_t* sg = reinterpret_cast<uint16_t*>(sv + S * T);
    uint64_t* full = reinterpret_cast<uint64_t*>(sg + S * G * T);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t mine = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    auto issue = [&](uint64_t k) {
        const int s = static_cast<int>(k % S);
        const uint64_t off = (blockIdx.x + k * gridDim.x) * static_cast<uint64_t>(T);
        mbar_arrive_expect_tx(&full[s], (12u + 2u * G) * T);
        bulk_load(sp + s * T, p + off, 4u * T, &full[s]);
        bulk_load(sm + s * T, m + off, 4u * T, &full[s]);
        bulk_load(sv + s * T, v + off, 4u * T, &full[s]);
#pragma unroll
        for (int j = 0; j < G; ++j)
            bulk_load(sg + (s * G + j) * T, static_cast<const uint16_t*>(gs.src[j]) + off, 2u * T, &full[s]);
    };
    if (threadIdx.x == 0)
        for (uint64_t k = 0; k + 1 < static_cast<uint64_t>(S) && k < mine; ++k) issue(k);
    unsigned nonfinite = 0, overflow = 0;
    const int qi = threadIdx.x;
    for (uint64_t k = 0; k < mine; ++k) {
        if (threadIdx.x == 0 && k + S - 1 < mine) issue(k + S - 1);  // into the stage tile k-1 released
        if constexpr (PFL2 > 0) {  // tuning: tile k + S - 1 + PFL2 pulled into L2 ahead of its bulk load
            if (threadIdx.x == 0 && k + S - 1 + PFL2 < mine) {
                const uint64_t po = (blockIdx.x + (k + S - 1 + PFL2) * gridDim.x) * static_cast<uint64_t>(T);
                prefetch_l2(p + po, 4u * T);
                prefetch_l2(m + po, 4u * T);
                prefetch_l2(v + po, 4u * T);
                prefetch_l2(g + po, 2u * T);
            }
        }
        const int s = static_cast<int>(k % S);
        mbar_wait(&full[s], static_cast<uint32_t>(k / S) & 1u);
        const uint64_t off = (blockIdx.x + k * gridDim.x) * static_cast<uint64_t>(T);
#pragma unroll 1
        for (int qq = 0; qq < Q; ++qq) {
            const int qj = qi + qq * NT;
            const float4 rp = reinterpret_cast<const float4*>(sp + s * T)[qj];
            const float4 rm = reinterpret_cast<const float4*>(sm + s * T)[qj];
            const float4 rv = reinterpret_cast<const float4*>(sv + s * T)[qj];
            uint2 graw;
            if constexpr (NS == 0) {
                graw = reinterpret_cast<const uint2*>(sg + s * T)[qj];
            } else {
                U16x4 x[NS];
#pragma unroll
                for (int j = 0; j < NS; ++j) {
                    const uint2 r = reinterpret_cast<const uint2*>(sg + (s * G + j) * T)[qj];
                    x[j] = U16x4{static_cast<uint16_t>(r.x & 0xFFFFu), static_cast<uint16_t>(r.x >> 16),
                                 static_cast<uint16_t>(r.y & 0xFFFFu), static_cast<uint16_t>(r.y >> 16)};
                }
                graw = pack_u16x4(sum16x4<GK, NS>(x));
            }
            staged_quad<GK, OK, WD, CNT, MATH>(rp, rm, rv, graw, c, nonfinite, overflow, p + off, m + off, v + off,
                                               p16 + off, qj);
        }
        __syncthreads();  // stage s retired: it is refilled at iteration k + 1
    }
    // The n % T tail (fewer than T params, whole quads then scalars) from
    // global memory, by the last CTA.
    if (blockIdx.x == gridDim.x - 1) {
        const uint64_t done = ntiles * T;
        const uint64_t nq = (n - done) / 4;
        for (uint64_t j = threadIdx.x; j < nq; j += NT) {
            const uint64_t q = done / 4 + j;
            const float4 rp = __ldcs(reinterpret_cast<const float4*>(p) + q);
            const float4 rm = __ldcs(reinterpret_cast<const float4*>(m) + q);
            const float4 rv = __ldcs(reinterpret_cast<const float4*>(v) + q);
            uint2 graw;
            if constexpr (NS == 0) graw = __ldcs(reinterpret_cast<const uint2*>(g) + q);
            else graw = pack_u16x4(sum_quad16<GK, NS>(gs, q));
            staged_quad<GK, OK, WD, CNT, MATH>(rp, rm, rv, graw, c, nonfinite, overflow, p + done, m + done,
                                               v + done, p16 + done, static_cast<int>(j));
        }
        const uint64_t i = done + 4 * nq + threadIdx.x;
        if (i < n) {
            float pf = __ldcs(p + i), mf = __ldcs(m + i), vf = __ldcs(v + i);
            uint16_t gh;
            if constexpr (NS == 0) {
                gh = __ldcs(g + i);
            } else {
                float acc = -0.f;  // -0 + x == x: the sum starts at source 0
#pragma unroll
                for (int j = 0; j < NS; ++j)
                    acc = __fadd_rn(acc, widen16<GK>(__ldcs(static_cast<const uint16_t*>(gs.src[j]) + i)));
                gh = narrow16<GK>(acc);
            }
            if constexpr (CNT) nonfinite += nonfinite16<GK>(gh);
            adam_math<WD, 1>(pf, mf, vf, widen16<GK>(gh), c);
            const uint16_t h = narrow16<OK>(pf);
            overflow += is_inf16<OK>(h);
            __stcs(p + i, pf);
            __stcs(m + i, mf);
            __stcs(v + i, vf);
            p16[i] = h;
        }
    }
    if (counters != nullptr) {
        if constexpr (CNT) warp_count_add(counters + 0, nonfinite);
        warp_count_add(counters + 1, overflow);
    }
}


template <int UNROLL, int DIVC, int MINB, int PF = 0, int OPT = 0>
struct Cfg {
    static constexpr int kUnroll = UNROLL;
    static constexpr int kDivc = DIVC;
    static constexpr int kMinBlocks = MINB;
    static constexpr int kPrefetch = PF;
    static constexpr int kOpt = OPT;
};

GradSources sources_of(const AdamLaunch& a) {
    GradSources gs{};
    if (a.n_peers > 0) {
        for (int s = 0; s < a.n_peers; ++s) gs.src[s] = a.peers[s];
        gs.n = a.n_peers;
    } else {
        gs.src[0] = a.g;
        gs.n = 1;
    }
    return gs;
}

StateIO state_io(const AdamLaunch& a) {
    return StateIO{a.p, a.m, a.v, a.p_out ? a.p_out : a.p, a.m_out ? a.m_out : a.m, a.v_out ? a.v_out : a.v};
}

bool is_vec(const AdamLaunch& a) {
    const StateIO io = state_io(a);
    const uintptr_t state = reinterpret_cast<uintptr_t>(io.p) | reinterpret_cast<uintptr_t>(io.m) |
                            reinterpret_cast<uintptr_t>(io.v) | reinterpret_cast<uintptr_t>(io.po) |
                            reinterpret_cast<uintptr_t>(io.mo) | reinterpret_cast<uintptr_t>(io.vo);
    uintptr_t grads = 0;
    const GradSources gs = sources_of(a);
    for (int s = 0; s < gs.n; ++s) grads |= reinterpret_cast<uintptr_t>(gs.src[s]);
    const uintptr_t galign = a.grad_kind == kF32 ? 15u : 7u;
    return (state & 15u) == 0 && (grads & galign) == 0 && (reinterpret_cast<uintptr_t>(a.p16) & 7u) == 0;
}

template <int GK, int GMODE, int OK, bool WD, class C, int NS = 0>
cudaError_t launch_cfg(const AdamLaunch& a, cudaStream_t stream) {
    constexpr int U = C::kUnroll;
    constexpr int B = C::kMinBlocks;
    const GradSources gs = sources_of(a);
    if (is_vec(a)) {
        const unsigned grid = grid_for((a.n / 4 + U - 1) / U, B);
        adam_fused_kernel<GK, GMODE, OK, WD, true, U, C::kDivc, B, NS, C::kPrefetch, C::kOpt>
            <<<grid, kThreads, 0, stream>>>(state_io(a), gs, a.p16, a.n, a.c, a.counters, a.gate);
    } else {
        const unsigned grid = grid_for(a.n, B);
        adam_fused_kernel<GK, GMODE, OK, WD, false, 1, C::kDivc, B>
            <<<grid, kThreads, 0, stream>>>(state_io(a), gs, a.p16, a.n, a.c, a.counters, a.gate);
    }
    return cudaGetLastError();
}

template <int GK, int GMODE, int OK, class C, int NS = 0>
cudaError_t launch_wd(const AdamLaunch& a, cudaStream_t stream) {
    return a.c.lr_wd != 0.0 ? launch_cfg<GK, GMODE, OK, true, C, NS>(a, stream)
                            : launch_cfg<GK, GMODE, OK, false, C, NS>(a, stream);
}

// Summed sources: a compile-time source count (unrolled loads, no
// per-source predicates) measured at 0.92-0.93 of the HBM roofline for 1, 2
// and 4 sources against 0.75-0.77 for the run-time loop
// (profiles/multi_sweep_r1.json).
template <int GK, int OK, class C>
cudaError_t launch_sum(const AdamLaunch& a, cudaStream_t stream) {
    switch (a.n_peers) {
        case 1: return launch_wd<GK, 2, OK, C, 1>(a, stream);
        case 2: return launch_wd<GK, 2, OK, C, 2>(a, stream);
        case 3: return launch_wd<GK, 2, OK, C, 3>(a, stream);
        case 4: return launch_wd<GK, 2, OK, C, 4>(a, stream);
        case 5: return launch_wd<GK, 2, OK, C, 5>(a, stream);
        case 6: return launch_wd<GK, 2, OK, C, 6>(a, stream);
        case 7: return launch_wd<GK, 2, OK, C, 7>(a, stream);
        case 8: return launch_wd<GK, 2, OK, C, 8>(a, stream);
        default: return cudaErrorInvalidValue;
    }
}

template <class C>
cudaError_t launch_dtypes(const AdamLaunch& a, cudaStream_t stream) {
    if (a.out_kind != kF16 && a.out_kind != kBF16) return cudaErrorInvalidValue;
    if (a.n_peers > 0) {  // fused multi-source reduction: 16-bit sources, same kind in and out
        if (a.n_peers > kMaxGradSources || a.grad_kind == kF32) return cudaErrorInvalidValue;
        if (a.grad_kind == kF16)
            return a.out_kind == kF16 ? launch_sum<kF16, kF16, C>(a, stream) : launch_sum<kF16, kBF16, C>(a, stream);
        return a.out_kind == kF16 ? launch_sum<kBF16, kF16, C>(a, stream) : launch_sum<kBF16, kBF16, C>(a, stream);
    }
    if (a.grad_kind == kF32)
        return a.out_kind == kF16 ? launch_wd<kF32, 1, kF16, C>(a, stream) : launch_wd<kF32, 1, kBF16, C>(a, stream);
    if (a.grad_kind == kF16 && a.out_kind == kF16) return launch_wd<kF16, 0, kF16, C>(a, stream);
    if (a.grad_kind == kF16 && a.out_kind == kBF16) return launch_wd<kF16, 0, kBF16, C>(a, stream);
    if (a.grad_kind == kBF16 && a.out_kind == kF16) return launch_wd<kBF16, 0, kF16, C>(a, stream);
    return launch_wd<kBF16, 0, kBF16, C>(a, stream);
}


// One launch of the staged kernel (its last CTA takes the n % 1024 tail).
// NS > 0: the fused multi-source form, a.n_peers == NS. Returns
// cudaErrorNotSupported, launching nothing, when the launch does not fit the
// staged form (fp32 gradients, a source count other than NS, separate
// outputs, 16-byte misalignment, fewer than one tile); the caller then
// launches the register kernel.
template <int S, int MINB, int MATH = 1, int Q = 1, int PFL2 = 0, int NS = 0, int NT = kThreads>
cudaError_t launch_staged(const AdamLaunch& a, cudaStream_t stream) {
    constexpr uint64_t T = 4 * NT * Q;
    constexpr int G = NS > 0 ? NS : 1;
    const GradSources gs = sources_of(a);
    uintptr_t addr = reinterpret_cast<uintptr_t>(a.p) | reinterpret_cast<uintptr_t>(a.m) |
                     reinterpret_cast<uintptr_t>(a.v) | reinterpret_cast<uintptr_t>(a.p16);
    for (int j = 0; j < gs.n; ++j) addr |= reinterpret_cast<uintptr_t>(gs.src[j]);
    if (a.n_peers != NS || a.p_out || a.m_out || a.v_out || (a.grad_kind != kF16 && a.grad_kind != kBF16) ||
        (a.out_kind != kF16 && a.out_kind != kBF16) || (addr & 15u) != 0 || a.n < T)
        return cudaErrorNotSupported;
    const uint64_t ntiles = a.n / T;
    // a summed gradient is only known after the sum: counted in-kernel
    const bool cnt = NS > 0 || !(a.grads_verified || a.gate != nullptr);
    const bool wd = a.c.lr_wd != 0.0;
    using K = void (*)(float*, float*, float*, const GradSources, uint16_t*, uint64_t, AdamConsts,
                       unsigned long long*, const unsigned long long*);
    K kern = nullptr;
    auto pick = [&](auto gk, auto ok) {
        constexpr int GKc = decltype(gk)::value, OKc = decltype(ok)::value;
        if constexpr (NS > 0) {
            kern = wd ? adam_staged_kernel<GKc, OKc, true, S, true, MINB, MATH, Q, PFL2, NS, NT>
                      : adam_staged_kernel<GKc, OKc, false, S, true, MINB, MATH, Q, PFL2, NS, NT>;
        } else if (cnt) {
            kern = wd ? adam_staged_kernel<GKc, OKc, true, S, true, MINB, MATH, Q, PFL2, 0, NT>
                      : adam_staged_kernel<GKc, OKc, false, S, true, MINB, MATH, Q, PFL2, 0, NT>;
        } else {
            kern = wd ? adam_staged_kernel<GKc, OKc, true, S, false, MINB, MATH, Q, PFL2, 0, NT>
                      : adam_staged_kernel<GKc, OKc, false, S, false, MINB, MATH, Q, PFL2, 0, NT>;
        }
    };
    using F = std::integral_constant<int, kF16>;
    using B = std::integral_constant<int, kBF16>;
    if (a.grad_kind == kF16) a.out_kind == kF16 ? pick(F{}, F{}) : pick(F{}, B{});
    else a.out_kind == kF16 ? pick(B{}, F{}) : pick(B{}, B{});
    constexpr size_t smem = static_cast<size_t>(S) * T * (12 + 2 * G) + S * sizeof(uint64_t);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(ntiles, static_cast<uint64_t>(num_sms()) * MINB));
    kern<<<grid, NT, smem, stream>>>(a.p, a.m, a.v, gs, a.p16, a.n, a.c, a.counters, a.gate);
    return cudaGetLastError();
}

}  // namespace
}  // namespace tfb
