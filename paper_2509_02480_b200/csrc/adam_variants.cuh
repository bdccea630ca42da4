// Tuning variants of the fused Adam kernel, for scripts/kernel_sweep.py and
// the bit-parity test that checks every variant against the others
// (tests/test_kernel_parity.py::test_kernel_variants_bitwise). None is
// shipped; DESIGN.md §5.1 records what each one measured:
//   1-11, 18-20, 24-31  launch shapes / element math of the register kernel
//   12-15               TMA producer warp + consumer warps (cp.async.bulk, mbarriers)
//   16-17               cp.async double buffer
//   21-23               scalar elements at higher occupancy
//   32-37               TMA multistage pipeline, every warp computing
//   38-40               per-warp TMA pipelines (no CTA barrier)
//   41-43               software-pipelined register kernel (next quad's loads before the math)
//   44-46               verified fast path, second form (numerics.cuh adam_element_fast2)
//   47                  in-range correctly rounded sqrt / division without the special-operand checks
//   48-50               state-stream cache hints: L2::256B fetches (evict-first or not), plain cached
//   51-53               OPT bits of the shipped form: no per-element gradient non-finite count behind a
//                       whole-phase check (53), f16 gradients widened straight to binary64 (52), both (51)
//   54-57               the staged kernel (adam_fused.cuh adam_staged_kernel): S = 2 / 4 CTAs counting (54)
//                       and verified (55), S = 3 / 4 CTAs (56), S = 3 / 3 CTAs (57); 55 with variant 47's
//                       in-range sqrt / division (58); 3 stages / 4 CTAs (59), 2-quad tiles: 2 stages /
//                       3 CTAs (60), 3 stages / 2 CTAs (61), 4 stages / 2 CTAs (62); 4-quad tiles at 1 CTA
//                       per SM: 3 stages (63), 2 stages (64); the shipped shape with an L2 bulk prefetch 1 (65)
//                       or 2 (66) tiles beyond its look-ahead
//   68-71               the staged kernel with larger CTAs: 320 threads x 3 (68), 384 x 2 (69), 512 x 2 with
//                       2 (70) or 3 (71) stages — tiles of 4 x threads params
//   67                  tile-interleaved state layout ([P | m | v] per 1024-param tile; timing only, its bits
//                       land in the interleaved positions — scripts/layout_probe.py, not the bitwise test)
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "adam_fused.cuh"
#include "tma.cuh"

namespace tfb {
namespace {

// ---------------------------------------------------------------------------
// TMA-staged variant: one producer warp streams tiles of P, m, v and g into a
// ring of shared-memory stages with 1D bulk copies (cp.async.bulk, completion
// counted on an mbarrier), the consumer warps compute from shared memory and
// store straight to global. Memory parallelism comes from the stage ring
// (S x 14 KiB per CTA in flight) instead of registers.

constexpr int kTmaConsumerWarps = 8;

template <int T, int S, bool WD, int MINB>
__global__ void __launch_bounds__((kTmaConsumerWarps + 1) * 32, MINB)
    adam_tma_kernel(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                    const uint16_t* __restrict__ g, uint16_t* __restrict__ p16, uint64_t ntiles, AdamConsts c,
                    unsigned long long* __restrict__ counters) {
    extern __shared__ __align__(128) unsigned char smem[];
    float* sp = reinterpret_cast<float*>(smem);
    float* sm = sp + S * T;
    float* sv = sm + S * T;
    uint16_t* sg = reinterpret_cast<uint16_t*>(sv + S * T);
    uint64_t* full = reinterpret_cast<uint64_t*>(sg + S * T);
    uint64_t* empty = full + S;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kTmaConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kTmaConsumerWarps) {  // producer warp: one lane issues the bulk copies
        if (lane == 0) {
            uint64_t k = 0;
            for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
                const int s = static_cast<int>(k % S);
                const uint32_t round = static_cast<uint32_t>(k / S);
                if (k >= static_cast<uint64_t>(S)) mbar_wait(&empty[s], (round - 1) & 1u);
                mbar_arrive_expect_tx(&full[s], 14u * T);
                const uint64_t off = tile * T;
                bulk_load(sp + s * T, p + off, 4u * T, &full[s]);
                bulk_load(sm + s * T, m + off, 4u * T, &full[s]);
                bulk_load(sv + s * T, v + off, 4u * T, &full[s]);
                bulk_load(sg + s * T, g + off, 2u * T, &full[s]);
            }
        }
        return;
    }
    unsigned nonfinite = 0, overflow = 0;
    uint64_t k = 0;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
        const int s = static_cast<int>(k % S);
        mbar_wait(&full[s], static_cast<uint32_t>(k / S) & 1u);
        const uint64_t off = tile * T;
        const float4* tp = reinterpret_cast<const float4*>(sp + s * T);
        const float4* tm = reinterpret_cast<const float4*>(sm + s * T);
        const float4* tv = reinterpret_cast<const float4*>(sv + s * T);
        const uint2* tg = reinterpret_cast<const uint2*>(sg + s * T);
#pragma unroll 1
        for (int qi = threadIdx.x; qi < T / 4; qi += kTmaConsumerWarps * 32) {
            float4 rp = tp[qi], rm = tm[qi], rv = tv[qi];
            const uint2 graw = tg[qi];
            U16x4 gh;
            gh.x = static_cast<uint16_t>(graw.x & 0xFFFFu);
            gh.y = static_cast<uint16_t>(graw.x >> 16);
            gh.z = static_cast<uint16_t>(graw.y & 0xFFFFu);
            gh.w = static_cast<uint16_t>(graw.y >> 16);
            nonfinite += nonfinite16<kF16>(gh.x) + nonfinite16<kF16>(gh.y) + nonfinite16<kF16>(gh.z) +
                         nonfinite16<kF16>(gh.w);
            adam_element<WD, true>(rp.x, rm.x, rv.x, widen16<kF16>(gh.x), c);
            adam_element<WD, true>(rp.y, rm.y, rv.y, widen16<kF16>(gh.y), c);
            adam_element<WD, true>(rp.z, rm.z, rv.z, widen16<kF16>(gh.z), c);
            adam_element<WD, true>(rp.w, rm.w, rv.w, widen16<kF16>(gh.w), c);
            U16x4 h;
            h.x = narrow16<kF16>(rp.x);
            h.y = narrow16<kF16>(rp.y);
            h.z = narrow16<kF16>(rp.z);
            h.w = narrow16<kF16>(rp.w);
            overflow += is_inf16<kF16>(h.x) + is_inf16<kF16>(h.y) + is_inf16<kF16>(h.z) + is_inf16<kF16>(h.w);
            __stcs(reinterpret_cast<float4*>(p + off) + qi, rp);
            __stcs(reinterpret_cast<float4*>(m + off) + qi, rm);
            __stcs(reinterpret_cast<float4*>(v + off) + qi, rv);
            store_u16x4(p16 + off + 4 * qi, h);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (counters != nullptr) {
        warp_count_add(counters + 0, nonfinite);
        warp_count_add(counters + 1, overflow);
    }
}

template <int T, int S, int MINB>
cudaError_t launch_tma(const AdamLaunch& a, cudaStream_t stream) {
    const bool aligned = ((reinterpret_cast<uintptr_t>(a.p) | reinterpret_cast<uintptr_t>(a.m) |
                           reinterpret_cast<uintptr_t>(a.v) | reinterpret_cast<uintptr_t>(a.g) |
                           reinterpret_cast<uintptr_t>(a.p16)) & 15u) == 0;
    if (!aligned || a.n_peers > 0 || a.p_out || a.grad_kind != kF16 || a.out_kind != kF16)
        return cudaErrorInvalidValue;
    const uint64_t ntiles = a.n / T;
    constexpr size_t smem = static_cast<size_t>(S) * T * 14 + 2 * S * sizeof(uint64_t);
    if (ntiles > 0) {
        auto kern = a.c.lr_wd != 0.0 ? adam_tma_kernel<T, S, true, MINB> : adam_tma_kernel<T, S, false, MINB>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(ntiles, static_cast<uint64_t>(num_sms()) * MINB));
        kern<<<grid, (kTmaConsumerWarps + 1) * 32, smem, stream>>>(a.p, a.m, a.v, static_cast<const uint16_t*>(a.g),
                                                                   a.p16, ntiles, a.c, a.counters);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const uint64_t done = ntiles * T;
    if (done == a.n) return cudaSuccess;
    AdamLaunch tail = a;  // the n % T remainder through the register-streaming kernel
    tail.p += done;
    tail.m += done;
    tail.v += done;
    tail.g = static_cast<const uint16_t*>(a.g) + done;
    tail.p16 += done;
    tail.n = a.n - done;
    return launch_dtypes<Cfg<1, true, 4>>(tail, stream);
}

// ---------------------------------------------------------------------------
// TMA multistage pipeline without warp specialisation: every warp computes;
// one elected thread keeps S-1 tiles (1024 params, 14 KiB) of P, m, v, g in
// flight into a shared-memory ring with cp.async.bulk, so the bytes in flight
// per SM (4 CTAs x (S-1) x 14 KiB) no longer depend on how long the FP64
// chain of the current quad takes. One __syncthreads per tile retires a stage
// before it is refilled.
// REL = true: warps release a stage through a per-stage mbarrier (one
// arrival per warp) instead of a CTA barrier, so only the issuing warp ever
// waits for the slowest warp of a tile.
template <int S, bool WD, int MINB, bool REL = false>
__global__ void __launch_bounds__(kThreads, MINB)
    adam_tma_pipe_kernel(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                         const uint16_t* __restrict__ g, uint16_t* __restrict__ p16, uint64_t ntiles, AdamConsts c,
                         unsigned long long* __restrict__ counters) {
    constexpr int T = 4 * kThreads;  // one quad per thread per tile
    extern __shared__ __align__(128) unsigned char smem[];
    float* sp = reinterpret_cast<float*>(smem);
    float* sm = sp + S * T;
    float* sv = sm + S * T;
    uint16_t* sg = reinterpret_cast<uint16_t*>(sv + S * T);
    uint64_t* full = reinterpret_cast<uint64_t*>(sg + S * T);
    uint64_t* empty = full + S;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            if constexpr (REL) mbar_init(&empty[s], kThreads / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t mine = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    auto issue = [&](uint64_t k) {
        const int s = static_cast<int>(k % S);
        const uint64_t off = (blockIdx.x + k * gridDim.x) * static_cast<uint64_t>(T);
        mbar_arrive_expect_tx(&full[s], 14u * T);
        bulk_load(sp + s * T, p + off, 4u * T, &full[s]);
        bulk_load(sm + s * T, m + off, 4u * T, &full[s]);
        bulk_load(sv + s * T, v + off, 4u * T, &full[s]);
        bulk_load(sg + s * T, g + off, 2u * T, &full[s]);
    };
    if (threadIdx.x == 0)
        for (uint64_t k = 0; k + 1 < static_cast<uint64_t>(S) && k < mine; ++k) issue(k);
    unsigned nonfinite = 0, overflow = 0;
    const int qi = threadIdx.x;
    for (uint64_t k = 0; k < mine; ++k) {
        if (threadIdx.x == 0 && k + S - 1 < mine) {  // refills the stage of tile k-1
            if constexpr (REL)
                if (k > 0) mbar_wait(&empty[(k - 1) % S], static_cast<uint32_t>((k - 1) / S) & 1u);
            issue(k + S - 1);
        }
        const int s = static_cast<int>(k % S);
        mbar_wait(&full[s], static_cast<uint32_t>(k / S) & 1u);
        const uint64_t off = (blockIdx.x + k * gridDim.x) * static_cast<uint64_t>(T);
        float4 rp = reinterpret_cast<const float4*>(sp + s * T)[qi];
        float4 rm = reinterpret_cast<const float4*>(sm + s * T)[qi];
        float4 rv = reinterpret_cast<const float4*>(sv + s * T)[qi];
        const uint2 graw = reinterpret_cast<const uint2*>(sg + s * T)[qi];
        U16x4 gh;
        gh.x = static_cast<uint16_t>(graw.x & 0xFFFFu);
        gh.y = static_cast<uint16_t>(graw.x >> 16);
        gh.z = static_cast<uint16_t>(graw.y & 0xFFFFu);
        gh.w = static_cast<uint16_t>(graw.y >> 16);
        nonfinite += nonfinite16<kF16>(gh.x) + nonfinite16<kF16>(gh.y) + nonfinite16<kF16>(gh.z) +
                     nonfinite16<kF16>(gh.w);
        adam_element<WD, true>(rp.x, rm.x, rv.x, widen16<kF16>(gh.x), c);
        adam_element<WD, true>(rp.y, rm.y, rv.y, widen16<kF16>(gh.y), c);
        adam_element<WD, true>(rp.z, rm.z, rv.z, widen16<kF16>(gh.z), c);
        adam_element<WD, true>(rp.w, rm.w, rv.w, widen16<kF16>(gh.w), c);
        U16x4 h;
        h.x = narrow16<kF16>(rp.x);
        h.y = narrow16<kF16>(rp.y);
        h.z = narrow16<kF16>(rp.z);
        h.w = narrow16<kF16>(rp.w);
        overflow += is_inf16<kF16>(h.x) + is_inf16<kF16>(h.y) + is_inf16<kF16>(h.z) + is_inf16<kF16>(h.w);
        __stcs(reinterpret_cast<float4*>(p + off) + qi, rp);
        __stcs(reinterpret_cast<float4*>(m + off) + qi, rm);
        __stcs(reinterpret_cast<float4*>(v + off) + qi, rv);
        store_u16x4(p16 + off + 4 * qi, h);
        if constexpr (REL) {
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
        } else {
            __syncthreads();  // stage s retired: it is refilled at iteration k + 1
        }
    }
    if (counters != nullptr) {
        warp_count_add(counters + 0, nonfinite);
        warp_count_add(counters + 1, overflow);
    }
}

template <int S, int MINB, bool REL = false>
cudaError_t launch_tma_pipe(const AdamLaunch& a, cudaStream_t stream) {
    constexpr int T = 4 * kThreads;
    const bool aligned = ((reinterpret_cast<uintptr_t>(a.p) | reinterpret_cast<uintptr_t>(a.m) |
                           reinterpret_cast<uintptr_t>(a.v) | reinterpret_cast<uintptr_t>(a.g) |
                           reinterpret_cast<uintptr_t>(a.p16)) & 15u) == 0;
    if (!aligned || a.n_peers > 0 || a.p_out || a.grad_kind != kF16 || a.out_kind != kF16)
        return cudaErrorInvalidValue;
    const uint64_t ntiles = a.n / T;
    constexpr size_t smem = static_cast<size_t>(S) * T * 14 + 2 * S * sizeof(uint64_t);
    if (ntiles > 0) {
        auto kern = a.c.lr_wd != 0.0 ? adam_tma_pipe_kernel<S, true, MINB, REL>
                                     : adam_tma_pipe_kernel<S, false, MINB, REL>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(ntiles, static_cast<uint64_t>(num_sms()) * MINB));
        kern<<<grid, kThreads, smem, stream>>>(a.p, a.m, a.v, static_cast<const uint16_t*>(a.g), a.p16, ntiles, a.c,
                                               a.counters);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const uint64_t done = ntiles * T;
    if (done == a.n) return cudaSuccess;
    AdamLaunch tail = a;  // the n % T remainder through the register-streaming kernel
    tail.p += done;
    tail.m += done;
    tail.v += done;
    tail.g = static_cast<const uint16_t*>(a.g) + done;
    tail.p16 += done;
    tail.n = a.n - done;
    return launch_dtypes<Cfg<1, true, 4>>(tail, stream);
}

// ---------------------------------------------------------------------------
// Per-warp TMA pipelines: every warp owns a ring of S stages of 128 params
// (one quad per lane; 1.75 KiB) and its own mbarriers. Lane 0 keeps S-1 of
// the warp's tiles in flight with cp.async.bulk; the warp consumes a stage,
// __syncwarp, and lane 0 refills that same stage. No CTA-wide barrier: warps
// never wait for one another, and the bytes in flight per SM (32 warps x
// (S-1) x 1.75 KiB) do not depend on how long the FP64 chain takes.
template <int S, bool WD, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    adam_warp_pipe_kernel(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                          const uint16_t* __restrict__ g, uint16_t* __restrict__ p16, uint64_t ntiles, AdamConsts c,
                          unsigned long long* __restrict__ counters) {
    constexpr int T = 128;                  // params per warp tile
    constexpr int kStage = T * 14;          // bytes per stage
    constexpr int kWarps = kThreads / 32;
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    unsigned char* mine_smem = smem + static_cast<size_t>(warp) * S * kStage;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(kWarps) * S * kStage) + warp * S;
    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // Warp-global tile index: tile j of this warp is gw + j * (grid warps).
    const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kWarps + warp;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kWarps;
    const uint64_t mine = ntiles > gw ? (ntiles - 1 - gw) / stride + 1 : 0;
    auto stage_p = [&](int s) { return reinterpret_cast<float*>(mine_smem + s * kStage); };
    auto issue = [&](uint64_t k) {
        const int s = static_cast<int>(k % S);
        const uint64_t off = (gw + k * stride) * T;
        float* sp = stage_p(s);
        mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(kStage));
        bulk_load(sp, p + off, 4u * T, &full[s]);
        bulk_load(sp + T, m + off, 4u * T, &full[s]);
        bulk_load(sp + 2 * T, v + off, 4u * T, &full[s]);
        bulk_load(sp + 3 * T, g + off, 2u * T, &full[s]);
    };
    if (lane == 0)
        for (uint64_t k = 0; k + 1 < static_cast<uint64_t>(S) && k < mine; ++k) issue(k);
    unsigned nonfinite = 0, overflow = 0;
    for (uint64_t k = 0; k < mine; ++k) {
        if (lane == 0 && k + S - 1 < mine) issue(k + S - 1);  // the stage of tile k-1, retired by the __syncwarp
        const int s = static_cast<int>(k % S);
        mbar_wait(&full[s], static_cast<uint32_t>(k / S) & 1u);
        const uint64_t off = (gw + k * stride) * T;
        const float* sp = stage_p(s);
        float4 rp = reinterpret_cast<const float4*>(sp)[lane];
        float4 rm = reinterpret_cast<const float4*>(sp + T)[lane];
        float4 rv = reinterpret_cast<const float4*>(sp + 2 * T)[lane];
        const uint2 graw = reinterpret_cast<const uint2*>(sp + 3 * T)[lane];
        __syncwarp();  // every lane has its quad in registers: the stage may be refilled
        U16x4 gh;
        gh.x = static_cast<uint16_t>(graw.x & 0xFFFFu);
        gh.y = static_cast<uint16_t>(graw.x >> 16);
        gh.z = static_cast<uint16_t>(graw.y & 0xFFFFu);
        gh.w = static_cast<uint16_t>(graw.y >> 16);
        nonfinite += nonfinite16<kF16>(gh.x) + nonfinite16<kF16>(gh.y) + nonfinite16<kF16>(gh.z) +
                     nonfinite16<kF16>(gh.w);
        adam_element<WD, true>(rp.x, rm.x, rv.x, widen16<kF16>(gh.x), c);
        adam_element<WD, true>(rp.y, rm.y, rv.y, widen16<kF16>(gh.y), c);
        adam_element<WD, true>(rp.z, rm.z, rv.z, widen16<kF16>(gh.z), c);
        adam_element<WD, true>(rp.w, rm.w, rv.w, widen16<kF16>(gh.w), c);
        U16x4 h;
        h.x = narrow16<kF16>(rp.x);
        h.y = narrow16<kF16>(rp.y);
        h.z = narrow16<kF16>(rp.z);
        h.w = narrow16<kF16>(rp.w);
        overflow += is_inf16<kF16>(h.x) + is_inf16<kF16>(h.y) + is_inf16<kF16>(h.z) + is_inf16<kF16>(h.w);
        __stcs(reinterpret_cast<float4*>(p + off) + lane, rp);
        __stcs(reinterpret_cast<float4*>(m + off) + lane, rm);
        __stcs(reinterpret_cast<float4*>(v + off) + lane, rv);
        store_u16x4(p16 + off + 4 * lane, h);
    }
    if (counters != nullptr) {
        warp_count_add(counters + 0, nonfinite);
        warp_count_add(counters + 1, overflow);
    }
}

template <int S, int MINB>
cudaError_t launch_warp_pipe(const AdamLaunch& a, cudaStream_t stream) {
    constexpr int T = 128;
    const bool aligned = ((reinterpret_cast<uintptr_t>(a.p) | reinterpret_cast<uintptr_t>(a.m) |
                           reinterpret_cast<uintptr_t>(a.v) | reinterpret_cast<uintptr_t>(a.g) |
                           reinterpret_cast<uintptr_t>(a.p16)) & 15u) == 0;
    if (!aligned || a.n_peers > 0 || a.p_out || a.grad_kind != kF16 || a.out_kind != kF16)
        return cudaErrorInvalidValue;
    const uint64_t ntiles = a.n / T;
    constexpr size_t smem = static_cast<size_t>(kThreads / 32) * S * (T * 14 + sizeof(uint64_t));
    if (ntiles > 0) {
        auto kern = a.c.lr_wd != 0.0 ? adam_warp_pipe_kernel<S, true, MINB> : adam_warp_pipe_kernel<S, false, MINB>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        const uint64_t warps = (ntiles + 0);  // one warp per tile at most
        const unsigned grid = static_cast<unsigned>(
            std::min<uint64_t>((warps + kThreads / 32 - 1) / (kThreads / 32), static_cast<uint64_t>(num_sms()) * MINB));
        kern<<<grid, kThreads, smem, stream>>>(a.p, a.m, a.v, static_cast<const uint16_t*>(a.g), a.p16, ntiles, a.c,
                                               a.counters);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const uint64_t done = ntiles * T;
    if (done == a.n) return cudaSuccess;
    AdamLaunch tail = a;
    tail.p += done;
    tail.m += done;
    tail.v += done;
    tail.g = static_cast<const uint16_t*>(a.g) + done;
    tail.p16 += done;
    tail.n = a.n - done;
    return launch_dtypes<Cfg<1, true, 4>>(tail, stream);
}

// ---------------------------------------------------------------------------
// cp.async double-buffered variant: each thread copies its NEXT quad of P, m,
// v, g into its own shared-memory slots with cp.async (LDGSTS, no registers
// held) before computing the current one, so memory latency overlaps the FP64
// chain without giving up occupancy. Same element math and stores as the
// register kernel; F16 in and out.

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <bool WD, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    adam_cpasync_kernel(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                        const uint16_t* __restrict__ g, uint16_t* __restrict__ p16, uint64_t nq, AdamConsts c,
                        unsigned long long* __restrict__ counters) {
    __shared__ float4 sbuf[2][3][kThreads];
    __shared__ uint2 sgrad[2][kThreads];
    unsigned nonfinite = 0, overflow = 0;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int t = threadIdx.x;
    float4* p4 = reinterpret_cast<float4*>(p);
    float4* m4 = reinterpret_cast<float4*>(m);
    float4* v4 = reinterpret_cast<float4*>(v);
    const uint2* g2 = reinterpret_cast<const uint2*>(g);
    auto issue = [&](uint64_t qq, int s) {
        cp_async16(&sbuf[s][0][t], p4 + qq);
        cp_async16(&sbuf[s][1][t], m4 + qq);
        cp_async16(&sbuf[s][2][t], v4 + qq);
        cp_async8(&sgrad[s][t], g2 + qq);
    };
    int s = 0;
    if (q < nq) issue(q, 0);
    cp_async_commit();
    for (; q < nq; q += nthreads, s ^= 1) {
        const uint64_t nxt = q + nthreads;
        if (nxt < nq) issue(nxt, s ^ 1);
        cp_async_commit();
        cp_async_wait<1>();  // the current quad has landed; the next stays in flight
        float4 rp = sbuf[s][0][t], rm = sbuf[s][1][t], rv = sbuf[s][2][t];
        const uint2 graw = sgrad[s][t];
        U16x4 gh;
        gh.x = static_cast<uint16_t>(graw.x & 0xFFFFu);
        gh.y = static_cast<uint16_t>(graw.x >> 16);
        gh.z = static_cast<uint16_t>(graw.y & 0xFFFFu);
        gh.w = static_cast<uint16_t>(graw.y >> 16);
        nonfinite += nonfinite16<kF16>(gh.x) + nonfinite16<kF16>(gh.y) + nonfinite16<kF16>(gh.z) +
                     nonfinite16<kF16>(gh.w);
        adam_element<WD, true>(rp.x, rm.x, rv.x, widen16<kF16>(gh.x), c);
        adam_element<WD, true>(rp.y, rm.y, rv.y, widen16<kF16>(gh.y), c);
        adam_element<WD, true>(rp.z, rm.z, rv.z, widen16<kF16>(gh.z), c);
        adam_element<WD, true>(rp.w, rm.w, rv.w, widen16<kF16>(gh.w), c);
        U16x4 h;
        h.x = narrow16<kF16>(rp.x);
        h.y = narrow16<kF16>(rp.y);
        h.z = narrow16<kF16>(rp.z);
        h.w = narrow16<kF16>(rp.w);
        overflow += is_inf16<kF16>(h.x) + is_inf16<kF16>(h.y) + is_inf16<kF16>(h.z) + is_inf16<kF16>(h.w);
        __stcs(p4 + q, rp);
        __stcs(m4 + q, rm);
        __stcs(v4 + q, rv);
        store_u16x4(p16 + 4 * q, h);
    }
    cp_async_wait<0>();
    if (counters != nullptr) {
        warp_count_add(counters + 0, nonfinite);
        warp_count_add(counters + 1, overflow);
    }
}

template <int MINB>
cudaError_t launch_cpasync(const AdamLaunch& a, cudaStream_t stream) {
    const bool aligned = ((reinterpret_cast<uintptr_t>(a.p) | reinterpret_cast<uintptr_t>(a.m) |
                           reinterpret_cast<uintptr_t>(a.v)) & 15u) == 0 &&
                         ((reinterpret_cast<uintptr_t>(a.g) | reinterpret_cast<uintptr_t>(a.p16)) & 7u) == 0;
    if (!aligned || a.n_peers > 0 || a.p_out || a.grad_kind != kF16 || a.out_kind != kF16)
        return cudaErrorInvalidValue;
    const uint64_t nq = a.n / 4;
    if (nq > 0) {
        const unsigned grid = grid_for(nq, MINB);
        if (a.c.lr_wd != 0.0)
            adam_cpasync_kernel<true, MINB><<<grid, kThreads, 0, stream>>>(
                a.p, a.m, a.v, static_cast<const uint16_t*>(a.g), a.p16, nq, a.c, a.counters);
        else
            adam_cpasync_kernel<false, MINB><<<grid, kThreads, 0, stream>>>(
                a.p, a.m, a.v, static_cast<const uint16_t*>(a.g), a.p16, nq, a.c, a.counters);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (nq * 4 == a.n) return cudaSuccess;
    AdamLaunch tail = a;  // the n % 4 remainder through the register-streaming kernel
    const uint64_t done = nq * 4;
    tail.p += done;
    tail.m += done;
    tail.v += done;
    tail.g = static_cast<const uint16_t*>(a.g) + done;
    tail.p16 += done;
    tail.n = a.n - done;
    return launch_dtypes<Cfg<1, true, 4>>(tail, stream);
}

// Scalar-element form at a given occupancy (tuning variants): 4-byte
// coalesced streams, one element per thread per iteration.
template <bool WD, int MINB>
cudaError_t launch_scalar(const AdamLaunch& a, cudaStream_t stream) {
    const unsigned grid = grid_for(a.n, MINB);
    adam_fused_kernel<kF16, 0, kF16, WD, false, 1, 1, MINB>
        <<<grid, kThreads, 0, stream>>>(state_io(a), sources_of(a), a.p16, a.n, a.c, a.counters, nullptr);
    return cudaGetLastError();
}
template <int MINB>
cudaError_t launch_scalar_wd(const AdamLaunch& a, cudaStream_t stream) {
    return a.c.lr_wd != 0.0 ? launch_scalar<true, MINB>(a, stream) : launch_scalar<false, MINB>(a, stream);
}

// Software-pipelined register form (variants 41-43): each thread issues the
// loads of its next grid-stride quad before the binary64 chain of the
// current one, so a warp keeps a quad's 28 bytes in flight through its whole
// compute phase (memory parallelism that does not shrink when the SM clock
// drops under the power cap), at the price of ~14 more registers (MINB 3).
template <bool WD, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    adam_swp_kernel(const StateIO io, const uint16_t* __restrict__ g, uint16_t* __restrict__ p16, uint64_t nq,
                    AdamConsts c, unsigned long long* __restrict__ counters) {
    unsigned nonfinite = 0, overflow = 0;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const float4* p4 = reinterpret_cast<const float4*>(io.p);
    const float4* m4 = reinterpret_cast<const float4*>(io.m);
    const float4* v4 = reinterpret_cast<const float4*>(io.v);
    float4 rp{}, rm{}, rv{};
    U16x4 rg{};
    if (q < nq) {
        rp = __ldcs(p4 + q);
        rm = __ldcs(m4 + q);
        rv = __ldcs(v4 + q);
        rg = load_u16x4(g + 4 * q);
    }
    while (q < nq) {
        const uint64_t qn = q + nthreads;
        float4 np{}, nm{}, nv{};
        U16x4 ng{};
        if (qn < nq) {  // next quad's loads in flight during this quad's math
            np = __ldcs(p4 + qn);
            nm = __ldcs(m4 + qn);
            nv = __ldcs(v4 + qn);
            ng = load_u16x4(g + 4 * qn);
        }
        nonfinite += nonfinite16<kF16>(rg.x) + nonfinite16<kF16>(rg.y) + nonfinite16<kF16>(rg.z) +
                     nonfinite16<kF16>(rg.w);
        adam_math<WD, 1>(rp.x, rm.x, rv.x, widen16<kF16>(rg.x), c);
        adam_math<WD, 1>(rp.y, rm.y, rv.y, widen16<kF16>(rg.y), c);
        adam_math<WD, 1>(rp.z, rm.z, rv.z, widen16<kF16>(rg.z), c);
        adam_math<WD, 1>(rp.w, rm.w, rv.w, widen16<kF16>(rg.w), c);
        U16x4 h;
        h.x = narrow16<kF16>(rp.x);
        h.y = narrow16<kF16>(rp.y);
        h.z = narrow16<kF16>(rp.z);
        h.w = narrow16<kF16>(rp.w);
        overflow += is_inf16<kF16>(h.x) + is_inf16<kF16>(h.y) + is_inf16<kF16>(h.z) + is_inf16<kF16>(h.w);
        __stcs(reinterpret_cast<float4*>(io.po) + q, rp);
        __stcs(reinterpret_cast<float4*>(io.mo) + q, rm);
        __stcs(reinterpret_cast<float4*>(io.vo) + q, rv);
        store_u16x4(p16 + 4 * q, h);
        rp = np;
        rm = nm;
        rv = nv;
        rg = ng;
        q = qn;
    }
    if (counters != nullptr) {
        warp_count_add(counters + 0, nonfinite);
        warp_count_add(counters + 1, overflow);
    }
}

template <bool WD, int MINB>
cudaError_t launch_swp(const AdamLaunch& a, cudaStream_t stream) {
    if (!is_vec(a)) return launch_dtypes<Cfg<1, true, 4>>(a, stream);
    const uint64_t nq = a.n / 4;
    if (nq > 0)
        adam_swp_kernel<WD, MINB><<<grid_for(nq, MINB), kThreads, 0, stream>>>(
            state_io(a), static_cast<const uint16_t*>(a.g), a.p16, nq, a.c, a.counters);
    if (nq * 4 == a.n) return cudaGetLastError();
    AdamLaunch tail = a;  // the n % 4 remainder through the shipped kernel
    const uint64_t done = nq * 4;
    tail.p += done;
    tail.m += done;
    tail.v += done;
    tail.g = static_cast<const uint16_t*>(a.g) + done;
    tail.p16 += done;
    tail.n = a.n - done;
    return launch_dtypes<Cfg<1, true, 4>>(tail, stream);
}
template <int MINB>
cudaError_t launch_swp_wd(const AdamLaunch& a, cudaStream_t stream) {
    return a.c.lr_wd != 0.0 ? launch_swp<true, MINB>(a, stream) : launch_swp<false, MINB>(a, stream);
}

// The operand domain of adam_element_rn (numerics.cuh): lr in [2^-600, 2^600],
// eps in [2^-600, 2^96], lr / eps <= 2^600, bias corrections in [2^-64, 1].
bool fast_rn_domain(const AdamConsts& c) {
    auto in = [](double x, double lo, double hi) { return x >= lo && x <= hi; };
    return in(c.lr, 0x1p-600, 0x1p600) && in(c.eps, 0x1p-600, 0x1p96) && c.lr / c.eps <= 0x1p600 &&
           in(c.bc1, 0x1p-64, 1.0) && in(c.bc2, 0x1p-64, 1.0);
}

// Self-test of sqrt_rn_in_range / div_rn_in_range against __dsqrt_rn /
// __ddiv_rn: random significands (plus all-ones / power-of-two / exact
// multiples) over the domain's exponent ranges; counts mismatches.
__global__ void fast_rn_selftest_kernel(uint64_t n, uint64_t seed, unsigned long long* bad) {
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    unsigned nb = 0;
    for (uint64_t i = tid; i < n; i += nthreads) {
        const uint64_t r1 = splitmix64(seed ^ (3 * i)), r2 = splitmix64(seed ^ (3 * i + 1)),
                       r3 = splitmix64(seed ^ (3 * i + 2));
        auto mant = [](uint64_t r) {
            uint64_t m = r & 0xFFFFFFFFFFFFFULL;
            const int sel = static_cast<int>((r >> 52) & 7u);
            if (sel == 0) m |= 0xFFFFFFFFFF000ULL;
            if (sel == 1) m &= 0x0000000000FFFULL;
            return m;
        };
        // sqrt: x in [2^-960, 2^960) (the Adam chain's v/bc2 lies in [2^-149, 2^192])
        const int ex = -960 + static_cast<int>((r1 >> 53) % 1920);
        const double x = __longlong_as_double(static_cast<long long>((static_cast<uint64_t>(ex + 1023) << 52) | mant(r1)));
        nb += __double_as_longlong(sqrt_rn_in_range(x)) != __double_as_longlong(__dsqrt_rn(x));
        // division: b in [2^-600, 2^160), a in [2^-960, 2^1000), a / b in [2^-846, 2^792)
        const int eb = -600 + static_cast<int>((r2 >> 53) % 760);
        const int lo = max(-846, -960 - eb), hi = min(792, 1000 - eb);
        const int eq = lo + static_cast<int>((r3 >> 53) % static_cast<uint64_t>(hi - lo));
        const double b = __longlong_as_double(static_cast<long long>((static_cast<uint64_t>(eb + 1023) << 52) | mant(r2)));
        double a = __longlong_as_double(static_cast<long long>((static_cast<uint64_t>(eb + eq + 1023) << 52) | mant(r3)));
        if ((r3 & 15) == 0) a = __dmul_rn(b, static_cast<double>(static_cast<int>((r3 >> 4) & 0xFFFF) + 1));
        if (r3 >> 63) a = -a;
        nb += __double_as_longlong(div_rn_in_range(a, b)) != __double_as_longlong(__ddiv_rn(a, b));
    }
    warp_count_add(bad, nb);
}


// ---------------------------------------------------------------------------
// Layout experiment (variant 67): the state tile-interleaved in HBM — for each
// tile of T = 1024 params, P, m and v contiguous ([P | m | v], 12 KiB) — so a
// tile is one 12 KiB bulk load and three contiguous stores, and the DRAM
// sees two read and two write streams per tile instead of four and four.
// `p` is the interleaved buffer's base (m, v unused); g and p16 as usual.
// Same element math; the bits land in the interleaved positions.
template <bool WD>
__global__ void __launch_bounds__(kThreads, 4)
    adam_staged_interleaved_kernel(float* __restrict__ st, const uint16_t* __restrict__ g, uint16_t* __restrict__ p16,
                                   uint64_t ntiles, AdamConsts c, unsigned long long* __restrict__ counters) {
    constexpr int S = 2;
    constexpr int T = 4 * kThreads;
    extern __shared__ __align__(128) unsigned char smem[];
    float* sst = reinterpret_cast<float*>(smem);                    // S x [P | m | v]
    uint16_t* sg = reinterpret_cast<uint16_t*>(sst + S * 3 * T);     // S x g
    uint64_t* full = reinterpret_cast<uint64_t*>(sg + S * T);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t mine = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    auto issue = [&](uint64_t k) {
        const int s = static_cast<int>(k % S);
        const uint64_t t = blockIdx.x + k * gridDim.x;
        mbar_arrive_expect_tx(&full[s], 14u * T);
        bulk_load(sst + s * 3 * T, st + t * 3 * T, 12u * T, &full[s]);
        bulk_load(sg + s * T, g + t * T, 2u * T, &full[s]);
    };
    if (threadIdx.x == 0 && mine > 0) issue(0);
    unsigned nonfinite = 0, overflow = 0;
    const int qi = threadIdx.x;
    for (uint64_t k = 0; k < mine; ++k) {
        if (threadIdx.x == 0 && k + 1 < mine) issue(k + 1);
        const int s = static_cast<int>(k % S);
        mbar_wait(&full[s], static_cast<uint32_t>(k / S) & 1u);
        const uint64_t t = blockIdx.x + k * gridDim.x;
        const float* ss = sst + s * 3 * T;
        const float4 rp = reinterpret_cast<const float4*>(ss)[qi];
        const float4 rm = reinterpret_cast<const float4*>(ss + T)[qi];
        const float4 rv = reinterpret_cast<const float4*>(ss + 2 * T)[qi];
        const uint2 graw = reinterpret_cast<const uint2*>(sg + s * T)[qi];
        float* dst = st + t * 3 * T;
        staged_quad<kF16, kF16, WD, false, 1>(rp, rm, rv, graw, c, nonfinite, overflow, dst, dst + T, dst + 2 * T,
                                              p16 + t * T, qi);
        __syncthreads();
    }
    if (counters != nullptr) warp_count_add(counters + 1, overflow);
}

cudaError_t launch_staged_interleaved(const AdamLaunch& a, cudaStream_t stream) {
    constexpr uint64_t T = 4 * kThreads;
    const uint64_t ntiles = a.n / T;  // timing experiment: whole tiles only
    if (ntiles == 0) return cudaErrorInvalidValue;
    constexpr size_t smem = 2 * T * 14 + 2 * sizeof(uint64_t);
    auto kern = a.c.lr_wd != 0.0 ? adam_staged_interleaved_kernel<true> : adam_staged_interleaved_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(ntiles, static_cast<uint64_t>(num_sms()) * 4));
    kern<<<grid, kThreads, smem, stream>>>(a.p, static_cast<const uint16_t*>(a.g), a.p16, ntiles, a.c, a.counters);
    return cudaGetLastError();
}

template <int V>
cudaError_t launch_variant(const AdamLaunch& a, cudaStream_t stream) {
    if constexpr (V == 1) return launch_wd<kF16, 0, kF16, Cfg<2, false, 1>>(a, stream);
    if constexpr (V == 2) return launch_wd<kF16, 0, kF16, Cfg<1, false, 4>>(a, stream);
    if constexpr (V == 3) return launch_wd<kF16, 0, kF16, Cfg<2, false, 3>>(a, stream);
    if constexpr (V == 4) return launch_wd<kF16, 0, kF16, Cfg<1, true, 4>>(a, stream);
    if constexpr (V == 5) return launch_wd<kF16, 0, kF16, Cfg<2, true, 3>>(a, stream);
    if constexpr (V == 6) return launch_wd<kF16, 0, kF16, Cfg<2, true, 2>>(a, stream);
    if constexpr (V == 7) return launch_wd<kF16, 0, kF16, Cfg<1, true, 3>>(a, stream);
    if constexpr (V == 8) return launch_wd<kF16, 0, kF16, Cfg<4, true, 2>>(a, stream);
    if constexpr (V == 9) return launch_wd<kF16, 0, kF16, Cfg<1, true, 5>>(a, stream);
    if constexpr (V == 10) return launch_wd<kF16, 0, kF16, Cfg<2, true, 4>>(a, stream);
    if constexpr (V == 11) return launch_wd<kF16, 0, kF16, Cfg<1, true, 6>>(a, stream);
    if constexpr (V == 12) return launch_tma<1024, 4, 2>(a, stream);
    if constexpr (V == 13) return launch_tma<1024, 3, 3>(a, stream);
    if constexpr (V == 14) return launch_tma<2048, 3, 2>(a, stream);
    if constexpr (V == 15) return launch_tma<512, 4, 4>(a, stream);
    if constexpr (V == 16) return launch_cpasync<4>(a, stream);
    if constexpr (V == 17) return launch_cpasync<3>(a, stream);
    if constexpr (V == 18) return launch_wd<kF16, 0, kF16, Cfg<1, 2, 4>>(a, stream);
    if constexpr (V == 19) return launch_wd<kF16, 0, kF16, Cfg<2, 2, 3>>(a, stream);
    if constexpr (V == 20) return launch_wd<kF16, 0, kF16, Cfg<1, 2, 5>>(a, stream);
    if constexpr (V == 21) return launch_scalar_wd<4>(a, stream);
    if constexpr (V == 22) return launch_scalar_wd<5>(a, stream);
    if constexpr (V == 23) return launch_scalar_wd<6>(a, stream);
    if constexpr (V == 24) return launch_wd<kF16, 0, kF16, Cfg<1, 3, 5>>(a, stream);
    if constexpr (V == 25) return launch_wd<kF16, 0, kF16, Cfg<1, 3, 6>>(a, stream);
    if constexpr (V == 26) return launch_wd<kF16, 0, kF16, Cfg<1, 4, 4>>(a, stream);
    if constexpr (V == 27) return launch_wd<kF16, 0, kF16, Cfg<1, 4, 5>>(a, stream);
    if constexpr (V == 28) return launch_wd<kF16, 0, kF16, Cfg<1, 1, 4, 1>>(a, stream);
    if constexpr (V == 29) return launch_wd<kF16, 0, kF16, Cfg<1, 1, 4, 2>>(a, stream);
    if constexpr (V == 30) return launch_wd<kF16, 0, kF16, Cfg<1, 1, 4, 4>>(a, stream);
    if constexpr (V == 31) return launch_wd<kF16, 0, kF16, Cfg<1, 1, 3, 2>>(a, stream);
    if constexpr (V == 32) return launch_tma_pipe<3, 4>(a, stream);
    if constexpr (V == 33) return launch_tma_pipe<2, 4>(a, stream);
    if constexpr (V == 34) return launch_tma_pipe<4, 3>(a, stream);
    if constexpr (V == 35) return launch_tma_pipe<3, 3>(a, stream);
    if constexpr (V == 36) return launch_tma_pipe<3, 4, true>(a, stream);
    if constexpr (V == 37) return launch_tma_pipe<2, 4, true>(a, stream);
    if constexpr (V == 38) return launch_warp_pipe<3, 4>(a, stream);
    if constexpr (V == 39) return launch_warp_pipe<2, 4>(a, stream);
    if constexpr (V == 40) return launch_warp_pipe<4, 3>(a, stream);
    if constexpr (V == 41) return launch_swp_wd<3>(a, stream);
    if constexpr (V == 42) return launch_swp_wd<4>(a, stream);
    if constexpr (V == 43) return launch_swp_wd<2>(a, stream);
    if constexpr (V == 44) return launch_wd<kF16, 0, kF16, Cfg<1, 5, 4>>(a, stream);
    if constexpr (V == 45) return launch_wd<kF16, 0, kF16, Cfg<1, 5, 3>>(a, stream);
    if constexpr (V == 46) return launch_wd<kF16, 0, kF16, Cfg<1, 6, 4>>(a, stream);
    if constexpr (V == 48) return launch_wd<kF16, 0, kF16, Cfg<1, 1, 4, -1>>(a, stream);
    if constexpr (V == 49) return launch_wd<kF16, 0, kF16, Cfg<1, 1, 4, -2>>(a, stream);
    if constexpr (V == 50) return launch_wd<kF16, 0, kF16, Cfg<1, 1, 4, -3>>(a, stream);
    if constexpr (V == 51) return launch_wd<kF16, 0, kF16, Cfg<1, 1, 4, 0, kOptVerified | kOptF64Widen>>(a, stream);
    if constexpr (V == 52) return launch_wd<kF16, 0, kF16, Cfg<1, 1, 4, 0, kOptF64Widen>>(a, stream);
    if constexpr (V == 53) return launch_wd<kF16, 0, kF16, Cfg<1, 1, 4, 0, kOptVerified>>(a, stream);
    if constexpr (V >= 54 && V <= 57) {
        AdamLaunch b = a;
        b.grads_verified = V != 54;
        constexpr int S = V >= 56 ? 3 : 2;
        constexpr int M = V == 57 ? 3 : 4;
        return launch_staged<S, M>(b, stream);
    }
    if constexpr (V >= 59 && V <= 64) {  // deeper staging / larger tiles (S stages, M CTAs per SM, Q quads per thread)
        AdamLaunch b = a;
        b.grads_verified = true;
        if constexpr (V == 59) return launch_staged<3, 4>(b, stream);
        if constexpr (V == 60) return launch_staged<2, 3, 1, 2>(b, stream);
        if constexpr (V == 61) return launch_staged<3, 2, 1, 2>(b, stream);
        if constexpr (V == 62) return launch_staged<4, 2, 1, 2>(b, stream);
        if constexpr (V == 63) return launch_staged<3, 1, 1, 4>(b, stream);
        return launch_staged<2, 1, 1, 4>(b, stream);
    }
    if constexpr (V == 67) return launch_staged_interleaved(a, stream);
    if constexpr (V == 65 || V == 66) {  // shipped shape + L2 prefetch 1 / 2 tiles beyond the staged look-ahead
        AdamLaunch b = a;
        b.grads_verified = true;
        return launch_staged<2, 4, 1, 1, V == 65 ? 1 : 2>(b, stream);
    }
    if constexpr (V == 58) {  // staged + in-range sqrt / division (domain-gated, as variant 47)
        AdamLaunch b = a;
        b.grads_verified = true;
        return fast_rn_domain(a.c) ? launch_staged<2, 4, 7>(b, stream)
                                   : launch_staged<2, 4>(b, stream);
    }
    if constexpr (V == 47)
        return fast_rn_domain(a.c) ? launch_wd<kF16, 0, kF16, Cfg<1, 7, 4>>(a, stream)
                                   : launch_dtypes<Cfg<1, true, 4>>(a, stream);
    return cudaErrorInvalidValue;
}

}  // namespace

// Variants 34 and up, compiled in adam_variants_hi.cu (the two halves build in parallel).
cudaError_t launch_adam_fused_variant_hi(const AdamLaunch& a, int variant, cudaStream_t stream);

}  // namespace tfb
