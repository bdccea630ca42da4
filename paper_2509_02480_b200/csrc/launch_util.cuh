// Launch helpers shared by the kernel translation units.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

namespace tfb {
namespace detail {

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

inline int g_num_sms = 0;

inline int num_sms() {
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
inline unsigned grid_for(uint64_t work_items, int ctas_per_sm) {
    const uint64_t need = (work_items + kThreads - 1) / kThreads;
    const uint64_t cap = static_cast<uint64_t>(num_sms()) * static_cast<uint64_t>(ctas_per_sm);
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min(need, cap)));
}

}  // namespace detail
}  // namespace tfb
