// Page-aligned host buffer laid out like a subgroup file: a 32-byte header
// area followed by the P||m||v payload. Engine staging slots and host-DRAM tier
// blobs are HostBlocks, so a file tier can O_DIRECT-read a whole subgroup file
// (header included) straight into the pinned buffer the H2D DMA reads from,
// and a host-DRAM tier can hand blobs to the pipeline by exchanging blocks
// instead of copying them.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "common.hpp"

namespace tfb {

constexpr std::size_t kHeaderBytes = 32;
constexpr std::size_t kPageBytes = 4096;

inline std::size_t round_up(std::size_t x, std::size_t a) { return (x + a - 1) / a * a; }

// Live host blocks (count, bytes) in the process: leak accounting for tests.
inline std::atomic<std::int64_t> g_host_blocks_live{0};
inline std::atomic<std::int64_t> g_host_bytes_live{0};
inline std::atomic<std::int64_t> g_host_free_failures{0};

// Bytes a block needs for a subgroup of `params` parameters.
inline std::size_t block_bytes_for(std::uint64_t params) {
    return round_up(kHeaderBytes + 12 * static_cast<std::size_t>(params), kPageBytes);
}

class HostBlock {
public:
    HostBlock() = default;
    HostBlock(const HostBlock&) = delete;
    HostBlock& operator=(const HostBlock&) = delete;
    HostBlock(HostBlock&& o) noexcept { *this = std::move(o); }
    HostBlock& operator=(HostBlock&& o) noexcept {
        if (this != &o) {
            release();
            base_ = std::exchange(o.base_, nullptr);
            bytes_ = std::exchange(o.bytes_, 0);
            pinned_ = std::exchange(o.pinned_, false);
        }
        return *this;
    }
    ~HostBlock() { release(); }

    // Pinned (cudaHostAlloc) when a CUDA device is usable; plain page-aligned
    // memory is accepted only when require_pinned is false (storage-only use).
    static HostBlock allocate(std::size_t bytes, bool require_pinned) {
        HostBlock b;
        bytes = round_up(bytes, kPageBytes);
        void* p = nullptr;
        const cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocPortable | cudaHostAllocMapped);
        if (e == cudaSuccess) {
            b.pinned_ = true;
        } else {
            (void)cudaGetLastError();
            if (require_pinned)
                throw CudaError(std::string("cudaHostAlloc of ") + std::to_string(bytes) +
                                " bytes failed: " + cudaGetErrorString(e));
            if (posix_memalign(&p, kPageBytes, bytes) != 0) throw IoError("host block allocation failed");
        }
        b.base_ = static_cast<std::uint8_t*>(p);
        b.bytes_ = bytes;
        if (log_enabled()) std::fprintf(stderr, "hostblock alloc %p %zu pinned=%d\n", p, bytes, int(b.pinned_));
        g_host_blocks_live.fetch_add(1, std::memory_order_relaxed);
        g_host_bytes_live.fetch_add(static_cast<std::int64_t>(bytes), std::memory_order_relaxed);
        return b;
    }

    std::uint8_t* base() const { return base_; }
    float* payload() const { return reinterpret_cast<float*>(base_ + kHeaderBytes); }
    std::size_t bytes() const { return bytes_; }
    std::size_t payload_capacity_params() const { return bytes_ > kHeaderBytes ? (bytes_ - kHeaderBytes) / 12 : 0; }
    bool pinned() const { return pinned_; }
    explicit operator bool() const { return base_ != nullptr; }

private:
    // TFB_HOSTBLOCK_LOG=1: every allocation and release on stderr (leak forensics).
    static bool log_enabled() {
        static const bool on = std::getenv("TFB_HOSTBLOCK_LOG") != nullptr;
        return on;
    }

    void release() {
        if (base_ == nullptr) return;
        if (log_enabled()) std::fprintf(stderr, "hostblock free %p pinned=%d\n", static_cast<void*>(base_), int(pinned_));
        g_host_blocks_live.fetch_sub(1, std::memory_order_relaxed);
        g_host_bytes_live.fetch_sub(static_cast<std::int64_t>(bytes_), std::memory_order_relaxed);
        if (pinned_) {
            if (cudaFreeHost(base_) != cudaSuccess) {
                (void)cudaGetLastError();
                g_host_free_failures.fetch_add(1, std::memory_order_relaxed);
            }
        } else
            std::free(base_);
        base_ = nullptr;
        bytes_ = 0;
        pinned_ = false;
    }

    std::uint8_t* base_ = nullptr;
    std::size_t bytes_ = 0;
    bool pinned_ = false;
};

}  // namespace tfb
