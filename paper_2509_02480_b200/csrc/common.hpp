// Shared host-side vocabulary: ids, timestamps, transfer stats and the error
// hierarchy. The error classes carry the C-ABI status code they map to, one to
// one with the reference hierarchy (reference proj/include/tierflow/common.hpp:36-78).
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace tfb {

using SubgroupId = std::uint32_t;
using TierId = int;
using WorkerId = int;

inline constexpr TierId kNoTier = -1;

// Status codes of the C ABI (include/tierflow_b200.h).
enum Status : int {
    kOk = 0,
    kErrGeneric = 1,
    kErrIo = 2,
    kErrFormat = 3,
    kErrConfig = 4,
    kErrPlacement = 5,
    kErrScheduling = 6,
    kErrGradientOverflow = 7,
    kErrCuda = 8,
};

// CLOCK_MONOTONIC nanoseconds: one epoch for every process on the host, so
// per-rank traces merge by timestamp.
inline std::int64_t now_ns() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

struct IoStats {
    std::uint64_t bytes = 0;
    double seconds = 0.0;
};

class Error : public std::runtime_error {
public:
    explicit Error(const std::string& what, int code = kErrGeneric)
        : std::runtime_error(what), code_(code) {}
    int code() const { return code_; }

private:
    int code_;
};

#define TFB_ERROR_CLASS(Name, Code)                                           \
    class Name : public Error {                                               \
    public:                                                                   \
        explicit Name(const std::string& what) : Error(what, Code) {}         \
    };

TFB_ERROR_CLASS(IoError, kErrIo)                           // storage backend failure
TFB_ERROR_CLASS(FormatError, kErrFormat)                   // malformed subgroup file
TFB_ERROR_CLASS(ConfigError, kErrConfig)                   // bad configuration
TFB_ERROR_CLASS(PlacementInconsistencyError, kErrPlacement)  // read of an absent subgroup
TFB_ERROR_CLASS(SchedulingBugError, kErrScheduling)        // watchdog: no progress
TFB_ERROR_CLASS(GradientOverflowError, kErrGradientOverflow)  // non-finite gradients
TFB_ERROR_CLASS(CudaError, kErrCuda)                       // CUDA runtime failure
#undef TFB_ERROR_CLASS

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw CudaError(std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                        cudaGetErrorString(e) + ")");
}

}  // namespace tfb
