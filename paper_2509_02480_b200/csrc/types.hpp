// Plain-C++ types shared by the kernels (nvcc) and the host engine (g++).
#pragma once

#include <cstdint>

namespace tfb {

// Gradient / working-parameter element kinds (16-bit storage).
// kF32 is a gradient kind only: the ZeRO-3 baseline flow fetches fp32
// gradients from storage (reference scheduler.hpp:377-391, 667-680).
enum Half16Kind : int { kF16 = 0, kBF16 = 1, kF32 = 2 };

// Per-launch Adam constants, all computed on the host in double exactly as the
// reference does (bc_k = 1 - pow(beta_k, t), reference optimizer.hpp:129-130).
struct AdamConsts {
    double lr;
    double beta1;
    double beta2;
    double one_minus_beta1;  // (1.0 - beta1), the reference loop invariant
    double one_minus_beta2;
    double eps;
    double lr_wd;  // lr * weight_decay; 0 disables decay (optimizer.hpp:94)
    double bc1;
    double bc2;
    double inv_bc1;  // RN(1 / bc1): the constant-divisor path
    double inv_bc2;  // RN(1 / bc2)
};

// splitmix64 (reference scheduler.hpp:76-81) for the host-folded prefixes of
// the synthetic generators.
inline std::uint64_t splitmix64_host(std::uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

// Prefix of SyntheticGradSource::sample (scheduler.hpp:88-92); element i is
// splitmix64(prefix ^ i).
inline std::uint64_t grad_prefix(std::uint64_t seed, std::uint32_t sg, int iteration, int step) {
    std::uint64_t x = splitmix64_host(seed ^ 0xC2B2AE3D27D4EB4FULL);
    x = splitmix64_host(x ^ sg);
    x = splitmix64_host(x ^ static_cast<std::uint64_t>(iteration));
    return splitmix64_host(x ^ static_cast<std::uint64_t>(step));
}

// Prefix of synthetic_param_init (scheduler.hpp:104-107).
inline std::uint64_t param_prefix(std::uint64_t seed, std::uint32_t sg) {
    return splitmix64_host(splitmix64_host(seed ^ 0xA0761D6478BD642FULL) ^ sg);
}

}  // namespace tfb
