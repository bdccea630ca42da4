// extern "C" entry points of the tuning library (include/tierflow_b200_tuning.h):
// the fused kernel's measured variants (adam_variants.cu), for the kernel
// sweeps and the bit-parity test over every variant. Linked against the
// product library for the shared host code (AdamHyper::consts, the shipped
// launch as variant 0); the product library never loads this one.
#include "../../include/tierflow_b200_tuning.h"

#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "capi_internal.hpp"
#include "common.hpp"
#include "engine.hpp"
#include "kernels.hpp"

namespace {

template <class F>
int guard(F&& f) {
    try {
        f();
        return TFG_OK;
    } catch (const tfb::Error& e) {
        tfb::set_last_error(e.what());
        return e.code();
    } catch (const std::exception& e) {
        tfb::set_last_error(e.what());
        return TFG_ERROR;
    }
}

}  // namespace

extern "C" {

int tfg_adam_variant_count(int* count) {
    return guard([&] {
        if (count == nullptr) throw tfb::ConfigError("count must not be NULL");
        *count = tfb::adam_variant_count();
    });
}

int tfg_adam_fused_variant(int variant, float* p, float* m, float* v, const uint16_t* grad, uint16_t* param16,
                           uint64_t n, const tfg_adam_hyper* hyper, uint64_t t, unsigned long long* counters,
                           void* stream) {
    return guard([&] {
        if (variant < 0 || variant >= tfb::adam_variant_count()) throw tfb::ConfigError("unknown kernel variant");
        if (hyper == nullptr) throw tfb::ConfigError("hyper must not be NULL");
        if (n > 0 && (!p || !m || !v || !grad || !param16)) throw tfb::ConfigError("null buffer");
        tfb::AdamHyper h;
        h.lr = hyper->lr;
        h.beta1 = hyper->beta1;
        h.beta2 = hyper->beta2;
        h.eps = hyper->eps;
        h.weight_decay = hyper->weight_decay;
        tfb::AdamLaunch a;
        a.p = p;
        a.m = m;
        a.v = v;
        a.g = grad;
        a.p16 = param16;
        a.n = n;
        a.grad_kind = TFG_F16;
        a.out_kind = TFG_F16;
        a.c = h.consts(t);
        a.counters = counters;
        tfb::cuda_check(tfb::launch_adam_fused_variant(a, variant, static_cast<cudaStream_t>(stream)),
                        "adam_fused_variant");
    });
}

int tfg_adam_fused_multi_variant(int variant, float* p, float* m, float* v, const void* const* grads, int n_sources,
                                 uint16_t* param16, uint64_t n, const tfg_adam_hyper* hyper, uint64_t t,
                                 unsigned long long* counters, void* stream) {
    return guard([&] {
        if (variant < 0 || variant > 1) throw tfb::ConfigError("unknown multi-source kernel form");
        if (hyper == nullptr) throw tfb::ConfigError("hyper must not be NULL");
        if (n_sources < 1 || n_sources > tfb::kMaxGradSources) throw tfb::ConfigError("1..8 gradient sources");
        if (n > 0 && (!p || !m || !v || !grads || !param16)) throw tfb::ConfigError("null buffer");
        tfb::AdamHyper h;
        h.lr = hyper->lr;
        h.beta1 = hyper->beta1;
        h.beta2 = hyper->beta2;
        h.eps = hyper->eps;
        h.weight_decay = hyper->weight_decay;
        tfb::AdamLaunch a;
        a.p = p;
        a.m = m;
        a.v = v;
        for (int s = 0; s < n_sources; ++s) a.peers[s] = grads[s];
        a.n_peers = n_sources;
        a.p16 = param16;
        a.n = n;
        a.grad_kind = TFG_F16;
        a.out_kind = TFG_F16;
        a.c = h.consts(t);
        a.counters = counters;
        tfb::cuda_check(tfb::launch_adam_fused_multi_variant(a, variant, static_cast<cudaStream_t>(stream)),
                        "adam_fused_multi_variant");
    });
}

int tfg_selftest_fast_step(uint64_t n, uint64_t seed, double* worst_rel_err, uint64_t* mismatches) {
    return guard([&] {
        unsigned long long* d = nullptr;
        tfb::cuda_check(cudaMalloc(reinterpret_cast<void**>(&d), 2 * sizeof(unsigned long long)), "cudaMalloc");
        unsigned long long h[2] = {0, 0};
        cudaMemset(d, 0, sizeof(h));
        const cudaError_t e = tfb::launch_fast_step_selftest(n, seed, d, nullptr);
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        cudaFree(d);
        tfb::cuda_check(e, "fast_step_selftest");
        double w = 0.0;
        std::memcpy(&w, &h[0], sizeof(w));
        if (worst_rel_err) *worst_rel_err = w;
        if (mismatches) *mismatches = h[1];
    });
}

int tfg_selftest_fast_rn(uint64_t n, uint64_t seed, uint64_t* mismatches) {
    return guard([&] {
        unsigned long long* d = nullptr;
        tfb::cuda_check(cudaMalloc(reinterpret_cast<void**>(&d), sizeof(unsigned long long)), "cudaMalloc");
        unsigned long long h = 0;
        cudaMemset(d, 0, sizeof(h));
        const cudaError_t e = tfb::launch_fast_rn_selftest(n, seed, d, nullptr);
        cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
        cudaFree(d);
        tfb::cuda_check(e, "fast_rn_selftest");
        if (mismatches) *mismatches = h;
    });
}

}  // extern "C"
