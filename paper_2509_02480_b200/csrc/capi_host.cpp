// Host-buffer entry points of the C ABI (include/tierflow_b200.h, "host-side
// reference API"): the calls the reference's own C++ API makes on host
// spans — adam_step, upscale_f16_to_f32, downscale_f32_to_f16 (optimizer.hpp,
// precision.hpp), HostBufferPool (pool.hpp), the Subgroup residency machine
// (optimizer.hpp:39-73) — served by the B200 engine's own objects and sm_100a
// kernels. The numeric calls stage the caller's host arrays through HBM: H2D,
// one kernel, D2H; a rejected step (non-finite gradient) never copies back,
// so the caller's arrays are untouched, as in the reference.
#include "../../include/tierflow_b200.h"

#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <string>

#include "capi_internal.hpp"
#include "engine.hpp"
#include "kernels.hpp"

struct tfg_pool {
    std::unique_ptr<tfb::HostBufferPool> pool;
    std::uint64_t max_params = 0;
    std::size_t state_bytes = 0;  // header + P||m||v of max_params, 4 KiB multiple
};

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

void need(const void* p, const char* what) {
    if (p == nullptr) throw tfb::ConfigError(std::string(what) + " must not be NULL");
}

// Device scratch for one host call, freed on every path.
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(std::size_t bytes) {
        if (bytes) tfb::cuda_check(cudaMalloc(&p, bytes), "cudaMalloc(host-call scratch)");
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

void h2d(void* d, const void* h, std::size_t bytes) {
    if (bytes) tfb::cuda_check(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice), "cudaMemcpy(H2D)");
}
void d2h(void* h, const void* d, std::size_t bytes) {
    if (bytes) tfb::cuda_check(cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost), "cudaMemcpy(D2H)");
}

}  // namespace

extern "C" {

int tfg_now_ns(int64_t* out) {
    return guard([&] {
        need(out, "out");
        *out = tfb::now_ns();
    });
}

int tfg_upscale16_host(const uint16_t* src, float* dst, uint64_t n, int dtype, int* all_finite) {
    return guard([&] {
        if (dtype != TFG_F16 && dtype != TFG_BF16) throw tfb::ConfigError("unknown 16-bit dtype");
        if (n > 0) {
            need(src, "src");
            need(dst, "dst");
        }
        DevBuf ds(2 * n), dd(4 * n), dc(sizeof(unsigned long long));
        tfb::cuda_check(cudaMemset(dc.p, 0, sizeof(unsigned long long)), "cudaMemset");
        h2d(ds.p, src, 2 * n);
        tfb::cuda_check(tfb::launch_widen16(ds.as<uint16_t>(), dd.as<float>(), n, dtype, dc.as<unsigned long long>(),
                                            nullptr),
                        "upscale16");
        unsigned long long bad = 0;
        d2h(dst, dd.p, 4 * n);
        d2h(&bad, dc.p, sizeof(bad));
        if (all_finite) *all_finite = bad == 0;
    });
}

int tfg_downscale16_host(const float* src, uint16_t* dst, uint64_t n, int dtype, uint64_t* overflows) {
    return guard([&] {
        if (dtype != TFG_F16 && dtype != TFG_BF16) throw tfb::ConfigError("unknown 16-bit dtype");
        if (n > 0) {
            need(src, "src");
            need(dst, "dst");
        }
        DevBuf ds(4 * n), dd(2 * n), dc(sizeof(unsigned long long));
        tfb::cuda_check(cudaMemset(dc.p, 0, sizeof(unsigned long long)), "cudaMemset");
        h2d(ds.p, src, 4 * n);
        tfb::cuda_check(tfb::launch_narrow16(ds.as<float>(), dd.as<uint16_t>(), n, dtype, dc.as<unsigned long long>(),
                                             nullptr),
                        "downscale16");
        unsigned long long over = 0;
        d2h(dst, dd.p, 2 * n);
        d2h(&over, dc.p, sizeof(over));
        if (overflows) *overflows = over;
    });
}

int tfg_f16_to_f32(uint16_t h, int dtype, float* out) {
    return guard([&] {
        if (dtype != TFG_F16 && dtype != TFG_BF16) throw tfb::ConfigError("unknown 16-bit dtype");
        need(out, "out");
        *out = tfb::widen16_scalar(h, dtype);
    });
}

int tfg_f32_to_f16(float x, int dtype, uint16_t* out) {
    return guard([&] {
        if (dtype != TFG_F16 && dtype != TFG_BF16) throw tfb::ConfigError("unknown 16-bit dtype");
        need(out, "out");
        *out = tfb::narrow16_scalar(x, dtype);
    });
}

int tfg_accumulate16_host(uint16_t* acc, const uint16_t* grads, uint64_t n, int dtype) {
    return guard([&] {
        if (dtype != TFG_F16 && dtype != TFG_BF16) throw tfb::ConfigError("unknown 16-bit dtype");
        if (n == 0) return;
        need(acc, "acc");
        need(grads, "grads");
        DevBuf da(2 * n), dg(2 * n), dout(2 * n);
        h2d(da.p, acc, 2 * n);
        h2d(dg.p, grads, 2 * n);
        const void* srcs[2] = {da.p, dg.p};
        tfb::cuda_check(tfb::launch_reduce_sum16(srcs, 2, n, dtype, dout.as<uint16_t>(), nullptr, nullptr),
                        "accumulate16");
        d2h(acc, dout.p, 2 * n);
    });
}

int tfg_adam_step_host(float* p, float* m, float* v, const float* g, uint64_t n, const tfg_adam_hyper* hyper,
                       uint64_t t) {
    return guard([&] {
        need(hyper, "hyper");
        tfb::AdamHyper h;
        h.lr = hyper->lr;
        h.beta1 = hyper->beta1;
        h.beta2 = hyper->beta2;
        h.eps = hyper->eps;
        h.weight_decay = hyper->weight_decay;
        tfb::AdamLaunch a;
        a.c = h.consts(t);  // Error for t < 1, ConfigError for bad hyperparameters (optimizer.hpp:24-30, 120-121)
        if (n == 0) return;
        need(p, "p");
        need(m, "m");
        need(v, "v");
        need(g, "g");
        DevBuf st(12 * n), dg(4 * n), d16(2 * n), dc(2 * sizeof(unsigned long long));
        float* dp = st.as<float>();
        h2d(dp, p, 4 * n);
        h2d(dp + n, m, 4 * n);
        h2d(dp + 2 * n, v, 4 * n);
        h2d(dg.p, g, 4 * n);
        tfb::cuda_check(cudaMemset(dc.p, 0, 2 * sizeof(unsigned long long)), "cudaMemset");
        a.p = dp;
        a.m = dp + n;
        a.v = dp + 2 * n;
        a.g = dg.p;
        a.grad_kind = TFG_F32;
        a.p16 = d16.as<uint16_t>();
        a.out_kind = TFG_F16;
        a.n = n;
        a.counters = dc.as<unsigned long long>();
        tfb::cuda_check(tfb::launch_adam_fused(a, nullptr), "adam_step");
        unsigned long long cnt[2] = {0, 0};
        d2h(cnt, dc.p, sizeof(cnt));
        // The reference rejects a non-finite gradient before mutating
        // (optimizer.hpp:123-127): the device copy is discarded, the caller's
        // arrays were never written.
        if (cnt[0] != 0) throw tfb::GradientOverflowError("adam_step: non-finite gradient");
        d2h(p, dp, 4 * n);
        d2h(m, dp + n, 4 * n);
        d2h(v, dp + 2 * n, 4 * n);
    });
}

// --- HostBufferPool (pool.hpp:35-161) ----------------------------------------

int tfg_pool_create(int slots, uint64_t max_params, tfg_pool** out) {
    return guard([&] {
        need(out, "out");
        auto p = std::make_unique<tfg_pool>();
        p->max_params = max_params;
        p->state_bytes = tfb::block_bytes_for(max_params);
        const std::size_t annex = tfb::round_up(4 * static_cast<std::size_t>(max_params), tfb::kPageBytes);
        p->pool = std::make_unique<tfb::HostBufferPool>(slots, p->state_bytes + annex, /*require_pinned=*/false);
        *out = p.release();
    });
}

int tfg_pool_destroy(tfg_pool* pool) {
    delete pool;
    return TFG_OK;
}

int tfg_pool_slot_count(tfg_pool* pool, int* out) {
    return guard([&] {
        need(pool, "pool");
        need(out, "out");
        *out = pool->pool->slot_count();
    });
}

int tfg_pool_try_reserve(tfg_pool* pool, uint32_t owner, int* slot_out) {
    return guard([&] {
        need(pool, "pool");
        need(slot_out, "slot_out");
        *slot_out = pool->pool->try_reserve(owner);
    });
}

int tfg_pool_find_cached(tfg_pool* pool, uint32_t owner, int* slot_out) {
    return guard([&] {
        need(pool, "pool");
        need(slot_out, "slot_out");
        *slot_out = pool->pool->find_cached(owner);
    });
}

int tfg_pool_transition(tfg_pool* pool, int slot, int op) {
    return guard([&] {
        need(pool, "pool");
        tfb::HostBufferPool& p = *pool->pool;
        switch (op) {
            case TFG_POOL_PREFETCH_DONE: p.prefetch_done(slot); break;
            case TFG_POOL_BEGIN_UPDATE: p.begin_update(slot); break;
            case TFG_POOL_END_UPDATE: p.end_update(slot); break;
            case TFG_POOL_BEGIN_FLUSH: p.begin_flush(slot); break;
            case TFG_POOL_FLUSH_DONE: p.flush_done(slot); break;
            case TFG_POOL_EVICT: p.evict(slot); break;
            default: throw tfb::ConfigError("unknown pool transition " + std::to_string(op));
        }
    });
}

int tfg_pool_query(tfg_pool* pool, int slot, int* state_out, uint32_t* owner_out) {
    return guard([&] {
        need(pool, "pool");
        if (state_out) *state_out = static_cast<int>(pool->pool->state(slot));
        if (owner_out) *owner_out = pool->pool->owner(slot);
    });
}

int tfg_pool_span(tfg_pool* pool, int slot, uint64_t params, int which, float** ptr_out, uint64_t* len_out) {
    return guard([&] {
        need(pool, "pool");
        need(ptr_out, "ptr_out");
        if (params > pool->max_params)
            throw tfb::Error("pool span: " + std::to_string(params) + " params exceed the slot capacity " +
                             std::to_string(pool->max_params));
        tfb::HostBlock& b = pool->pool->block(slot);
        if (which == 0) {
            *ptr_out = b.payload();
            if (len_out) *len_out = 3 * params;
        } else {
            *ptr_out = reinterpret_cast<float*>(b.base() + pool->state_bytes);
            if (len_out) *len_out = params;
        }
    });
}

// --- Subgroup residency (optimizer.hpp:39-73) --------------------------------

int tfg_subgroup_step(tfg_subgroup_meta* sg, int op, int arg) {
    return guard([&] {
        need(sg, "subgroup");
        tfb::Subgroup s;
        s.id = sg->id;
        s.param_count = sg->param_count;
        s.residency = static_cast<tfb::Residency>(sg->residency);
        s.tier = sg->tier;
        s.slot = sg->slot;
        s.step_count = sg->step_count;
        switch (op) {
            case TFG_SG_BEGIN_FLUSH: s.begin_flush(); break;
            case TFG_SG_FINISH_FLUSH: s.finish_flush(arg); break;
            case TFG_SG_BEGIN_PREFETCH: s.begin_prefetch(); break;
            case TFG_SG_FINISH_PREFETCH: s.finish_prefetch(arg); break;
            default: throw tfb::ConfigError("unknown residency step " + std::to_string(op));
        }
        sg->residency = static_cast<int32_t>(s.residency);
        sg->tier = s.tier;
        sg->slot = s.slot;
    });
}

}  // extern "C"
