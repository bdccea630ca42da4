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

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

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

// Staging for the host-span calls. The caller's arrays are pageable
// (std::vector in the reference's API), so every copy goes through two
// pinned chunks: chunk i+1 is memcpy'd on the CPU while chunk i is on the
// link. Device scratch is kept across calls (a cudaMalloc/cudaFree pair per
// call costs more than the copies at the reference suites' sizes); a call
// larger than kKeepBytes gets its own scratch, freed on return. One stage
// per device, calls on it serialised.
class HostStage {
   public:
    static constexpr std::size_t kChunk = std::size_t{8} << 20;
    static constexpr std::size_t kKeepBytes = std::size_t{1} << 30;
    static constexpr int kScratch = 5;  // 4 data arrays + the counters

    static HostStage& get() {
        int dev = 0;
        tfb::cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
        static std::mutex map_mu;
        static std::map<int, std::unique_ptr<HostStage>> stages;
        std::lock_guard<std::mutex> g(map_mu);
        auto& s = stages[dev];
        if (!s) s.reset(new HostStage());
        return *s;
    }

    std::mutex mu;  // held for the whole host call
    cudaStream_t stream = nullptr;

    // Device scratch i of at least `bytes` (valid until the call returns).
    void* scratch(int i, std::size_t bytes) {
        if (bytes == 0) return nullptr;
        if (bytes > kKeepBytes) {
            void* p = nullptr;
            tfb::cuda_check(cudaMalloc(&p, bytes), "cudaMalloc(host-call scratch)");
            oversize_.push_back(p);
            return p;
        }
        if (cap_[i] < bytes) {
            if (dev_[i]) tfb::cuda_check(cudaFree(dev_[i]), "cudaFree");
            dev_[i] = nullptr;
            cap_[i] = 0;
            tfb::cuda_check(cudaMalloc(&dev_[i], bytes), "cudaMalloc(host-call scratch)");
            cap_[i] = bytes;
        }
        return dev_[i];
    }

    // Frees this call's oversize scratch (after the stream has drained).
    void end_call() {
        for (void* p : oversize_) cudaFree(p);
        oversize_.clear();
    }

    void h2d(void* d, const void* h, std::size_t bytes) {
        auto* dst = static_cast<char*>(d);
        auto* src = static_cast<const char*>(h);
        for (std::size_t off = 0, i = 0; off < bytes; off += kChunk, ++i) {
            const std::size_t n = std::min(kChunk, bytes - off);
            const int b = static_cast<int>(i & 1);
            tfb::cuda_check(cudaEventSynchronize(done_[b]), "cudaEventSynchronize");  // its last DMA has read it
            std::memcpy(pin_[b], src + off, n);
            tfb::cuda_check(cudaMemcpyAsync(dst + off, pin_[b], n, cudaMemcpyHostToDevice, stream), "cudaMemcpyAsync");
            tfb::cuda_check(cudaEventRecord(done_[b], stream), "cudaEventRecord");
        }
    }

    // Copies after the work queued on `stream`; returns with the host array written.
    void d2h(void* h, const void* d, std::size_t bytes) {
        auto* dst = static_cast<char*>(h);
        auto* src = static_cast<const char*>(d);
        const std::size_t chunks = (bytes + kChunk - 1) / kChunk;
        auto issue = [&](std::size_t i) {
            const std::size_t off = i * kChunk, n = std::min(kChunk, bytes - off);
            const int b = static_cast<int>(i & 1);
            tfb::cuda_check(cudaMemcpyAsync(pin_[b], src + off, n, cudaMemcpyDeviceToHost, stream), "cudaMemcpyAsync");
            tfb::cuda_check(cudaEventRecord(done_[b], stream), "cudaEventRecord");
        };
        if (chunks > 0) issue(0);
        for (std::size_t i = 0; i < chunks; ++i) {
            const int b = static_cast<int>(i & 1);
            tfb::cuda_check(cudaEventSynchronize(done_[b]), "cudaEventSynchronize");
            if (i + 1 < chunks) issue(i + 1);  // into the other chunk while this one is copied out
            const std::size_t off = i * kChunk;
            std::memcpy(dst + off, pin_[b], std::min(kChunk, bytes - off));
        }
    }

    void sync() { tfb::cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize"); }

   private:
    HostStage() {
        tfb::cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
        for (int b = 0; b < 2; ++b) {
            tfb::cuda_check(cudaHostAlloc(&pin_[b], kChunk, cudaHostAllocPortable), "cudaHostAlloc(staging)");
            tfb::cuda_check(cudaEventCreateWithFlags(&done_[b], cudaEventDisableTiming), "cudaEventCreate");
            tfb::cuda_check(cudaEventRecord(done_[b], stream), "cudaEventRecord");
        }
    }
    // Never destroyed: process-lifetime resources, released with the context.
    void* pin_[2] = {nullptr, nullptr};
    cudaEvent_t done_[2] = {nullptr, nullptr};
    void* dev_[kScratch] = {};
    std::size_t cap_[kScratch] = {};
    std::vector<void*> oversize_;
};

// One host call on the stage: serialised, drained and oversize scratch freed on every path.
struct StagedCall {
    HostStage& st;
    std::lock_guard<std::mutex> lock;
    StagedCall() : st(HostStage::get()), lock(st.mu) {}
    ~StagedCall() {
        cudaStreamSynchronize(st.stream);
        st.end_call();
    }
    template <class T>
    T* scratch(int i, std::size_t bytes) { return static_cast<T*>(st.scratch(i, bytes)); }
};

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
        StagedCall c;
        auto* ds = c.scratch<uint16_t>(0, 2 * n);
        auto* dd = c.scratch<float>(1, 4 * n);
        auto* dc = c.scratch<unsigned long long>(4, sizeof(unsigned long long));
        tfb::cuda_check(cudaMemsetAsync(dc, 0, sizeof(unsigned long long), c.st.stream), "cudaMemsetAsync");
        c.st.h2d(ds, src, 2 * n);
        tfb::cuda_check(tfb::launch_widen16(ds, dd, n, dtype, dc, c.st.stream), "upscale16");
        unsigned long long bad = 0;
        c.st.d2h(dst, dd, 4 * n);
        c.st.d2h(&bad, dc, sizeof(bad));
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
        StagedCall c;
        auto* ds = c.scratch<float>(0, 4 * n);
        auto* dd = c.scratch<uint16_t>(1, 2 * n);
        auto* dc = c.scratch<unsigned long long>(4, sizeof(unsigned long long));
        tfb::cuda_check(cudaMemsetAsync(dc, 0, sizeof(unsigned long long), c.st.stream), "cudaMemsetAsync");
        c.st.h2d(ds, src, 4 * n);
        tfb::cuda_check(tfb::launch_narrow16(ds, dd, n, dtype, dc, c.st.stream), "downscale16");
        unsigned long long over = 0;
        c.st.d2h(dst, dd, 2 * n);
        c.st.d2h(&over, dc, sizeof(over));
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
        StagedCall c;
        auto* da = c.scratch<uint16_t>(0, 2 * n);
        auto* dg = c.scratch<uint16_t>(1, 2 * n);
        auto* dout = c.scratch<uint16_t>(2, 2 * n);
        c.st.h2d(da, acc, 2 * n);
        c.st.h2d(dg, grads, 2 * n);
        const void* srcs[2] = {da, dg};
        tfb::cuda_check(tfb::launch_reduce_sum16(srcs, 2, n, dtype, dout, nullptr, c.st.stream), "accumulate16");
        c.st.d2h(acc, dout, 2 * n);
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
        StagedCall c;
        float* dp = c.scratch<float>(0, 12 * n);
        auto* dg = c.scratch<float>(1, 4 * n);
        auto* d16 = c.scratch<uint16_t>(2, 2 * n);
        auto* dc = c.scratch<unsigned long long>(4, 2 * sizeof(unsigned long long));
        c.st.h2d(dp, p, 4 * n);
        c.st.h2d(dp + n, m, 4 * n);
        c.st.h2d(dp + 2 * n, v, 4 * n);
        c.st.h2d(dg, g, 4 * n);
        tfb::cuda_check(cudaMemsetAsync(dc, 0, 2 * sizeof(unsigned long long), c.st.stream), "cudaMemsetAsync");
        a.p = dp;
        a.m = dp + n;
        a.v = dp + 2 * n;
        a.g = dg;
        a.grad_kind = TFG_F32;
        a.p16 = d16;
        a.out_kind = TFG_F16;
        a.n = n;
        a.counters = dc;
        tfb::cuda_check(tfb::launch_adam_fused(a, c.st.stream), "adam_step");
        unsigned long long cnt[2] = {0, 0};
        c.st.d2h(cnt, dc, sizeof(cnt));
        // The reference rejects a non-finite gradient before mutating
        // (optimizer.hpp:123-127): the device copy is discarded, the caller's
        // arrays were never written.
        if (cnt[0] != 0) throw tfb::GradientOverflowError("adam_step: non-finite gradient");
        c.st.d2h(p, dp, 4 * n);
        c.st.d2h(m, dp + n, 4 * n);
        c.st.d2h(v, dp + 2 * n, 4 * n);
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
