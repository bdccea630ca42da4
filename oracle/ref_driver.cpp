// ref_driver.cpp — extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/tierflow), compiled in place by
// oracle/Makefile into oracle/_ref/libtierflow_ref.so. TEST INFRASTRUCTURE
// ONLY: it generates the golden fixtures (tests/golden/make_golden.py), pins
// the C restatement (oracle/tierflow_oracle.c) and is the reference arm /
// cpu_baseline of bench.py. Nothing here is shipped or measured as product.
#include <cstdint>
#include <cstring>
#include <exception>
#include <filesystem>
#include <memory>
#include <string>
#include <vector>

#include "tierflow/scheduler.hpp"

using namespace tierflow;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const GradientOverflowError& e) {
        g_err = e.what();
        return 7;
    } catch (const SchedulingBugError& e) {
        g_err = e.what();
        return 6;
    } catch (const PlacementInconsistencyError& e) {
        g_err = e.what();
        return 5;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 4;
    } catch (const FormatError& e) {
        g_err = e.what();
        return 3;
    } catch (const IoError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_adam_step(float* p, float* m, float* v, const float* g, uint64_t n, double lr, double b1, double b2,
                  double eps, double wd, uint64_t t, int threads) {
    return guard([&] {
        AdamHyper h;
        h.lr = lr;
        h.beta1 = b1;
        h.beta2 = b2;
        h.eps = eps;
        h.weight_decay = wd;
        adam_step(StateView{std::span<float>(p, n), std::span<float>(m, n), std::span<float>(v, n)},
                  std::span<const float>(g, n), h, t, threads);
    });
}

uint16_t ref_f32_to_f16(float f) { return f32_to_f16(f).bits; }
float ref_f16_to_f32(uint16_t h) { return f16_to_f32(f16{h}); }

int ref_upscale(const uint16_t* src, float* dst, uint64_t n, int* finite) {
    return guard([&] {
        *finite = upscale_f16_to_f32(std::span<const f16>(reinterpret_cast<const f16*>(src), n),
                                     std::span<float>(dst, n))
                      ? 1
                      : 0;
    });
}

int ref_downscale(const float* src, uint16_t* dst, uint64_t n, uint64_t* overflows) {
    return guard([&] {
        *overflows = downscale_f32_to_f16(std::span<const float>(src, n), std::span<f16>(reinterpret_cast<f16*>(dst), n));
    });
}

int ref_assign_subgroups(int M, const double* bw, int n, int* counts) {
    return guard([&] {
        const auto a = assign_subgroups(M, std::span<const double>(bw, static_cast<std::size_t>(n)));
        for (int i = 0; i < n; ++i) counts[i] = a.counts[static_cast<std::size_t>(i)];
    });
}

int ref_destination_plan(const uint32_t* order, int M, int capacity, const double* bw, int n, int* retain, int* tier,
                         int* alloc) {
    return guard([&] {
        const DestinationPlan plan(std::span<const SubgroupId>(order, static_cast<std::size_t>(M)), CachePlan{capacity},
                                   std::span<const double>(bw, static_cast<std::size_t>(n)));
        for (int k = 0; k < M; ++k) {
            const auto a = plan.assign_storage_tier(order[k]);
            retain[k] = a.host_retain ? 1 : 0;
            tier[k] = a.tier;
        }
        for (int i = 0; i < n; ++i) alloc[i] = plan.flush_allocation().counts[static_cast<std::size_t>(i)];
    });
}

void ref_synthetic_grads(uint16_t* out, uint64_t n, uint64_t seed, uint32_t sg, int iteration, int step) {
    SyntheticGradSource src{seed};
    src.fill(sg, iteration, step, std::span<f16>(reinterpret_cast<f16*>(out), n));
}

// GradBufferF16 over accum_steps steps of SyntheticGradSource (scheduler.hpp:365-376).
int ref_accumulated_grads(uint16_t* out, uint64_t n, uint64_t seed, uint32_t sg, int iteration, int steps) {
    return guard([&] {
        SyntheticGradSource src{seed};
        GradBufferF16 buf(sg, n);
        std::vector<f16> scratch(n);
        for (int s = 0; s < steps; ++s) {
            src.fill(sg, iteration, s, scratch);
            buf.accumulate(scratch);
        }
        std::memcpy(out, buf.values().data(), 2 * n);
    });
}

void ref_synthetic_params(float* out, uint64_t n, uint64_t seed, uint32_t sg) {
    for (uint64_t i = 0; i < n; ++i) out[i] = synthetic_param_init(seed, sg, i);
}

int ref_update_order(int iteration, const uint32_t* sorted, int M, int alternate, uint32_t* out) {
    return guard([&] {
        const auto p = UpdatePlan::make(iteration, std::vector<SubgroupId>(sorted, sorted + M), alternate != 0);
        for (int k = 0; k < M; ++k) out[k] = p.order[static_cast<std::size_t>(k)];
    });
}

int ref_retention_capacity(int caching, int pool_slots, int cache_slots, int M) {
    ScheduleOptions o;
    o.enable_caching = caching != 0;
    o.pool_slots = pool_slots;
    o.cache_slots = cache_slots;
    return o.retention_capacity(M);
}

// ---------------------------------------------------------------------------
// The real reference engine on configured tiers.

struct RefTierCfg {
    int kind;  // 0 local_dir, 1 remote_dir, 2 mem_throttled
    const char* root;
    double read_bps;
    double write_bps;
    int io_parallelism;
};

struct RefRunCfg {
    int n_subgroups;
    const uint64_t* params;  // per subgroup
    int n_tiers;
    const RefTierCfg* tiers;
    const double* fixed_ratio;  // NULL = bandwidth model
    int pool_slots;
    int cache_slots;
    int enable_caching;
    int multi_path;
    int atomic_rw;
    int update_threads;
    const char* lock_dir;
    uint64_t seed;
    int iterations;
    int accum_steps;
    double lr, beta1, beta2, eps, weight_decay;
    uint32_t skip_mask;  // bit i: skip iteration i's update (non-finite step)
    int skip_gradients;  // 0: the ZeRO-3 baseline flow (fp32 gradients through storage)
    int backward_once;   // 1: run_backward_sim at iteration 0 only, later phases reuse its gradients
                         //    (bench timing samples: the update's cost does not depend on their values)
};

struct RefIterOut {
    double update_seconds;
    double backward_seconds;
    uint64_t params_updated;
    uint64_t cache_hits;
    uint64_t overflows;
    int retained;
    int flush_allocation[8];
    uint64_t trace_begin;  // event index at run_update entry
    uint64_t trace_end;    // event index at run_update exit
};

struct RefEvent {
    int64_t ts;
    int32_t worker;
    int32_t kind;
    int64_t sg;
    int32_t tier;
    int32_t pad;
    uint64_t bytes;
};

// Runs init_and_flush_all + iterations x (run_backward_sim, run_update).
// states_out (optional): final P||m||v of every subgroup in id order.
int ref_run_engine(const RefRunCfg* c, RefIterOut* iters_out, float* states_out, RefEvent* events_out,
                   uint64_t events_cap, uint64_t* n_events) {
    return guard([&] {
        std::vector<std::shared_ptr<Tier>> tiers;
        for (int i = 0; i < c->n_tiers; ++i) {
            TierSpec s;
            s.tier_id = i;
            s.kind = static_cast<TierKind>(c->tiers[i].kind);
            s.root = c->tiers[i].root ? c->tiers[i].root : ("mem" + std::to_string(i));
            s.read_bw = c->tiers[i].read_bps;
            s.write_bw = c->tiers[i].write_bps;
            s.io_parallelism = c->tiers[i].io_parallelism > 0 ? c->tiers[i].io_parallelism : 1;
            tiers.push_back(std::make_shared<Tier>(s));
        }
        ScheduleOptions o;
        o.pool_slots = c->pool_slots;
        o.cache_slots = c->cache_slots;
        o.enable_caching = c->enable_caching != 0;
        o.skip_gradients = c->skip_gradients != 0;
        o.atomic_rw = c->atomic_rw != 0;
        o.multi_path = c->multi_path != 0;
        o.update_threads = c->update_threads;
        if (c->lock_dir) o.lock_dir = c->lock_dir;
        AdamHyper h;
        h.lr = c->lr;
        h.beta1 = c->beta1;
        h.beta2 = c->beta2;
        h.eps = c->eps;
        h.weight_decay = c->weight_decay;
        EventTrace trace;
        auto w = std::make_unique<OffloadWorker>(0, tiers, o, h, trace);
        if (c->fixed_ratio) w->set_fixed_ratio(std::vector<double>(c->fixed_ratio, c->fixed_ratio + c->n_tiers));
        for (int i = 0; i < c->n_subgroups; ++i) w->add_subgroup(static_cast<SubgroupId>(i), c->params[i]);
        w->init_and_flush_all(c->seed);
        SyntheticGradSource src{c->seed};
        for (int it = 0; it < c->iterations; ++it) {
            RefIterOut r{};
            const auto b0 = std::chrono::steady_clock::now();
            if (it == 0 || !c->backward_once) w->run_backward_sim(it, src, c->accum_steps);
            r.backward_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - b0).count();
            r.trace_begin = r.trace_end = trace.size();
            if (!((c->skip_mask >> it) & 1u)) {
                const auto u0 = std::chrono::steady_clock::now();
                const PhaseStats st = w->run_update(it);
                r.trace_end = trace.size();
                r.update_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - u0).count();
                r.params_updated = st.params_updated;
                r.cache_hits = st.cache_hits;
                r.overflows = st.downscale_overflows;
                r.retained = st.retained;
                for (std::size_t t = 0; t < st.flush_allocation.size() && t < 8; ++t)
                    r.flush_allocation[t] = st.flush_allocation[t];
            }
            if (iters_out) iters_out[it] = r;
        }
        if (states_out) {
            std::size_t off = 0;
            for (int i = 0; i < c->n_subgroups; ++i) {
                const auto s = w->read_current_state(static_cast<SubgroupId>(i));
                std::memcpy(states_out + off, s.data(), s.size() * sizeof(float));
                off += s.size();
            }
        }
        const auto ev = trace.snapshot();
        if (n_events) *n_events = ev.size();
        if (events_out) {
            const int64_t t0 = ev.empty() ? 0 : ev.front().timestamp_ns;
            for (std::size_t i = 0; i < ev.size() && i < events_cap; ++i)
                events_out[i] = RefEvent{ev[i].timestamp_ns - t0, ev[i].worker_id, static_cast<int32_t>(ev[i].kind),
                                         ev[i].subgroup_id, ev[i].tier_id, 0, ev[i].bytes};
        }
        w.reset();
        for (int i = 0; i < c->n_tiers; ++i)
            if (c->tiers[i].kind != 2 && c->tiers[i].root) {
                std::error_code ec;
                for (int s = 0; s < c->n_subgroups; ++s) tiers[static_cast<std::size_t>(i)]->remove_subgroup(static_cast<SubgroupId>(s));
            }
    });
}

}  // extern "C"
