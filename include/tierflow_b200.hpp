// tierflow_b200.hpp — header-only C++ adapter over the C ABI, shaped like the
// reference engine's own C++ API (/root/reference/proj/include/tierflow/), so
// a reference caller switches engines by including this header and linking
// libtierflow_b200.so. Only the hot-path surface is mirrored:
// Tier / TierSpec (tier.hpp:43-241), EventTrace (trace.hpp:77-171),
// ScheduleOptions / AdamHyper / OffloadWorker / PhaseStats
// (scheduler.hpp:32-864, optimizer.hpp:17-31), assign_subgroups
// (placement.hpp:30). Errors are rethrown as the reference's exception types
// (common.hpp:36-78), re-declared here under tierflow_b200::.
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "tierflow_b200.h"

namespace tierflow_b200 {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IoError : Error { using Error::Error; };
struct FormatError : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
struct PlacementInconsistencyError : Error { using Error::Error; };
struct SchedulingBugError : Error { using Error::Error; };
struct GradientOverflowError : Error { using Error::Error; };
struct CudaError : Error { using Error::Error; };

inline void check(int rc) {
    if (rc == TFG_OK) return;
    const std::string msg = tfg_last_error();
    switch (rc) {
        case TFG_IO_ERROR: throw IoError(msg);
        case TFG_FORMAT_ERROR: throw FormatError(msg);
        case TFG_CONFIG_ERROR: throw ConfigError(msg);
        case TFG_PLACEMENT_INCONSISTENCY: throw PlacementInconsistencyError(msg);
        case TFG_SCHEDULING_BUG: throw SchedulingBugError(msg);
        case TFG_GRADIENT_OVERFLOW: throw GradientOverflowError(msg);
        case TFG_CUDA_ERROR: throw CudaError(msg);
        default: throw Error(msg);
    }
}

using SubgroupId = std::uint32_t;
using TierId = int;
using WorkerId = int;

enum class TierKind : int { local_dir = TFG_LOCAL_DIR, remote_dir = TFG_REMOTE_DIR,
                            mem_throttled = TFG_MEM_THROTTLED, host_dram = TFG_HOST_DRAM };

struct TierSpec {
    TierId tier_id = 0;
    TierKind kind = TierKind::local_dir;
    std::string root;
    double read_bw = 0.0;
    double write_bw = 0.0;
    int io_parallelism = 1;
    bool persistent = false;
    int lock_width = 1;
    bool direct_io = true;
    int lock_device = 0;  // > 0: semaphore shared with every tier of the same physical device
    std::uint64_t capacity_bytes = 0;  // 0: unlimited; caps the subgroups Eq. 1 places here
};

struct IoStats {
    std::uint64_t bytes = 0;
    double seconds = 0.0;
};

struct AllocationVector {
    std::vector<int> counts;
    int total = 0;
};

inline AllocationVector assign_subgroups(int M, const std::vector<double>& bandwidths) {
    AllocationVector a;
    a.counts.assign(bandwidths.size(), 0);
    a.total = M;
    check(tfg_assign_subgroups(M, bandwidths.data(), static_cast<int>(bandwidths.size()), a.counts.data()));
    return a;
}

class EventTrace {
public:
    EventTrace() { check(tfg_trace_create(&h_)); }
    ~EventTrace() { tfg_trace_destroy(h_); }
    EventTrace(const EventTrace&) = delete;
    EventTrace& operator=(const EventTrace&) = delete;
    tfg_trace* handle() const { return h_; }
    std::size_t size() const {
        std::uint64_t n = 0;
        check(tfg_trace_size(h_, &n));
        return n;
    }
    std::vector<tfg_event> snapshot_from(std::size_t begin) const {
        std::vector<tfg_event> out(size() > begin ? size() - begin : 0);
        std::uint64_t n = 0;
        if (!out.empty()) check(tfg_trace_copy(h_, begin, out.data(), out.size(), &n));
        out.resize(n);
        return out;
    }
    std::vector<tfg_event> snapshot() const { return snapshot_from(0); }
    void write(const std::string& path) const { check(tfg_trace_write(h_, path.c_str())); }

private:
    tfg_trace* h_ = nullptr;
};

class Tier {
public:
    explicit Tier(TierSpec spec) : spec_(std::move(spec)) {
        tfg_tier_spec s{spec_.tier_id, static_cast<int32_t>(spec_.kind), spec_.root.c_str(), spec_.read_bw,
                        spec_.write_bw, spec_.io_parallelism, spec_.persistent ? 1 : 0, spec_.lock_width,
                        spec_.direct_io ? 1 : 0, spec_.lock_device, spec_.capacity_bytes};
        check(tfg_tier_create(&s, &h_));
    }
    ~Tier() { tfg_tier_destroy(h_); }
    Tier(const Tier&) = delete;
    Tier& operator=(const Tier&) = delete;
    tfg_tier* handle() const { return h_; }
    TierId id() const { return spec_.tier_id; }

    IoStats write_subgroup(SubgroupId id, std::uint64_t params, const std::vector<float>& state) {
        if (state.size() != 3 * params) throw Error("write_subgroup: state length mismatch");
        IoStats st;
        check(tfg_tier_write_subgroup(h_, id, params, state.data(), &st.bytes, &st.seconds));
        return st;
    }
    IoStats read_subgroup(SubgroupId id, std::uint64_t params, std::vector<float>& state) {
        state.resize(3 * params);
        IoStats st;
        check(tfg_tier_read_subgroup(h_, id, params, state.data(), &st.bytes, &st.seconds));
        return st;
    }
    bool has_subgroup(SubgroupId id) const {
        int out = 0;
        check(tfg_tier_has_subgroup(h_, id, &out));
        return out != 0;
    }
    void remove_subgroup(SubgroupId id) { check(tfg_tier_remove_subgroup(h_, id)); }
    void set_throttle_rates(double r, double w) { check(tfg_tier_set_throttle_rates(h_, r, w)); }
    std::pair<double, double> probe_bandwidth(std::uint64_t bytes, int reps) {
        double r = 0, w = 0;
        int lc = 0;
        check(tfg_tier_probe(h_, bytes, reps, &r, &w, &lc));
        return {r, w};
    }

private:
    TierSpec spec_;
    tfg_tier* h_ = nullptr;
};

struct ScheduleOptions {
    int pool_slots = 4;
    int cache_slots = -1;
    bool enable_caching = true;
    bool skip_gradients = true;
    bool atomic_rw = true;
    bool multi_path = true;
    std::string lock_dir;
    int update_threads = 1;
    double deadlock_timeout_s = 30.0;
    std::uint64_t update_pad_ns = 0;
};

struct AdamHyper {
    double lr = 1e-3;
    double beta1 = 0.9;
    double beta2 = 0.999;
    double eps = 1e-8;
    double weight_decay = 0.0;
};

struct DeviceOptions {
    int device = 0;
    int grad_dtype = TFG_F16;
    int param_dtype = TFG_F16;
    int device_buffers = 3;
    bool zero_copy = false;
    int d2h_split = 1;
    int hbm_retain = 1;  // 0 off, 1 host slot kept, 2 HBM cache (see tfg_device_options)
    int h2d_split = 1;
    int hbm_cache_slots = 0;  // hbm_retain 2: HBM part of C (0: all)
    bool host_grads = false;  // 16-bit gradients / working params in pinned host memory (ABI 3)
};

using PhaseStats = tfg_phase_stats;

class OffloadWorker {
public:
    OffloadWorker(WorkerId id, const std::vector<std::shared_ptr<Tier>>& tiers, const ScheduleOptions& o,
                  const AdamHyper& h, EventTrace& trace, const DeviceOptions& d = DeviceOptions{})
        : tiers_(tiers) {
        std::vector<tfg_tier*> th;
        for (const auto& t : tiers_) th.push_back(t->handle());
        tfg_schedule_options so{o.pool_slots, o.cache_slots, o.enable_caching, o.skip_gradients, o.atomic_rw,
                                o.multi_path, o.lock_dir.c_str(), o.update_threads, o.deadlock_timeout_s,
                                o.update_pad_ns};
        tfg_adam_hyper ah{h.lr, h.beta1, h.beta2, h.eps, h.weight_decay};
        tfg_device_options dv{d.device, d.grad_dtype, d.param_dtype, d.device_buffers, d.zero_copy ? 1 : 0,
                              d.d2h_split, d.hbm_retain, d.h2d_split, d.hbm_cache_slots, d.host_grads ? 1 : 0};
        check(tfg_engine_create(id, th.data(), static_cast<int>(th.size()), &so, &ah, trace.handle(), &dv, &h_));
    }
    ~OffloadWorker() { tfg_engine_destroy(h_); }
    OffloadWorker(const OffloadWorker&) = delete;
    OffloadWorker& operator=(const OffloadWorker&) = delete;

    void set_alpha(double a) { check(tfg_engine_set_alpha(h_, a)); }
    void set_fixed_ratio(const std::vector<double>& r) {
        check(tfg_engine_set_fixed_ratio(h_, r.data(), static_cast<int>(r.size())));
    }
    void set_cache_slots(int c) { check(tfg_engine_set_cache_slots(h_, c)); }
    void add_subgroup(SubgroupId id, std::uint64_t params) {
        check(tfg_engine_add_subgroup(h_, id, params));
        params_.push_back({id, params});
    }
    void init_and_flush_all(std::uint64_t seed) { check(tfg_engine_init_and_flush_all(h_, seed)); }
    void run_backward_sim(int iteration, std::uint64_t seed, int accum_steps) {
        check(tfg_engine_run_backward_sim(h_, iteration, seed, accum_steps));
    }
    bool gradients_finite() {
        int out = 0;
        check(tfg_engine_gradients_finite(h_, &out));
        return out != 0;
    }
    PhaseStats run_update(int iteration) {
        PhaseStats st{};
        check(tfg_engine_run_update(h_, iteration, &st));
        return st;
    }
    int wait_host_resident(SubgroupId id) {
        int slot = -1;
        check(tfg_engine_wait_host_resident(h_, id, &slot));
        return slot;
    }
    // The backward's output buffer of a subgroup (16-bit, param_count elements).
    void* grad_buffer(SubgroupId id) {
        void* p = nullptr;
        check(tfg_engine_grad_buffer(h_, id, &p));
        return p;
    }
    void bind_grad_buffer(SubgroupId id, void* device_ptr) { check(tfg_engine_bind_grad_buffer(h_, id, device_ptr)); }
    // The stream that produces the gradients; updates are ordered after it.
    void set_producer_stream(void* cuda_stream) { check(tfg_engine_set_producer_stream(h_, cuda_stream)); }
    // The reduce-scatter fused into the update: every rank's contribution to
    // this subgroup (e.g. CUDA IPC-mapped peer buffers), summed in rank order.
    void bind_grad_sources(SubgroupId id, const std::vector<const void*>& sources) {
        check(tfg_engine_bind_grad_sources(h_, id, sources.data(), static_cast<int>(sources.size())));
    }
    // 16-bit working params (the reference's shadow_), device-resident.
    void* params16_buffer(SubgroupId id) {
        void* p = nullptr;
        check(tfg_engine_params16_buffer(h_, id, &p));
        return p;
    }
    std::vector<std::uint16_t> read_params16(SubgroupId id) {
        std::uint64_t n = 0;
        for (const auto& [sid, p] : params_)
            if (sid == id) n = p;
        std::vector<std::uint16_t> out(n);
        check(tfg_engine_read_params16(h_, id, out.data()));
        return out;
    }
    std::vector<float> read_current_state(SubgroupId id) {
        std::uint64_t n = 0;
        for (const auto& [sid, p] : params_)
            if (sid == id) n = p;
        std::vector<float> out(3 * n);
        check(tfg_engine_read_state(h_, id, out.data()));
        return out;
    }

private:
    std::vector<std::shared_ptr<Tier>> tiers_;
    std::vector<std::pair<SubgroupId, std::uint64_t>> params_;
    tfg_engine* h_ = nullptr;
};

}  // namespace tierflow_b200
