// tierflow/compat.hpp — the reference engine's C++ header API (namespace
// tierflow, /root/reference/proj/include/tierflow/*.hpp) re-declared over the
// B200 library's C ABI (include/tierflow_b200.h). A reference caller switches
// engines by putting include/tierflow_compat/ first on its include path and
// linking libtierflow_b200.so: `#include "tierflow/scheduler.hpp"` then binds
// OffloadWorker, Tier, EventTrace, HostBufferPool, adam_step, ... to the
// B200 engine (CUDA streams, pinned staging, sm_100a kernels). Nothing here
// computes: every call crosses the C ABI into the library's own objects.
//
// Covered (tests/dropin/ compiles the reference's own suites against it):
// common.hpp, fp16.hpp (f16), precision.hpp, optimizer.hpp, placement.hpp
// (TierObservation, assign_subgroups), trace.hpp, tier.hpp, tier_lock.hpp,
// pool.hpp, scheduler.hpp. Not covered: config.hpp / harness.hpp /
// report.hpp (the reference's JSON driver, out of scope per SURVEY.md §2).
//
// Differences a caller can observe, all by design of the B200 engine:
//  * adam_step's `threads` argument is accepted and ignored (the step runs on
//    the GPU); the numeric results are bit-identical to the reference.
//  * OffloadWorker::grad_buffer(id) returns a host view of the device
//    gradient buffer, read on every call (the gradients live in HBM); edits
//    through it are written back before the next gradients_finite() or
//    run_update().
//  * enqueue_prefetch / enqueue_flush futures are deferred waits on engine
//    tickets: the transfer is queued at the call, get() waits for it.
#pragma once

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdint>
#include <filesystem>
#include <future>
#include <istream>
#include <map>
#include <memory>
#include <optional>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include <unistd.h>  // the reference headers bring POSIX in (tier.hpp, tier_lock.hpp)

#include "../../tierflow_b200.h"

namespace tierflow {

// --- common.hpp ---------------------------------------------------------------

using SubgroupId = std::uint32_t;
using TierId = int;
using WorkerId = int;
inline constexpr TierId kNoTier = -1;

class Error : public std::runtime_error {
public:
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};
class IoError : public Error { public: using Error::Error; };
class FormatError : public Error { public: using Error::Error; };
class ConfigError : public Error { public: using Error::Error; };
class PlacementInconsistencyError : public Error { public: using Error::Error; };
class SchedulingBugError : public Error { public: using Error::Error; };
class GradientOverflowError : public Error { public: using Error::Error; };
class CudaError : public Error { public: using Error::Error; };

namespace detail {
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
}  // namespace detail

inline std::int64_t now_ns() {
    std::int64_t t = 0;
    detail::check(tfg_now_ns(&t));
    return t;
}

struct IoStats {
    std::uint64_t bytes = 0;
    double seconds = 0.0;
    double bytes_per_second() const { return seconds > 0.0 ? static_cast<double>(bytes) / seconds : 0.0; }
};

// --- fp16.hpp / precision.hpp ---------------------------------------------------

struct f16 {
    std::uint16_t bits = 0;
    friend bool operator==(f16 a, f16 b) { return a.bits == b.bits; }
    friend bool operator!=(f16 a, f16 b) { return a.bits != b.bits; }
};
static_assert(sizeof(f16) == 2);

inline bool f16_is_finite(f16 h) { return (h.bits & 0x7C00u) != 0x7C00u; }
inline bool f16_is_nan(f16 h) { return (h.bits & 0x7C00u) == 0x7C00u && (h.bits & 0x03FFu) != 0; }

inline bool upscale_f16_to_f32(std::span<const f16> src, std::span<float> dst) {
    if (src.size() != dst.size()) throw Error("upscale: length mismatch");
    int finite = 1;
    detail::check(tfg_upscale16_host(reinterpret_cast<const std::uint16_t*>(src.data()), dst.data(), src.size(),
                                     TFG_F16, &finite));
    return finite != 0;
}

inline std::size_t downscale_f32_to_f16(std::span<const float> src, std::span<f16> dst) {
    if (src.size() != dst.size()) throw Error("downscale: length mismatch");
    std::uint64_t over = 0;
    detail::check(tfg_downscale16_host(src.data(), reinterpret_cast<std::uint16_t*>(dst.data()), src.size(), TFG_F16,
                                       &over));
    return static_cast<std::size_t>(over);
}

inline float f16_to_f32(f16 h) {
    float out = 0.0f;
    detail::check(tfg_f16_to_f32(h.bits, TFG_F16, &out));
    return out;
}

inline f16 f32_to_f16(float x) {
    f16 out;
    detail::check(tfg_f32_to_f16(x, TFG_F16, &out.bits));
    return out;
}

inline bool all_finite(std::span<const f16> values) {
    return std::all_of(values.begin(), values.end(), [](f16 v) { return f16_is_finite(v); });
}

// Host 16-bit gradient buffer (precision.hpp:44-82). Standalone it is the
// reference's accumulation buffer, the fp32 add-and-round done by the
// library's reduce kernel; OffloadWorker::grad_buffer returns one as a host
// snapshot of the engine's HBM gradient.
class GradBufferF16 {
public:
    GradBufferF16() = default;
    GradBufferF16(SubgroupId id, std::size_t length) : id_(id), values_(length) {}
    SubgroupId id() const { return id_; }
    std::size_t size() const { return values_.size(); }
    int accumulation_steps() const { return steps_; }
    std::span<const f16> values() const { return values_; }
    std::span<f16> mutable_values() { return values_; }
    bool finite() const { return all_finite(values_); }

    void reset() {
        std::fill(values_.begin(), values_.end(), f16{});
        steps_ = 0;
    }
    void accumulate(std::span<const f16> grads) {
        if (grads.size() != values_.size()) throw Error("grad accumulate: length mismatch");
        if (steps_ == 0)
            std::copy(grads.begin(), grads.end(), values_.begin());
        else
            detail::check(tfg_accumulate16_host(reinterpret_cast<std::uint16_t*>(values_.data()),
                                                reinterpret_cast<const std::uint16_t*>(grads.data()), values_.size(),
                                                TFG_F16));
        ++steps_;
    }

private:
    friend class OffloadWorker;
    SubgroupId id_ = 0;
    std::vector<f16> values_;
    int steps_ = 0;
};

// --- optimizer.hpp ----------------------------------------------------------------

struct AdamHyper {
    double lr = 1e-3;
    double beta1 = 0.9;
    double beta2 = 0.999;
    double eps = 1e-8;
    double weight_decay = 0.0;

    tfg_adam_hyper c() const { return tfg_adam_hyper{lr, beta1, beta2, eps, weight_decay}; }
    void validate() const {  // the library's own check (optimizer.hpp:24-30)
        const tfg_adam_hyper h = c();
        detail::check(tfg_adam_step_host(nullptr, nullptr, nullptr, nullptr, 0, &h, 1));
    }
};

enum class Residency { host_cached = 0, in_flight = 1, on_tier = 2 };

struct Subgroup {
    SubgroupId id = 0;
    std::uint64_t param_count = 0;
    Residency residency = Residency::host_cached;
    TierId tier = kNoTier;
    int slot = -1;
    std::uint64_t step_count = 0;

    void begin_flush() { step(TFG_SG_BEGIN_FLUSH, 0); }
    void finish_flush(TierId dest) { step(TFG_SG_FINISH_FLUSH, dest); }
    void begin_prefetch() { step(TFG_SG_BEGIN_PREFETCH, 0); }
    void finish_prefetch(int pool_slot) { step(TFG_SG_FINISH_PREFETCH, pool_slot); }

private:
    void step(int op, int arg) {
        tfg_subgroup_meta m{id, static_cast<int32_t>(residency), tier, slot, param_count, step_count};
        detail::check(tfg_subgroup_step(&m, op, arg));
        residency = static_cast<Residency>(m.residency);
        tier = m.tier;
        slot = m.slot;
    }
};

struct StateView {
    std::span<float> params;
    std::span<float> momentum;
    std::span<float> variance;

    static StateView from_contiguous(std::span<float> state, std::uint64_t param_count) {
        if (state.size() != 3 * param_count) throw Error("state view: length mismatch");
        return StateView{state.subspan(0, param_count), state.subspan(param_count, param_count),
                         state.subspan(2 * param_count, param_count)};
    }
};

// The fused sm_100a kernel on the caller's host arrays (staged through HBM).
// `threads` is accepted for API parity: the step runs on the GPU.
inline void adam_step(StateView state, std::span<const float> grads, const AdamHyper& h, std::uint64_t t,
                      int threads = 1) {
    (void)threads;
    const std::size_t n = state.params.size();
    if (state.momentum.size() != n || state.variance.size() != n)
        throw Error("adam_step: state tensor length mismatch");
    if (grads.size() != n) throw Error("adam_step: gradient length mismatch");
    const tfg_adam_hyper hy = h.c();
    detail::check(tfg_adam_step_host(state.params.data(), state.momentum.data(), state.variance.data(), grads.data(),
                                     n, &hy, t));
}

inline double update_throughput_mparams(std::uint64_t params_updated, double wall_seconds) {
    if (!(wall_seconds > 0.0)) throw Error("update_throughput: wall time must be > 0");
    return static_cast<double>(params_updated) / wall_seconds / 1e6;
}

// --- placement.hpp ----------------------------------------------------------------

struct AllocationVector {
    std::vector<int> counts;
    int total = 0;
};

inline AllocationVector assign_subgroups(int M, std::span<const double> bandwidths) {
    AllocationVector a;
    a.counts.assign(bandwidths.size(), 0);
    a.total = M;
    detail::check(tfg_assign_subgroups(M, bandwidths.data(), static_cast<int>(bandwidths.size()), a.counts.data()));
    return a;
}

struct TierObservation {
    std::uint64_t read_transfers = 0;
    double read_bytes = 0.0;
    double read_seconds = 0.0;
    std::uint64_t write_transfers = 0;
    double write_bytes = 0.0;
    double write_seconds = 0.0;
};

// Per-tier bandwidth EMA (placement.hpp:102-162); init validates alpha and
// update_bandwidth_estimates runs in the library.
struct BandwidthEstimate {
    struct PerTier {
        double read_bw = 0.0;
        double write_bw = 0.0;
        std::uint64_t sample_count = 0;
    };
    std::vector<PerTier> tiers;
    double alpha = 0.5;

    static BandwidthEstimate init(std::span<const double> read_bw, std::span<const double> write_bw, double alpha) {
        detail::check(tfg_update_bandwidth_estimates(nullptr, nullptr, nullptr, 0, alpha, nullptr, 0));
        if (read_bw.size() != write_bw.size()) throw ConfigError("bandwidth estimate: tier count mismatch");
        BandwidthEstimate est;
        est.alpha = alpha;
        for (std::size_t i = 0; i < read_bw.size(); ++i) est.tiers.push_back(PerTier{read_bw[i], write_bw[i], 0});
        return est;
    }
    double effective(std::size_t i) const { return std::min(tiers.at(i).read_bw, tiers.at(i).write_bw); }
    std::vector<double> effective_all() const {
        std::vector<double> out;
        for (std::size_t i = 0; i < tiers.size(); ++i) out.push_back(effective(i));
        return out;
    }
};

inline void update_bandwidth_estimates(BandwidthEstimate& est, std::span<const TierObservation> observed) {
    const std::size_t n = est.tiers.size();
    std::vector<double> r(n), w(n);
    std::vector<std::uint64_t> c(n);
    for (std::size_t i = 0; i < n; ++i) {
        r[i] = est.tiers[i].read_bw;
        w[i] = est.tiers[i].write_bw;
        c[i] = est.tiers[i].sample_count;
    }
    std::vector<tfg_tier_observation> obs;
    for (const TierObservation& o : observed)
        obs.push_back(tfg_tier_observation{o.read_transfers, o.read_bytes, o.read_seconds, o.write_transfers,
                                           o.write_bytes, o.write_seconds});
    detail::check(tfg_update_bandwidth_estimates(r.data(), w.data(), c.data(), static_cast<int>(n), est.alpha,
                                                 obs.data(), static_cast<int>(obs.size())));
    for (std::size_t i = 0; i < n; ++i) est.tiers[i] = BandwidthEstimate::PerTier{r[i], w[i], c[i]};
}

struct CachePlan {
    int capacity = 0;
};

struct TierAssignment {
    bool host_retain = false;
    TierId tier = kNoTier;
};

// Flush destinations of one phase (placement.hpp:173-225), computed by the
// library (the engine's own plan).
class DestinationPlan {
public:
    DestinationPlan(std::span<const SubgroupId> order, CachePlan cache, std::span<const double> bandwidths) {
        const int M = static_cast<int>(order.size());
        const int T = static_cast<int>(bandwidths.size());
        std::vector<int> retain(order.size()), tier(order.size());
        alloc_.counts.assign(bandwidths.size(), 0);
        detail::check(tfg_destination_plan(order.data(), M, cache.capacity, bandwidths.data(), T, retain.data(),
                                           tier.data(), alloc_.counts.data()));
        retained_ = std::clamp(cache.capacity, 0, M);
        alloc_.total = M - retained_;
        for (std::size_t k = 0; k < order.size(); ++k) map_[order[k]] = TierAssignment{retain[k] != 0, tier[k]};
    }
    TierAssignment assign_storage_tier(SubgroupId sg) const {
        const auto it = map_.find(sg);
        if (it == map_.end()) throw Error("destination plan: unknown subgroup " + std::to_string(sg));
        return it->second;
    }
    const AllocationVector& flush_allocation() const { return alloc_; }
    int retained_count() const { return retained_; }

private:
    std::map<SubgroupId, TierAssignment> map_;
    AllocationVector alloc_;
    int retained_ = 0;
};

// --- trace.hpp ----------------------------------------------------------------------

enum class EventKind : int {
    prefetch_start,
    prefetch_end,
    update_start,
    update_end,
    flush_start,
    flush_end,
    lock_acquire,
    lock_release,
    h2d_start,
    h2d_end,
    grad_upscale_start,
    grad_upscale_end,
    cache_hit,
};

// Kind names of the trace schema (trace.hpp:31-62); the library writes the
// same names (tfg_trace_write).
inline const char* event_kind_name(EventKind k) {
    static constexpr const char* names[] = {"prefetch_start", "prefetch_end", "update_start", "update_end",
                                            "flush_start",    "flush_end",    "lock_acquire", "lock_release",
                                            "h2d_start",      "h2d_end",      "grad_upscale_start",
                                            "grad_upscale_end", "cache_hit"};
    const int i = static_cast<int>(k);
    return i >= 0 && i <= static_cast<int>(EventKind::cache_hit) ? names[i] : "unknown";
}

inline bool event_kind_from_name(std::string_view name, EventKind& out) {
    for (int i = 0; i <= static_cast<int>(EventKind::cache_hit); ++i)
        if (name == event_kind_name(static_cast<EventKind>(i))) {
            out = static_cast<EventKind>(i);
            return true;
        }
    return false;
}

struct Event {
    std::int64_t timestamp_ns = 0;
    WorkerId worker_id = 0;
    EventKind kind = EventKind::prefetch_start;
    std::int64_t subgroup_id = -1;
    TierId tier_id = kNoTier;
    std::uint64_t bytes = 0;
};

class EventTrace {
public:
    EventTrace() { detail::check(tfg_trace_create(&h_)); }
    ~EventTrace() { tfg_trace_destroy(h_); }
    EventTrace(const EventTrace&) = delete;
    EventTrace& operator=(const EventTrace&) = delete;

    void record(EventKind kind, WorkerId worker, std::int64_t subgroup, TierId tier, std::uint64_t bytes) {
        detail::check(tfg_trace_record(h_, static_cast<int>(kind), worker, subgroup, tier, bytes));
    }
    std::size_t size() const {
        std::uint64_t n = 0;
        detail::check(tfg_trace_size(h_, &n));
        return n;
    }
    std::vector<Event> snapshot_from(std::size_t begin) const {
        const std::size_t n = size();
        std::vector<tfg_event> raw(n > begin ? n - begin : 0);
        std::uint64_t got = 0;
        if (!raw.empty()) detail::check(tfg_trace_copy(h_, begin, raw.data(), raw.size(), &got));
        std::vector<Event> out;
        out.reserve(got);
        for (std::size_t i = 0; i < got; ++i) {
            const tfg_event& e = raw[i];
            out.push_back(Event{e.timestamp_ns, e.worker_id, static_cast<EventKind>(e.kind), e.subgroup_id, e.tier_id,
                                e.bytes});
        }
        return out;
    }
    std::vector<Event> snapshot() const { return snapshot_from(0); }
    void append(Event e) {
        detail::check(tfg_trace_record_at(h_, e.timestamp_ns, static_cast<int>(e.kind), e.worker_id, e.subgroup_id,
                                          e.tier_id, e.bytes));
    }
    std::uint64_t progress_count() const { return size(); }
    void clear() { detail::check(tfg_trace_clear(h_)); }
    void write_csv(const std::filesystem::path& p) const { detail::check(tfg_trace_write(h_, p.c_str())); }
    tfg_trace* handle() const { return h_; }

    // The trace file schema (trace.hpp:116-161): CSV with this header, or
    // one JSON object per line.
    static constexpr const char* kCsvHeader = "timestamp_ns,worker_id,kind,subgroup_id,tier_id,bytes";

    static void write_csv(std::ostream& os, const std::vector<Event>& events) {
        os << kCsvHeader << '\n';
        for (const Event& e : events)
            os << e.timestamp_ns << ',' << e.worker_id << ',' << event_kind_name(e.kind) << ',' << e.subgroup_id
               << ',' << e.tier_id << ',' << e.bytes << '\n';
    }
    static void write_jsonl(std::ostream& os, const std::vector<Event>& events) {
        for (const Event& e : events)
            os << "{\"timestamp_ns\":" << e.timestamp_ns << ",\"worker_id\":" << e.worker_id << ",\"kind\":\""
               << event_kind_name(e.kind) << "\",\"subgroup_id\":" << e.subgroup_id << ",\"tier_id\":" << e.tier_id
               << ",\"bytes\":" << e.bytes << "}\n";
    }
    static std::vector<Event> read_csv(std::istream& is) {
        std::vector<Event> out;
        std::string line;
        for (bool first = true; std::getline(is, line);) {
            if (line.empty()) continue;
            const bool header = first && line.rfind("timestamp_ns", 0) == 0;
            first = false;
            if (header) continue;
            std::vector<std::string> f;
            std::stringstream ss(line);
            for (std::string x; std::getline(ss, x, ',');) f.push_back(x);
            if (f.size() != 6) throw FormatError("trace line has " + std::to_string(f.size()) + " fields: " + line);
            Event e;
            e.timestamp_ns = std::stoll(f[0]);
            e.worker_id = std::stoi(f[1]);
            if (!event_kind_from_name(f[2], e.kind)) throw FormatError("unknown trace event kind: " + f[2]);
            e.subgroup_id = std::stoll(f[3]);
            e.tier_id = std::stoi(f[4]);
            e.bytes = std::stoull(f[5]);
            out.push_back(e);
        }
        return out;
    }

private:
    tfg_trace* h_ = nullptr;
};

// --- tier.hpp -----------------------------------------------------------------------

// host_dram is the B200 engine's pinned-host tier (no reference counterpart).
enum class TierKind { local_dir = TFG_LOCAL_DIR, remote_dir = TFG_REMOTE_DIR, mem_throttled = TFG_MEM_THROTTLED,
                      host_dram = TFG_HOST_DRAM };

// v1 subgroup file header (tier.hpp:92-134), encoded and checked by the
// library's tier code.
struct SubgroupFileHeader {
    static constexpr std::uint32_t kMagic = 0x4D4C504F;
    static constexpr std::uint16_t kVersion = 1;
    static constexpr std::uint16_t kElementF32 = 0;
    static constexpr std::size_t kSize = 32;

    std::uint32_t magic = kMagic;
    std::uint16_t version = kVersion;
    std::uint16_t element_kind = kElementF32;
    std::uint32_t subgroup_id = 0;
    std::uint64_t param_count = 0;

    std::array<std::uint8_t, kSize> encode() const {
        std::array<std::uint8_t, kSize> buf{};
        const tfg_file_header h = c();
        detail::check(tfg_file_header_encode(&h, buf.data()));
        return buf;
    }
    static SubgroupFileHeader decode(const std::uint8_t* buf) {
        tfg_file_header h{};
        detail::check(tfg_file_header_decode(buf, &h));
        SubgroupFileHeader out;
        out.magic = h.magic;
        out.version = h.version;
        out.element_kind = h.element_kind;
        out.subgroup_id = h.subgroup_id;
        out.param_count = h.param_count;
        return out;
    }
    void validate(std::uint32_t expected_id, std::uint64_t expected_params) const {
        const tfg_file_header h = c();
        detail::check(tfg_file_header_validate(&h, expected_id, expected_params));
    }

private:
    tfg_file_header c() const { return tfg_file_header{magic, version, element_kind, subgroup_id, param_count}; }
};

inline std::string subgroup_file_name(SubgroupId id) {
    char buf[64];
    detail::check(tfg_subgroup_file_name(id, buf, sizeof(buf)));
    return buf;
}

struct TierSpec {
    TierId tier_id = 0;
    TierKind kind = TierKind::local_dir;
    std::filesystem::path root;
    double read_bw = 0.0;
    double write_bw = 0.0;
    int io_parallelism = 1;
    bool persistent = false;
};

struct ProbeResult {
    double read_bw = 0.0;
    double write_bw = 0.0;
    bool low_confidence = false;
};

class Tier {
public:
    explicit Tier(TierSpec spec) : spec_(std::move(spec)) {
        const std::string root = spec_.root.string();
        tfg_tier_spec s{spec_.tier_id, static_cast<int32_t>(spec_.kind), root.c_str(), spec_.read_bw, spec_.write_bw,
                        spec_.io_parallelism, spec_.persistent ? 1 : 0, 1, 1, 0, 0};
        detail::check(tfg_tier_create(&s, &h_));
    }
    ~Tier() { tfg_tier_destroy(h_); }
    Tier(const Tier&) = delete;
    Tier& operator=(const Tier&) = delete;

    const TierSpec& spec() const {
        detail::check(tfg_tier_bandwidths(h_, &spec_.read_bw, &spec_.write_bw));  // probes update them
        return spec_;
    }
    TierId id() const { return spec_.tier_id; }
    tfg_tier* handle() const { return h_; }

    void set_throttle_rates(double read_bps, double write_bps) {
        detail::check(tfg_tier_set_throttle_rates(h_, read_bps, write_bps));
    }
    IoStats write_subgroup(SubgroupId id, std::uint64_t param_count, std::span<const float> state) {
        if (state.size() != 3 * param_count) throw Error("write_subgroup: state length mismatch");
        IoStats st;
        detail::check(tfg_tier_write_subgroup(h_, id, param_count, state.data(), &st.bytes, &st.seconds));
        return st;
    }
    IoStats read_subgroup(SubgroupId id, std::uint64_t param_count, std::span<float> state) {
        if (state.size() != 3 * param_count) throw Error("read_subgroup: state length mismatch");
        IoStats st;
        detail::check(tfg_tier_read_subgroup(h_, id, param_count, state.data(), &st.bytes, &st.seconds));
        return st;
    }
    IoStats write_grads(SubgroupId id, std::uint64_t param_count, std::span<const float> grads) {
        if (grads.size() != param_count) throw Error("write_grads: length mismatch");
        detail::check(tfg_tier_write_grads(h_, id, param_count, grads.data()));
        return IoStats{4 * param_count, 0.0};
    }
    IoStats read_grads(SubgroupId id, std::uint64_t param_count, std::span<float> grads) {
        if (grads.size() != param_count) throw Error("read_grads: length mismatch");
        detail::check(tfg_tier_read_grads(h_, id, param_count, grads.data()));
        return IoStats{4 * param_count, 0.0};
    }
    bool has_subgroup(SubgroupId id) const {
        int out = 0;
        detail::check(tfg_tier_has_subgroup(h_, id, &out));
        return out != 0;
    }
    void remove_subgroup(SubgroupId id) { detail::check(tfg_tier_remove_subgroup(h_, id)); }
    ProbeResult probe_bandwidth(std::uint64_t probe_bytes, int repetitions) {
        ProbeResult r;
        int low = 0;
        detail::check(tfg_tier_probe(h_, probe_bytes, repetitions, &r.read_bw, &r.write_bw, &low));
        r.low_confidence = low != 0;
        return r;
    }
    std::uint64_t available_bytes() const {
        std::uint64_t out = 0;
        detail::check(tfg_tier_available_bytes(h_, &out));
        return out;
    }

private:
    mutable TierSpec spec_;
    tfg_tier* h_ = nullptr;
};

// --- tier_lock.hpp ------------------------------------------------------------------

class TierLockGuard {
public:
    TierLockGuard(const std::filesystem::path& lock_dir, TierId tier, WorkerId worker, EventTrace* trace) {
        detail::check(tfg_tier_lock_acquire(lock_dir.c_str(), tier, worker, trace ? trace->handle() : nullptr, 1,
                                            &token_));
    }
    TierLockGuard(TierLockGuard&& o) noexcept : token_(std::exchange(o.token_, nullptr)) {}
    TierLockGuard& operator=(TierLockGuard&& o) noexcept {
        if (this != &o) {
            release();
            token_ = std::exchange(o.token_, nullptr);
        }
        return *this;
    }
    TierLockGuard(const TierLockGuard&) = delete;
    TierLockGuard& operator=(const TierLockGuard&) = delete;
    ~TierLockGuard() { release(); }

    void release() {
        if (token_ != nullptr) tfg_tier_lock_release(std::exchange(token_, nullptr));
    }
    bool held() const { return token_ != nullptr; }

private:
    void* token_ = nullptr;
};

inline TierLockGuard acquire_tier_lock(const std::filesystem::path& lock_dir, TierId tier, WorkerId worker,
                                       EventTrace* trace = nullptr) {
    return TierLockGuard(lock_dir, tier, worker, trace);
}

// --- pool.hpp -----------------------------------------------------------------------

// Same enumerators as the reference (pool.hpp:17); the values are the
// engine's slot-state codes.
enum class SlotState { free_slot = 0, prefetching = 1, updating = 2, flushing = 3, cached = 4 };

class HostBufferPool {
public:
    HostBufferPool(int slot_count, std::uint64_t max_param_count) : max_params_(max_param_count) {
        detail::check(tfg_pool_create(slot_count, max_param_count, &h_));
    }
    ~HostBufferPool() { tfg_pool_destroy(h_); }
    HostBufferPool(const HostBufferPool&) = delete;
    HostBufferPool& operator=(const HostBufferPool&) = delete;

    int slot_count() const {
        int n = 0;
        detail::check(tfg_pool_slot_count(h_, &n));
        return n;
    }
    std::uint64_t max_param_count() const { return max_params_; }
    int try_reserve(SubgroupId owner) {
        int s = -1;
        detail::check(tfg_pool_try_reserve(h_, owner, &s));
        return s;
    }
    int find_cached(SubgroupId owner) const {
        int s = -1;
        detail::check(tfg_pool_find_cached(h_, owner, &s));
        return s;
    }
    void prefetch_done(int slot) { detail::check(tfg_pool_transition(h_, slot, TFG_POOL_PREFETCH_DONE)); }
    void begin_update(int slot) { detail::check(tfg_pool_transition(h_, slot, TFG_POOL_BEGIN_UPDATE)); }
    void end_update(int slot) { detail::check(tfg_pool_transition(h_, slot, TFG_POOL_END_UPDATE)); }
    void begin_flush(int slot) { detail::check(tfg_pool_transition(h_, slot, TFG_POOL_BEGIN_FLUSH)); }
    void flush_done(int slot) { detail::check(tfg_pool_transition(h_, slot, TFG_POOL_FLUSH_DONE)); }
    void evict(int slot) { detail::check(tfg_pool_transition(h_, slot, TFG_POOL_EVICT)); }
    SlotState state(int slot) const {
        int st = 0;
        detail::check(tfg_pool_query(h_, slot, &st, nullptr));
        return static_cast<SlotState>(st);
    }
    SubgroupId owner(int slot) const {
        std::uint32_t o = 0;
        detail::check(tfg_pool_query(h_, slot, nullptr, &o));
        return o;
    }
    std::span<float> state_span(int slot, std::uint64_t param_count) { return span(slot, param_count, 0); }
    std::span<float> grad_span(int slot, std::uint64_t param_count) { return span(slot, param_count, 1); }

private:
    std::span<float> span(int slot, std::uint64_t params, int which) {
        float* p = nullptr;
        std::uint64_t len = 0;
        detail::check(tfg_pool_span(h_, slot, params, which, &p, &len));
        return std::span<float>(p, len);
    }
    tfg_pool* h_ = nullptr;
    std::uint64_t max_params_ = 0;
};

// --- scheduler.hpp ------------------------------------------------------------------

struct ScheduleOptions {
    int pool_slots = 4;
    int cache_slots = -1;
    bool enable_caching = true;
    bool skip_gradients = true;
    bool atomic_rw = true;
    bool multi_path = true;
    std::filesystem::path lock_dir;
    int update_threads = 1;
    double deadlock_timeout_s = 30.0;
    std::uint64_t update_pad_ns = 0;

    int retention_capacity(int subgroup_count) const {
        int out = 0;
        detail::check(tfg_retention_capacity(enable_caching, pool_slots, cache_slots, subgroup_count, &out));
        return out;
    }
};

struct UpdatePlan {
    int iteration = 0;
    bool ascending = true;
    std::vector<SubgroupId> order;

    static UpdatePlan make(int iteration, std::vector<SubgroupId> sorted_ids, bool alternate) {
        UpdatePlan p;
        p.iteration = iteration;
        p.order.resize(sorted_ids.size());
        detail::check(tfg_update_order(iteration, sorted_ids.data(), static_cast<int>(sorted_ids.size()),
                                       alternate ? 1 : 0, p.order.data()));
        p.ascending = p.order.size() < 2 ? (!alternate || iteration % 2 == 0) : p.order.front() <= p.order.back();
        return p;
    }

    std::optional<SubgroupId> next_after(SubgroupId id) const {
        for (std::size_t k = 0; k + 1 < order.size(); ++k)
            if (order[k] == id) return order[k + 1];
        return std::nullopt;
    }
};

// The engine generates these gradients on the GPU (the reference's
// splitmix64 chain, bit for bit); the source carries only the seed.
struct SyntheticGradSource {
    std::uint64_t seed = 42;
};

struct SubgroupIoTimes {
    SubgroupId id = 0;
    std::uint64_t state_bytes = 0;
    double read_seconds = 0.0;
    double write_seconds = 0.0;
    bool fetched = false;
    bool flushed = false;
};

struct PhaseStats {
    double wall_seconds = 0.0;
    std::uint64_t params_updated = 0;
    std::uint64_t cache_hits = 0;
    std::uint64_t downscale_overflows = 0;
    int retained = 0;
    std::vector<int> flush_allocation;
    std::vector<TierObservation> tier_obs;
    std::vector<SubgroupIoTimes> subgroup_io;
};

class OffloadWorker {
public:
    OffloadWorker(WorkerId id, std::vector<std::shared_ptr<Tier>> tiers, ScheduleOptions opt, AdamHyper hyper,
                  EventTrace& trace)
        : id_(id), tiers_(std::move(tiers)), opt_(std::move(opt)) {
        std::vector<tfg_tier*> th;
        for (const auto& t : tiers_) th.push_back(t->handle());
        const std::string lock = opt_.lock_dir.string();
        tfg_schedule_options so{opt_.pool_slots, opt_.cache_slots, opt_.enable_caching, opt_.skip_gradients,
                                opt_.atomic_rw, opt_.multi_path, lock.c_str(), opt_.update_threads,
                                opt_.deadlock_timeout_s, opt_.update_pad_ns};
        const tfg_adam_hyper ah = hyper.c();
        tfg_device_options dv{0, TFG_F16, TFG_F16, 3, 0, 1, 1, 1, 0, 0};
        detail::check(tfg_engine_create(id, th.data(), static_cast<int>(th.size()), &so, &ah, trace.handle(), &dv, &h_));
    }
    ~OffloadWorker() { tfg_engine_destroy(h_); }
    OffloadWorker(const OffloadWorker&) = delete;
    OffloadWorker& operator=(const OffloadWorker&) = delete;

    WorkerId id() const { return id_; }
    void set_alpha(double alpha) { detail::check(tfg_engine_set_alpha(h_, alpha)); }
    void set_fixed_ratio(std::vector<double> ratio) {
        detail::check(tfg_engine_set_fixed_ratio(h_, ratio.data(), static_cast<int>(ratio.size())));
    }
    void add_subgroup(SubgroupId id, std::uint64_t param_count) {
        detail::check(tfg_engine_add_subgroup(h_, id, param_count));
        params_[id] = param_count;
        ids_.push_back(id);
    }
    const std::vector<SubgroupId>& subgroup_ids() const { return ids_; }
    void init_and_flush_all(std::uint64_t seed) { detail::check(tfg_engine_init_and_flush_all(h_, seed)); }
    void run_backward_sim(int iteration, const SyntheticGradSource& src, int accum_steps) {
        lent_.clear();  // the backward rewrites the device gradients: earlier host views are stale
        detail::check(tfg_engine_run_backward_sim(h_, iteration, src.seed, accum_steps));
    }
    bool gradients_finite() {
        write_back_lent();
        int out = 0;
        detail::check(tfg_engine_gradients_finite(h_, &out));
        return out != 0;
    }
    // Host view of the subgroup's HBM gradient buffer, read here. Edits made
    // through mutable_values() reach the engine before the next
    // gradients_finite() or run_update() (the reference hands out the live
    // host buffer).
    GradBufferF16& grad_buffer(SubgroupId id) {
        GradBufferF16& b = grads_[id];
        b.id_ = id;
        b.values_.resize(params_.at(id));
        detail::check(tfg_engine_read_grads16(h_, id, reinterpret_cast<std::uint16_t*>(b.values_.data())));
        if (std::find(lent_.begin(), lent_.end(), id) == lent_.end()) lent_.push_back(id);
        return b;
    }

    PhaseStats run_update(int iteration) {
        write_back_lent();
        tfg_phase_stats st{};
        detail::check(tfg_engine_run_update(h_, iteration, &st));
        PhaseStats out;
        out.wall_seconds = st.wall_seconds;
        out.params_updated = st.params_updated;
        out.cache_hits = st.cache_hits;
        out.downscale_overflows = st.downscale_overflows;
        out.retained = st.retained;
        for (int t = 0; t < st.n_tiers; ++t) {
            out.flush_allocation.push_back(st.flush_allocation[t]);
            const tfg_tier_observation& o = st.tier_obs[t];
            out.tier_obs.push_back(TierObservation{o.read_transfers, o.read_bytes, o.read_seconds, o.write_transfers,
                                                   o.write_bytes, o.write_seconds});
        }
        std::vector<tfg_subgroup_io> io(st.n_subgroup_io);
        std::uint64_t got = 0;
        if (!io.empty()) detail::check(tfg_engine_last_subgroup_io(h_, io.data(), io.size(), &got));
        for (std::size_t i = 0; i < got; ++i)
            out.subgroup_io.push_back(SubgroupIoTimes{io[i].id, io[i].state_bytes, io[i].read_seconds,
                                                      io[i].write_seconds, io[i].fetched != 0, io[i].flushed != 0});
        return out;
    }

    int wait_host_resident(SubgroupId id) {
        int slot = -1;
        detail::check(tfg_engine_wait_host_resident(h_, id, &slot));
        return slot;
    }
    std::shared_future<IoStats> enqueue_flush(SubgroupId id, TierId dest) {
        std::uint64_t ticket = 0;
        detail::check(tfg_engine_enqueue_flush(h_, id, dest, &ticket));
        return ticket_future(ticket);
    }
    std::optional<std::shared_future<IoStats>> enqueue_prefetch(SubgroupId id) {
        std::uint64_t ticket = 0;
        detail::check(tfg_engine_enqueue_prefetch(h_, id, &ticket));
        if (ticket == 0) return std::nullopt;  // host-resident: a cache hit, nothing queued
        return ticket_future(ticket);
    }
    std::vector<float> read_current_state(SubgroupId id) {
        std::vector<float> out(3 * params_.at(id));
        detail::check(tfg_engine_read_state(h_, id, out.data()));
        return out;
    }
    Subgroup meta(SubgroupId id) const {
        tfg_subgroup_meta m{};
        detail::check(tfg_engine_meta(h_, id, &m));
        Subgroup s;
        s.id = m.id;
        s.param_count = m.param_count;
        s.residency = static_cast<Residency>(m.residency);
        s.tier = m.tier;
        s.slot = m.slot;
        s.step_count = m.step_count;
        return s;
    }
    std::uint64_t total_params() const {
        std::uint64_t n = 0;
        for (const auto& [id, p] : params_) n += p;
        return n;
    }
    std::pair<std::uint64_t, std::vector<std::uint64_t>> residency_census() const {
        std::pair<std::uint64_t, std::vector<std::uint64_t>> c{0, std::vector<std::uint64_t>(tiers_.size(), 0)};
        detail::check(tfg_engine_residency_census(h_, &c.first, c.second.data(), static_cast<int>(tiers_.size())));
        return c;
    }
    const ScheduleOptions& options() const { return opt_; }

private:
    void write_back_lent() {
        for (const SubgroupId id : lent_)
            detail::check(tfg_engine_write_grads16(h_, id, reinterpret_cast<const std::uint16_t*>(grads_[id].values_.data())));
        lent_.clear();
    }
    std::shared_future<IoStats> ticket_future(std::uint64_t ticket) {
        tfg_engine* h = h_;
        return std::async(std::launch::deferred, [h, ticket] {
                   IoStats st;
                   detail::check(tfg_engine_wait_ticket(h, ticket, &st.bytes, &st.seconds));
                   return st;
               }).share();
    }

    WorkerId id_;
    std::vector<std::shared_ptr<Tier>> tiers_;
    ScheduleOptions opt_;
    tfg_engine* h_ = nullptr;
    std::map<SubgroupId, std::uint64_t> params_;
    std::vector<SubgroupId> ids_;
    std::map<SubgroupId, GradBufferF16> grads_;
    std::vector<SubgroupId> lent_;  // grad_buffer views handed out since the last backward
};

}  // namespace tierflow
