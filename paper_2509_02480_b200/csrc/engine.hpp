// The B200 update-phase engine: one OffloadWorker per GPU rank.
//
// Drop-in for the reference engine's per-iteration API (reference
// proj/include/tierflow/scheduler.hpp:286-864): tier configuration,
// add_subgroup partitioning, init_and_flush_all, run_update, the op-level
// enqueue_prefetch / wait_host_resident / enqueue_flush / read_current_state.
// Placement, ordering, retention, prefetch frontier and per-tier queue
// discipline follow the reference rule for rule, so placement, fetch order
// and cache-hit sequences are bit-identical (SURVEY.md §8a rules 1-5).
//
// What is different is where the update runs. A host-resident subgroup's
// pinned slot is streamed through a ring of device buffers on three CUDA
// streams: H2D (slot -> HBM) -> fused sm_100a Adam kernel (gradient from the
// device-resident 16-bit gradient buffer, 16-bit working params written to
// the device-resident parameter buffer) -> D2H (HBM -> slot). The coordinator
// issues subgroups as they become host-resident, keeping a few state copies
// queued on the H2D stream (kH2dAhead); a completion thread retires finished subgroups (slot back to cached, lazy
// flush or retention, frontier pump) exactly where the reference's
// coordinator would after adam_step returns.
//
// Retention can live in HBM (DeviceOptions::hbm_retain): retained subgroups
// keep their updated state in HBM buffers between phases. In the HBM cache
// mode (2) their host slots stream again; a retained subgroup the next plan
// flushes is written back through a small lane of pinned blocks by its own
// thread and stream, so the misses' H2D starts at phase begin; with
// hbm_cache_slots < C the cache is two-level (the rest kept in host slots).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <condition_variable>
#include <deque>
#include <filesystem>
#include <functional>
#include <future>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.hpp"
#include "host_block.hpp"
#include "placement.hpp"
#include "tier.hpp"
#include "trace.hpp"
#include "types.hpp"

namespace tfb {

struct ScheduleOptions {
    int pool_slots = 4;
    int cache_slots = -1;         // host retention capacity C; -1 derives pool_slots - 3
    bool enable_caching = true;   // alternating order + host retention
    bool skip_gradients = true;   // delayed 16-bit -> fp32 gradient conversion (fused in the kernel)
    bool atomic_rw = true;        // tier semaphores around transfers
    bool multi_path = true;       // place across all tiers vs tier 0 only
    std::string lock_dir;
    int update_threads = 1;       // accepted for API parity; the update runs on the GPU
    double deadlock_timeout_s = 30.0;
    std::uint64_t update_pad_ns = 0;  // synthetic extra device time per subgroup update

    int retention_capacity(int subgroup_count) const {
        return tfb::retention_capacity(enable_caching, pool_slots, cache_slots, subgroup_count);
    }
};

struct AdamHyper {
    double lr = 1e-3;
    double beta1 = 0.9;
    double beta2 = 0.999;
    double eps = 1e-8;
    double weight_decay = 0.0;

    void validate() const;  // reference optimizer.hpp:24-30
    AdamConsts consts(std::uint64_t t) const;
};

struct DeviceOptions {
    int device = 0;
    int grad_kind = kF16;    // 16-bit gradient element kind
    int out_kind = kF16;     // 16-bit working-parameter element kind
    int device_buffers = 3;  // depth of the H2D -> kernel -> D2H ring
    int zero_copy = 0;       // 1: the kernel reads/writes the pinned slot over PCIe (no ring, no DMA)
    int d2h_split = 1;       // concurrent D2H copy streams per subgroup (1 or 2)
    int h2d_split = 1;       // concurrent H2D copy streams per subgroup (1 or 2)
    // hbm_retain 2: HBM buffers for retained subgroups (0: all of C). Fewer
    // than C gives a two-level cache, the rest retained in host slots.
    int hbm_cache_slots = 0;
    // Copy mode, 16-bit gradient flow: a subgroup the destination plan retains
    // keeps its updated state in HBM until its next update (no D2H now, no H2D
    // then). 1: the host slot stays reserved and is refreshed on demand, C is
    // the reference's min(cache_slots, pool_slots - 3). 2 (HBM cache): the
    // retained subgroup gives its host slot back and the retention capacity
    // C = cache_slots is bounded by HBM, not by the pool (cache_slots < 0:
    // pool_slots - 3); all pool slots stream. A retained subgroup the next
    // plan flushes takes a slot for its write-back in plan order.
    int hbm_retain = 1;
    // Host-resident 16-bit gradients and working params: pinned host blocks
    // per subgroup streamed with the state (2 B/param more each way through a
    // small device staging ring) instead of 4 B/param of HBM arenas for the
    // whole shard, so a rank's shard is bounded by host memory, not HBM.
    bool host_grads = false;
};

// HBM cache mode: pinned blocks in the write-back lane.
constexpr int kWritebackBlocks = 4;
// State H2D copies the coordinator keeps queued on the H2D stream. Enough to
// keep the stream busy across host issue latency; the resident subgroups
// beyond it wait on the host, where a later-resident one the plan flushes to
// a directory tier can still go first (pick_next_ready).
constexpr int kH2dAhead = 3;
// Baseline flow: pinned fp32-gradient staging blocks in rotation.
constexpr int kGradStages = 4;

enum class Residency : int { host_cached = 0, in_flight = 1, on_tier = 2 };

struct Subgroup {
    SubgroupId id = 0;
    std::uint64_t param_count = 0;
    Residency residency = Residency::host_cached;
    TierId tier = kNoTier;
    int slot = -1;
    std::uint64_t step_count = 0;

    // host_cached -> in_flight -> on_tier -> in_flight -> host_cached
    // (reference optimizer.hpp:47-72).
    void begin_flush();
    void finish_flush(TierId dest);
    void begin_prefetch();
    void finish_prefetch(int pool_slot);
};

struct SubgroupIoTimes {
    SubgroupId id = 0;
    std::uint64_t state_bytes = 0;
    double read_seconds = 0.0;
    double write_seconds = 0.0;
    bool fetched = false;
    bool flushed = false;
};

// Per-subgroup timeline of one phase, milliseconds from the phase start.
// Device times come from CUDA events on the pipeline streams (zero = the
// phase start on the H2D stream); host times from CLOCK_MONOTONIC (zero = run_update entry).
struct DeviceSpan {
    SubgroupId id = 0;
    float h2d_start = 0, h2d_end = 0, k_start = 0, k_end = 0, d2h_end = 0;
    float host_resident = 0;  // wait_host_resident returned
    float host_retired = 0;   // completion thread retired the subgroup
    float d2h_start = 0;      // its D2H began (= d2h_end when nothing went back)
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
    // Device side (CUDA events on the pipeline streams).
    double device_seconds = 0.0;  // phase start -> last D2H end
    double kernel_seconds = 0.0;  // sum of fused-kernel durations
    double h2d_seconds = 0.0;     // sum of state H2D durations
    double d2h_seconds = 0.0;     // sum of state D2H durations
    std::uint64_t h2d_bytes = 0;
    std::uint64_t d2h_bytes = 0;
    std::vector<DeviceSpan> timeline;  // plan order
};

// ---------------------------------------------------------------------------
// Pinned staging slots with the reference slot state machine
// (free -> prefetching -> cached -> updating -> cached -> flushing -> free;
// reference pool.hpp:17-161). Each slot owns one HostBlock.
enum class SlotState : int { free_slot = 0, prefetching, updating, flushing, cached };

const char* slot_state_name(SlotState s);

class HostBufferPool {
public:
    HostBufferPool(int slot_count, std::size_t block_bytes, bool require_pinned);

    int slot_count() const { return static_cast<int>(slots_.size()); }
    int try_reserve(SubgroupId owner);
    int find_cached(SubgroupId owner) const;
    void prefetch_done(int slot) { transition(slot, SlotState::prefetching, SlotState::cached); }
    void begin_update(int slot) { transition(slot, SlotState::cached, SlotState::updating); }
    void end_update(int slot) { transition(slot, SlotState::updating, SlotState::cached); }
    void begin_flush(int slot) { transition(slot, SlotState::cached, SlotState::flushing); }
    void flush_done(int slot);
    void flush_failed(int slot) { transition(slot, SlotState::flushing, SlotState::cached); }
    void evict(int slot);
    void release_failed(int slot);
    SlotState state(int slot) const;
    SubgroupId owner(int slot) const;
    int count(SlotState s) const;
    bool wait_for_free(std::chrono::milliseconds timeout);
    // The block is owned by whoever holds the slot in a non-free state.
    HostBlock& block(int slot) { return slots_[check(slot)].block; }

private:
    struct Slot {
        SlotState state = SlotState::free_slot;
        SubgroupId owner = 0;
        HostBlock block;
    };
    std::size_t check(int slot) const;
    void transition(int slot, SlotState expected, SlotState next);

    mutable std::mutex mu_;
    std::condition_variable free_cv_;
    std::vector<Slot> slots_;
};

// ---------------------------------------------------------------------------
// One I/O thread per (worker, tier) serving two lanes: a queued fetch always
// outranks a queued write-back (reference scheduler.hpp:142-266, the
// prefetch-before-flush rule at :222). Each transfer runs under the tier
// semaphore when atomic_rw is on, and is traced as one start/end interval.
class TierIoWorker {
public:
    using Completion = std::function<void(bool ok, const IoStats&)>;
    enum Lane : int { kFetch = 0, kWriteBack = 1 };

    TierIoWorker(std::shared_ptr<Tier> tier, WorkerId worker, bool use_lock, std::filesystem::path lock_dir,
                 EventTrace* trace);
    ~TierIoWorker();

    std::future<IoStats> submit(bool is_prefetch, std::int64_t sg, std::uint64_t bytes_hint,
                                std::function<IoStats()> transfer, Completion completion);
    void shutdown();

private:
    struct Job {
        Lane lane = kFetch;
        std::int64_t sg = -1;
        std::uint64_t bytes_hint = 0;
        std::function<IoStats()> transfer;
        Completion completion;
        std::promise<IoStats> promise;
    };
    bool next_job(Job& out);  // blocks; false once closed and drained
    void serve();
    IoStats transfer_traced(Job& job);
    static void cancel(Job& job);

    std::shared_ptr<Tier> tier_;
    WorkerId worker_;
    bool use_lock_;
    std::filesystem::path lock_dir_;
    EventTrace* trace_;
    std::mutex mu_;
    std::condition_variable wake_;
    std::array<std::deque<Job>, 2> lanes_;
    bool closed_ = false;
    std::thread thread_;
};

// ---------------------------------------------------------------------------

class OffloadWorker {
public:
    OffloadWorker(WorkerId id, std::vector<std::shared_ptr<Tier>> tiers, ScheduleOptions opt, AdamHyper hyper,
                  std::shared_ptr<EventTrace> trace, DeviceOptions dev);
    ~OffloadWorker();
    OffloadWorker(const OffloadWorker&) = delete;
    OffloadWorker& operator=(const OffloadWorker&) = delete;

    WorkerId id() const { return id_; }
    void set_alpha(double alpha);
    void set_fixed_ratio(std::vector<double> ratio);
    // Retention capacity for the following phases (ScheduleOptions::cache_slots;
    // between phases). In the HBM cache mode it may not exceed the HBM
    // buffers allocated at init.
    void set_cache_slots(int cache_slots);
    void add_subgroup(SubgroupId id, std::uint64_t param_count);

    // Seeded fp32 states (synthetic_param_init, zero moments) generated on the
    // GPU and flushed to the tiers Eq. 1 picks; every subgroup ends on_tier.
    void init_and_flush_all(std::uint64_t seed);

    // Backward stand-in: seeded 16-bit gradients generated on the GPU into the
    // device gradient buffers (SyntheticGradSource + GradBufferF16 semantics).
    void run_backward_sim(int iteration, std::uint64_t seed, int accum_steps);
    bool gradients_finite();
    // Device gradient buffer of a subgroup (param_count 16-bit elements); the
    // caller may fill it (e.g. from a reduce-scatter) or rebind it.
    void* grad_buffer(SubgroupId id);
    void bind_grad_buffer(SubgroupId id, void* device_ptr);
    // Several gradient sources (e.g. every data-parallel peer's contribution,
    // mapped over NVLink): each phase's gradient check sums them in fp32 in
    // order, rounds once to the gradient kind into the subgroup's own buffer
    // (one read of every source), and the update reads that buffer.
    void bind_grad_sources(SubgroupId id, const std::vector<const void*>& sources);
    void* params16_buffer(SubgroupId id);
    // The stream that produces the gradients (the backward / reduce-scatter).
    // Every run_update and gradients_finite first orders the engine's streams
    // after the work queued on it so far. Default: the legacy default stream
    // (also covers torch's default current stream).
    void set_producer_stream(cudaStream_t s);

    PhaseStats run_update(int iteration);

    int wait_host_resident(SubgroupId id);
    std::shared_future<IoStats> enqueue_flush(SubgroupId id, TierId dest);
    std::optional<std::shared_future<IoStats>> enqueue_prefetch(SubgroupId id);
    void read_current_state(SubgroupId id, float* out);

    const std::vector<SubgroupId>& subgroup_ids() const { return ids_; }
    Subgroup meta(SubgroupId id);
    std::uint64_t total_params() const;
    std::pair<std::uint64_t, std::vector<std::uint64_t>> residency_census();
    const BandwidthEstimate& estimates() const { return est_; }
    std::vector<SubgroupId> current_order();
    const ScheduleOptions& options() const { return opt_; }
    HostBufferPool& pool() { return *pool_; }
    const DeviceOptions& device_options() const { return dev_; }

    // Watchdog-guarded wait on an I/O future (rethrows tier errors).
    IoStats watchdog_wait_value(std::shared_future<IoStats>& fut);

private:
    struct DeviceEvents {
        cudaEvent_t h2d_start = nullptr, h2d_done = nullptr, k_start = nullptr, k_end = nullptr,
                    d2h_start = nullptr, d2h_end = nullptr, d2h_half = nullptr, h2d_half = nullptr;
    };
    struct Completion {
        SubgroupId id;
        int slot;
        int wb = -1;  // HBM cache mode: the write-back block the D2H went to
    };

    std::vector<double> placement_bandwidths() const;
    int retention_capacity() const;
    std::vector<int> tier_caps() const;
    bool hbm_cache_mode() const { return !hbm_cache_.empty() && dev_.hbm_retain == 2; }
    // HBM cache mode, op-level flush: a pool slot for an HBM-held subgroup's
    // write-back (no I/O; the slot goes straight to cached). Called with mu_
    // held; -1 if none free.
    int reserve_writeback_slot_locked(SubgroupId id);
    void pump_locked();
    std::shared_future<IoStats> start_prefetch_locked(SubgroupId id, int slot);
    // slot >= 0: flush from a pool slot; wb >= 0: from a write-back block.
    std::shared_future<IoStats> start_flush_locked(SubgroupId id, TierId dest, int slot, int wb = -1);
    void writeback_loop();
    enum class IoDir { read, write };
    void account_io_locked(SubgroupId id, TierId tier, const IoStats& st, IoDir dir, bool state_fetch);
    struct HostClaim {
        enum Kind { pending, hit, blocked } kind;
        std::shared_future<IoStats> fetch;  // pending: the fetch to wait on
    };
    HostClaim claim_host_locked(SubgroupId id);
    HostClaim claim_host(SubgroupId id);  // waits out `blocked`
    // ZeRO-3 baseline flow (skip_gradients = false): fp32 gradients through storage.
    void flush_grads_to_storage();
    void fetch_grads_for_cached(SubgroupId id);
    float* grad_annex(const HostBlock& blk) const {
        return reinterpret_cast<float*>(blk.base() + state_block_bytes_);
    }
    void wait_pool_free();

    void setup_device();
    void release_device();
    // Returns the PCIe bytes moved {H2D, D2H}.
    std::pair<std::uint64_t, std::uint64_t> issue_device_update(SubgroupId id, int slot, const AdamConsts& c);
    void device_state_to_host(const float* dev, float* host, std::uint64_t pc);
    void writeback_hbm_copy_locked(std::size_t k, int slot);
    // Header area + P||m||v of a contiguous state (seg_stride(pc) == pc):
    // block base <-> 32 bytes below P in a device state buffer.
    struct StateSpan {
        char* host;
        char* dev;
        std::size_t bytes;
    };
    static StateSpan state_span(float* dev_p, const HostBlock& blk, std::uint64_t pc) {
        return StateSpan{reinterpret_cast<char*>(blk.base()), reinterpret_cast<char*>(dev_p) - kHeaderBytes,
                         kHeaderBytes + 12 * static_cast<std::size_t>(pc)};
    }
    void copy_state(float* dev_base, const HostBlock& blk, std::uint64_t pc, bool to_device, cudaStream_t s);
    void completion_loop();
    static void CUDART_CB host_done(void* arg);
    std::size_t pick_next_ready(const std::vector<SubgroupId>& order, const std::vector<char>& issued,
                                std::size_t next);
    void count_grads_async();
    void launch_grad_check();
    std::int64_t await_grad_verdict();
    void roll_back_fetches();
    void order_after_producer();
    std::vector<unsigned long long> nonfinite_counts();

    WorkerId id_;
    std::vector<std::shared_ptr<Tier>> tiers_;
    ScheduleOptions opt_;
    AdamHyper hyper_;
    std::shared_ptr<EventTrace> trace_;
    DeviceOptions dev_;

    std::vector<std::unique_ptr<TierIoWorker>> io_;
    std::unique_ptr<HostBufferPool> pool_;
    std::unordered_map<SubgroupId, Subgroup> subgroups_;
    std::vector<SubgroupId> ids_;
    std::uint64_t max_params_ = 0;

    BandwidthEstimate est_;
    std::vector<double> fixed_ratio_;

    std::mutex mu_;
    std::vector<SubgroupId> order_;
    std::unique_ptr<DestinationPlan> dests_;
    std::size_t frontier_ = 0;
    std::unordered_map<SubgroupId, std::shared_future<IoStats>> prefetch_futures_;
    std::vector<std::pair<SubgroupId, std::shared_future<IoStats>>> flush_futures_;
    PhaseStats* phase_stats_ = nullptr;
    std::unordered_map<SubgroupId, std::size_t> io_index_;  // id -> phase_stats_->subgroup_io entry
    std::vector<char> updated_this_phase_;  // by index: issued in the current phase (the frontier skips it)
    std::uint64_t cache_hits_this_phase_ = 0;

    // Device resources.
    bool device_ready_ = false;
    cudaStream_t s_h2d_ = nullptr, s_k_ = nullptr, s_d2h_ = nullptr, s_d2h2_ = nullptr, s_h2d2_ = nullptr;
    std::vector<float*> ring_;
    std::vector<cudaEvent_t> ring_ready_;  // last D2H out of each ring buffer
    std::size_t ring_next_ = 0;           // round-robin ring cursor
    std::vector<float*> ring_grad_;  // baseline flow: fp32 gradient segment per ring buffer
    // HBM retention (DeviceOptions::hbm_retain): one device buffer per
    // retention slot. hbm_slot_[k] >= 0 while subgroup k's authoritative state
    // lives there (its host slot copy is stale); hbm_ready_[b] is the last D2H
    // out of buffer b, which a new occupant's H2D waits for.
    std::vector<float*> hbm_cache_;
    std::vector<cudaEvent_t> hbm_ready_;
    std::deque<int> hbm_free_;
    std::vector<int> hbm_slot_;
    // HBM cache mode: an HBM-held subgroup the plan flushes is written back
    // through its own small lane of pinned blocks (D2H -> block -> tier), so
    // the pool's slots serve only prefetches and the two directions overlap.
    // The coordinator only issues such a subgroup's kernel; the write-back
    // thread issues its D2H (on its own stream) once a block is free, then
    // releases the HBM buffer. Misses' H2D therefore start at phase begin.
    struct PendingWriteback {
        SubgroupId id;
        std::size_t k;
        int hslot;
        std::uint64_t pc;  // param count, captured when queued (read off the lock)
    };
    std::vector<HostBlock> wb_blocks_;
    std::deque<int> wb_free_;
    std::deque<PendingWriteback> wb_pending_;
    std::condition_variable wb_cv_;   // wb_free_ / wb_pending_ / hbm_free_ changed (with mu_)
    bool wb_stop_ = false;
    int wb_inflight_ = 0;  // deferred write-backs whose HBM buffer is not yet free
    // A write-back whose flush failed keeps its state in its block until a
    // pool slot adopts it (in plan order, pump_locked); id -> block.
    std::unordered_map<SubgroupId, int> wb_held_;
    // Two-level cache: HBM buffers this phase's newly retained subgroups may
    // still take (the rest stay in their host slots). Guarded by mu_.
    int hbm_budget_ = 0;
    int adopt_wb_held_locked(SubgroupId id);
    std::thread wb_thread_;
    float* grad32_dev_ = nullptr;    // baseline flow: widened gradients before the D2H
    // baseline flow: pinned D2H staging of fp32 gradients, a few in rotation so
    // the D2H of one subgroup overlaps the storage write of the previous ones
    std::vector<HostBlock> grad_stages_;
    std::vector<cudaEvent_t> grad_stage_ready_;
    std::deque<int> grad_stage_free_;
    std::condition_variable grad_stage_cv_;
    std::size_t state_block_bytes_ = 0;  // header + P||m||v of the largest subgroup, 4 KiB multiple
    std::size_t annex_bytes_ = 0;        // baseline flow: fp32 gradient annex after the state
    std::unordered_map<SubgroupId, TierId> grad_tier_;  // tier holding each subgroup's fp32 gradients
    std::uint64_t ring_stride_ = 0;  // floats per segment (P, m, v each) in a ring buffer
    void* grad_arena_ = nullptr;
    void* p16_arena_ = nullptr;
    // host_grads: per-subgroup pinned 16-bit gradient / working-param blocks,
    // and a device staging ring (gradient segment + params16 segment per
    // buffer) each update passes through; a buffer is free again once its
    // params16 D2H drained (aux_ready_).
    std::vector<HostBlock> grads_host_;
    std::vector<HostBlock> p16_host_;
    std::vector<std::uint16_t*> aux_;
    std::vector<cudaEvent_t> aux_ready_;
    std::size_t aux_next_ = 0;
    // Subgroups whose host gradients were produced by run_backward_sim (and
    // counted on the device as they were generated): their non-finite counts
    // need no second pass over PCIe. Cleared when the caller may write them.
    std::vector<char> grads_verified_;
    std::vector<unsigned long long> verified_counts_;

    cudaStream_t producer_ = cudaStreamLegacy;  // gradients' producer (set_producer_stream)
    cudaEvent_t producer_done_ = nullptr;
    cudaEvent_t verdict_ready_ = nullptr;            // per-subgroup non-finite counts landed in verdict_host_
    unsigned long long* verdict_host_ = nullptr;     // pinned, one count per subgroup (index order)
    unsigned long long* counters_ = nullptr;  // [0] non-finite grads, [1] narrowing overflows
    unsigned long long* sg_counts_ = nullptr; // per-subgroup non-finite counts (pre-check)
    std::unordered_map<SubgroupId, std::size_t> index_of_;
    std::vector<std::uint16_t*> grad_ptr_;
    std::vector<std::uint16_t*> arena_grad_;  // the engine's own gradient buffer per subgroup (bound sources reduce here)
    std::vector<std::vector<const void*>> grad_sources_;  // non-empty: fused multi-source reduction
    std::vector<std::uint16_t*> p16_ptr_;
    std::vector<DeviceEvents> events_;
    std::int64_t phase_t0_ns_ = 0;
    std::vector<std::int64_t> host_resident_ns_;  // per subgroup index
    std::vector<std::int64_t> host_retired_ns_;
    cudaEvent_t phase_origin_ = nullptr;  // recorded on the H2D stream at run_update entry

    // Completion thread: retires subgroups whose D2H finished.
    std::thread completer_;
    std::mutex cq_mu_;
    std::condition_variable cq_cv_;
    std::deque<Completion> cq_;
    bool cq_stop_ = false;
    std::size_t in_flight_ = 0;  // guarded by mu_
    std::condition_variable inflight_cv_;
    std::condition_variable resident_cv_;  // a fetch landed (or failed), with mu_
    std::exception_ptr completion_error_;
};

}  // namespace tfb
