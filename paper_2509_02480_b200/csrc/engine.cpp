// OffloadWorker: host scheduler + CUDA-stream update pipeline. See engine.hpp.
#include "engine.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels.hpp"
#include "nvtx.hpp"
#include "tier_lock.hpp"

namespace tfb {

namespace {

using Clock = std::chrono::steady_clock;

struct DeviceGuard {
    explicit DeviceGuard(int dev) { cuda_check(cudaSetDevice(dev), "cudaSetDevice"); }
};

constexpr std::uint64_t kSegAlign = 64;  // floats: 256-byte aligned P / m / v device segments

std::uint64_t seg_stride(std::uint64_t pc) { return (pc + kSegAlign - 1) / kSegAlign * kSegAlign; }

// Device state buffers (ring, HBM retention) keep kSegAlign floats of head
// room in front of P: the 32 bytes just below P mirror the host block's
// header area, so a contiguous P||m||v moves between the 4 KiB-aligned host
// block base and P - 32 as one copy with both ends on the block's alignment.
// (A copy starting at the payload, 32 bytes past a page boundary, loses
// ~8 GB/s of D2H when the H2D direction is busy: profiles/r2_align_probe.json.)
float* alloc_state_buffer(std::uint64_t stride, const char* what) {
    float* p = nullptr;
    cuda_check(cudaMalloc(reinterpret_cast<void**>(&p), (3 * stride + kSegAlign) * sizeof(float)), what);
    return p + kSegAlign;
}
void free_state_buffer(float* p) {
    if (p) cudaFree(p - kSegAlign);
}

}  // namespace

// --- hyperparameters ---------------------------------------------------------

void AdamHyper::validate() const {
    if (!(lr > 0.0)) throw ConfigError("optim.lr must be > 0");
    if (beta1 < 0.0 || beta1 >= 1.0) throw ConfigError("optim.beta1 must be in [0, 1)");
    if (beta2 < 0.0 || beta2 >= 1.0) throw ConfigError("optim.beta2 must be in [0, 1)");
    if (!(eps > 0.0)) throw ConfigError("optim.eps must be > 0");
    if (weight_decay < 0.0) throw ConfigError("optim.weight_decay must be >= 0");
}

AdamConsts AdamHyper::consts(std::uint64_t t) const {
    if (t < 1) throw Error("adam_step: timestep must be >= 1");
    validate();
    AdamConsts c{};
    c.lr = lr;
    c.beta1 = beta1;
    c.beta2 = beta2;
    c.one_minus_beta1 = 1.0 - beta1;
    c.one_minus_beta2 = 1.0 - beta2;
    c.eps = eps;
    c.lr_wd = weight_decay != 0.0 ? lr * weight_decay : 0.0;
    c.bc1 = 1.0 - std::pow(beta1, static_cast<double>(t));
    c.bc2 = 1.0 - std::pow(beta2, static_cast<double>(t));
    c.inv_bc1 = 1.0 / c.bc1;
    c.inv_bc2 = 1.0 / c.bc2;
    return c;
}

// --- residency ---------------------------------------------------------------

void Subgroup::begin_flush() {
    if (residency != Residency::host_cached)
        throw Error("subgroup " + std::to_string(id) + ": flush from non-host residency");
    residency = Residency::in_flight;
}
void Subgroup::finish_flush(TierId dest) {
    if (residency != Residency::in_flight)
        throw Error("subgroup " + std::to_string(id) + ": finish_flush while not in flight");
    residency = Residency::on_tier;
    tier = dest;
    slot = -1;
}
void Subgroup::begin_prefetch() {
    if (residency != Residency::on_tier)
        throw Error("subgroup " + std::to_string(id) + ": prefetch while not on a tier");
    residency = Residency::in_flight;
}
void Subgroup::finish_prefetch(int pool_slot) {
    if (residency != Residency::in_flight)
        throw Error("subgroup " + std::to_string(id) + ": finish_prefetch while not in flight");
    residency = Residency::host_cached;
    slot = pool_slot;
}

// --- pool --------------------------------------------------------------------

const char* slot_state_name(SlotState s) {
    switch (s) {
        case SlotState::free_slot: return "free";
        case SlotState::prefetching: return "prefetching";
        case SlotState::updating: return "updating";
        case SlotState::flushing: return "flushing";
        case SlotState::cached: return "cached";
    }
    return "unknown";
}

HostBufferPool::HostBufferPool(int slot_count, std::size_t block_bytes, bool require_pinned) {
    if (slot_count < 3) throw ConfigError("host buffer pool needs >= 3 slots");
    slots_.resize(static_cast<std::size_t>(slot_count));
    for (auto& s : slots_) s.block = HostBlock::allocate(block_bytes, require_pinned);
}

std::size_t HostBufferPool::check(int slot) const {
    if (slot < 0 || static_cast<std::size_t>(slot) >= slots_.size())
        throw Error("bad pool slot index " + std::to_string(slot));
    return static_cast<std::size_t>(slot);
}

void HostBufferPool::transition(int slot, SlotState expected, SlotState next) {
    std::lock_guard<std::mutex> g(mu_);
    Slot& s = slots_[check(slot)];
    if (s.state != expected)
        throw Error(std::string("pool slot ") + std::to_string(slot) + ": invalid transition " +
                    slot_state_name(s.state) + " -> " + slot_state_name(next) + " (expected " +
                    slot_state_name(expected) + ")");
    s.state = next;
}

int HostBufferPool::try_reserve(SubgroupId owner) {
    std::lock_guard<std::mutex> g(mu_);
    for (std::size_t i = 0; i < slots_.size(); ++i) {
        if (slots_[i].state == SlotState::free_slot) {
            slots_[i].state = SlotState::prefetching;
            slots_[i].owner = owner;
            return static_cast<int>(i);
        }
    }
    return -1;
}

int HostBufferPool::find_cached(SubgroupId owner) const {
    std::lock_guard<std::mutex> g(mu_);
    for (std::size_t i = 0; i < slots_.size(); ++i)
        if (slots_[i].state == SlotState::cached && slots_[i].owner == owner) return static_cast<int>(i);
    return -1;
}

void HostBufferPool::flush_done(int slot) {
    transition(slot, SlotState::flushing, SlotState::free_slot);
    free_cv_.notify_all();
}

void HostBufferPool::evict(int slot) {
    transition(slot, SlotState::cached, SlotState::free_slot);
    free_cv_.notify_all();
}

void HostBufferPool::release_failed(int slot) {
    std::lock_guard<std::mutex> g(mu_);
    slots_[check(slot)].state = SlotState::free_slot;
    free_cv_.notify_all();
}

SlotState HostBufferPool::state(int slot) const {
    std::lock_guard<std::mutex> g(mu_);
    return slots_[check(slot)].state;
}

SubgroupId HostBufferPool::owner(int slot) const {
    std::lock_guard<std::mutex> g(mu_);
    return slots_[check(slot)].owner;
}

int HostBufferPool::count(SlotState s) const {
    std::lock_guard<std::mutex> g(mu_);
    int n = 0;
    for (const auto& slot : slots_) n += slot.state == s;
    return n;
}

bool HostBufferPool::wait_for_free(std::chrono::milliseconds timeout) {
    std::unique_lock<std::mutex> g(mu_);
    return free_cv_.wait_for(g, timeout, [&] {
        for (const auto& s : slots_)
            if (s.state == SlotState::free_slot) return true;
        return false;
    });
}

// --- tier I/O workers ----------------------------------------------------------

TierIoWorker::TierIoWorker(std::shared_ptr<Tier> tier, WorkerId worker, bool use_lock,
                           std::filesystem::path lock_dir, EventTrace* trace)
    : tier_(std::move(tier)), worker_(worker), use_lock_(use_lock), lock_dir_(std::move(lock_dir)), trace_(trace) {
    thread_ = std::thread([this] { serve(); });
}

TierIoWorker::~TierIoWorker() { shutdown(); }

std::future<IoStats> TierIoWorker::submit(bool is_prefetch, std::int64_t sg, std::uint64_t bytes_hint,
                                          std::function<IoStats()> transfer, Completion completion) {
    Job job;
    job.lane = is_prefetch ? kFetch : kWriteBack;
    job.sg = sg;
    job.bytes_hint = bytes_hint;
    job.transfer = std::move(transfer);
    job.completion = std::move(completion);
    std::future<IoStats> result = job.promise.get_future();
    std::unique_lock<std::mutex> l(mu_);
    if (closed_) throw Error("tier I/O queue is shut down");
    lanes_[job.lane].push_back(std::move(job));
    l.unlock();
    wake_.notify_one();
    return result;
}

// A job that never ran: its owner learns through the completion (state
// rollback) and the future (the error).
void TierIoWorker::cancel(Job& job) {
    if (job.completion) job.completion(false, IoStats{});
    job.promise.set_exception(std::make_exception_ptr(Error("tier I/O queue shut down, operation cancelled")));
}

void TierIoWorker::shutdown() {
    std::unique_lock<std::mutex> l(mu_);
    if (closed_) return;
    closed_ = true;
    l.unlock();
    wake_.notify_all();
    if (thread_.joinable()) thread_.join();
    // The thread drains both lanes before it exits; a job that still shows up
    // here raced the close and is cancelled.
    for (auto& lane : lanes_) {
        while (!lane.empty()) {
            Job j = std::move(lane.front());
            lane.pop_front();
            cancel(j);
        }
    }
}

bool TierIoWorker::next_job(Job& out) {
    std::unique_lock<std::mutex> l(mu_);
    wake_.wait(l, [&] { return closed_ || !lanes_[kFetch].empty() || !lanes_[kWriteBack].empty(); });
    if (lanes_[kFetch].empty() && lanes_[kWriteBack].empty()) return false;  // closed and drained
    auto& lane = lanes_[kFetch].empty() ? lanes_[kWriteBack] : lanes_[kFetch];
    out = std::move(lane.front());
    lane.pop_front();
    return true;
}

void TierIoWorker::serve() {
    Job job;
    while (next_job(job)) {
        try {
            const IoStats st = transfer_traced(job);
            if (job.completion) job.completion(true, st);
            job.promise.set_value(st);
        } catch (...) {
            try {
                if (job.completion) job.completion(false, IoStats{});
            } catch (...) {
            }
            job.promise.set_exception(std::current_exception());
        }
        job = Job{};
    }
}

// The transfer under the tier semaphore; its traced interval (lock wait
// excluded) is the duration the metrics and the EMA use (reference
// scheduler.hpp:236-243). On failure the end event is still traced, with 0 bytes.
IoStats TierIoWorker::transfer_traced(Job& job) {
    const bool fetch = job.lane == kFetch;
    const TierId tid = tier_->id();
    const NvtxRange range("%s sg %lld tier %d", fetch ? "fetch" : "flush", static_cast<long long>(job.sg), tid);
    std::optional<TierLockGuard> sem;
    if (use_lock_)
        sem.emplace(lock_dir_, tid, worker_, trace_, tier_->spec().lock_width, tier_->spec().lock_device);
    const std::int64_t t0 = now_ns();
    if (trace_) {
        Event ev;
        ev.timestamp_ns = t0;
        ev.worker_id = worker_;
        ev.kind = static_cast<int>(fetch ? EventKind::prefetch_start : EventKind::flush_start);
        ev.subgroup_id = job.sg;
        ev.tier_id = tid;
        ev.bytes = job.bytes_hint;
        trace_->append(ev);
    }
    const EventKind end_kind = fetch ? EventKind::prefetch_end : EventKind::flush_end;
    IoStats st;
    try {
        st = job.transfer();
    } catch (...) {
        if (trace_) trace_->record(end_kind, worker_, job.sg, tid, 0);
        throw;
    }
    const std::int64_t t1 = now_ns();
    if (trace_) {
        Event ev;
        ev.timestamp_ns = t1;
        ev.worker_id = worker_;
        ev.kind = static_cast<int>(end_kind);
        ev.subgroup_id = job.sg;
        ev.tier_id = tid;
        ev.bytes = st.bytes;
        trace_->append(ev);
    }
    st.seconds = static_cast<double>(t1 - t0) / 1e9;
    return st;  // the semaphore is released here, before the completion runs
}

// --- OffloadWorker -------------------------------------------------------------

OffloadWorker::OffloadWorker(WorkerId id, std::vector<std::shared_ptr<Tier>> tiers, ScheduleOptions opt,
                             AdamHyper hyper, std::shared_ptr<EventTrace> trace, DeviceOptions dev)
    : id_(id), tiers_(std::move(tiers)), opt_(std::move(opt)), hyper_(hyper), trace_(std::move(trace)), dev_(dev) {
    if (tiers_.empty()) throw ConfigError("offload worker needs at least one tier");
    if (!trace_) trace_ = std::make_shared<EventTrace>();
    hyper_.validate();
    if (opt_.pool_slots < 3) throw ConfigError("host buffer pool needs >= 3 slots");
    if (dev_.device_buffers < 1) throw ConfigError("device_buffers must be >= 1");
    if (dev_.grad_kind != kF16 && dev_.grad_kind != kBF16) throw ConfigError("unknown gradient dtype");
    if (dev_.out_kind != kF16 && dev_.out_kind != kBF16) throw ConfigError("unknown working-param dtype");
    if (dev_.host_grads && (dev_.zero_copy != 0 || !opt_.skip_gradients))
        throw ConfigError("host_grads needs the copy pipeline (zero_copy 0) and the 16-bit gradient flow");
    if (opt_.lock_dir.empty()) opt_.lock_dir = (std::filesystem::temp_directory_path() / "tierflow-locks").string();
    std::vector<double> rbw, wbw;
    for (const auto& t : tiers_) {
        rbw.push_back(t->spec().read_bw);
        wbw.push_back(t->spec().write_bw);
    }
    est_ = BandwidthEstimate::init(rbw, wbw, 0.5);
    for (const auto& t : tiers_)
        io_.push_back(std::make_unique<TierIoWorker>(t, id_, opt_.atomic_rw, opt_.lock_dir, trace_.get()));
}

OffloadWorker::~OffloadWorker() {
    // Let in-flight device work retire before tearing the pipeline down.
    if (device_ready_) {
        cudaSetDevice(dev_.device);
        cudaStreamSynchronize(s_h2d_);
        cudaStreamSynchronize(s_k_);
        cudaStreamSynchronize(s_d2h_);
        cudaStreamSynchronize(s_d2h2_);
        cudaStreamSynchronize(s_h2d2_);
    }
    {
        std::lock_guard<std::mutex> g(mu_);
        wb_stop_ = true;
    }
    wb_cv_.notify_all();
    if (wb_thread_.joinable()) wb_thread_.join();
    {
        std::lock_guard<std::mutex> g(cq_mu_);
        cq_stop_ = true;
    }
    cq_cv_.notify_all();
    if (completer_.joinable()) completer_.join();
    for (auto& w : io_) w->shutdown();
    release_device();
}

void OffloadWorker::set_alpha(double alpha) {
    if (!(alpha > 0.0) || alpha > 1.0) throw ConfigError("placement.alpha must be in (0, 1]");
    est_.alpha = alpha;
}

void OffloadWorker::set_fixed_ratio(std::vector<double> ratio) { fixed_ratio_ = std::move(ratio); }

void OffloadWorker::set_cache_slots(int cache_slots) {
    std::lock_guard<std::mutex> g(mu_);
    if (in_flight_ != 0 || phase_stats_ != nullptr) throw Error("set_cache_slots during an update phase");
    if (hbm_cache_mode() && cache_slots > static_cast<int>(hbm_cache_.size()) &&
        !(dev_.hbm_cache_slots > 0))  // two-level: the excess is retained in host slots
        throw ConfigError("set_cache_slots: " + std::to_string(cache_slots) + " exceeds the " +
                          std::to_string(hbm_cache_.size()) + " HBM retention buffers allocated at init");
    opt_.cache_slots = cache_slots;
}

void OffloadWorker::add_subgroup(SubgroupId id, std::uint64_t param_count) {
    if (pool_) throw Error("add_subgroup after pipeline initialization");
    if (param_count == 0) throw ConfigError("subgroup param_count must be > 0");
    if (subgroups_.count(id)) throw ConfigError("duplicate subgroup id " + std::to_string(id));
    Subgroup sg;
    sg.id = id;
    sg.param_count = param_count;
    subgroups_.emplace(id, sg);
    ids_.push_back(id);
    max_params_ = std::max(max_params_, param_count);
}

std::vector<double> OffloadWorker::placement_bandwidths() const {
    std::vector<double> b = fixed_ratio_.empty() ? est_.effective_all() : fixed_ratio_;
    b.resize(tiers_.size(), 0.0);
    if (!opt_.multi_path)
        for (std::size_t i = 1; i < b.size(); ++i) b[i] = 0.0;
    return b;
}

// Per-tier subgroup capacity for the capacity-aware Eq. 1: the tier's
// capacity_bytes over the state block of the largest subgroup (-1: unlimited).
std::vector<int> OffloadWorker::tier_caps() const {
    std::vector<int> caps;
    for (const auto& t : tiers_) {
        const std::uint64_t cb = t->spec().capacity_bytes;
        caps.push_back(cb == 0 || state_block_bytes_ == 0 ? -1 : static_cast<int>(cb / state_block_bytes_));
    }
    return caps;
}

int OffloadWorker::retention_capacity() const {
    const int M = static_cast<int>(ids_.size());
    if (dev_.hbm_retain == 2 && dev_.zero_copy == 0 && opt_.skip_gradients && opt_.enable_caching) {
        int wanted = opt_.cache_slots < 0 ? opt_.pool_slots - 3 : opt_.cache_slots;
        if (dev_.hbm_cache_slots > 0)  // two-level: the host part keeps three slots streaming
            wanted = std::min(wanted, dev_.hbm_cache_slots + std::max(0, opt_.pool_slots - 3));
        return std::clamp(wanted, 0, M);
    }
    return opt_.retention_capacity(M);
}

int OffloadWorker::reserve_writeback_slot_locked(SubgroupId id) {
    const int slot = pool_->try_reserve(id);
    if (slot < 0) return -1;
    pool_->prefetch_done(slot);
    subgroups_.at(id).slot = slot;
    return slot;
}

void OffloadWorker::setup_device() {
    DeviceGuard dg(dev_.device);
    cuda_check(cudaStreamCreateWithFlags(&s_h2d_, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaStreamCreateWithFlags(&s_k_, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaStreamCreateWithFlags(&s_d2h_, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaStreamCreateWithFlags(&s_d2h2_, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaStreamCreateWithFlags(&s_h2d2_, cudaStreamNonBlocking), "cudaStreamCreate");
    ring_stride_ = seg_stride(max_params_);
    ring_.assign(static_cast<std::size_t>(dev_.device_buffers), nullptr);
    cuda_check(cudaEventCreate(&phase_origin_), "cudaEventCreate");
    ring_ready_.assign(ring_.size(), nullptr);
    for (std::size_t b = 0; b < ring_.size(); ++b) {
        ring_[b] = alloc_state_buffer(ring_stride_, "cudaMalloc(ring)");
        cuda_check(cudaEventCreateWithFlags(&ring_ready_[b], cudaEventDisableTiming), "cudaEventCreate");
    }
    ring_next_ = 0;
    if (!opt_.skip_gradients) {
        ring_grad_.assign(ring_.size(), nullptr);
        for (auto& r : ring_grad_)
            cuda_check(cudaMalloc(reinterpret_cast<void**>(&r), ring_stride_ * sizeof(float)), "cudaMalloc(ring grads)");
        cuda_check(cudaMalloc(reinterpret_cast<void**>(&grad32_dev_), ring_stride_ * sizeof(float)), "cudaMalloc");
        for (int b = 0; b < kGradStages; ++b) {
            grad_stages_.push_back(HostBlock::allocate(4 * static_cast<std::size_t>(max_params_), true));
            grad_stage_ready_.push_back(nullptr);
            cuda_check(cudaEventCreateWithFlags(&grad_stage_ready_.back(), cudaEventDisableTiming), "cudaEventCreate");
            grad_stage_free_.push_back(b);
        }
    }
    std::size_t arena = 0;
    std::vector<std::size_t> offs;
    for (const SubgroupId id : ids_) {
        offs.push_back(arena);
        arena += round_up(2 * subgroups_.at(id).param_count, 256);
    }
    if (dev_.host_grads) {
        for (const SubgroupId id : ids_) {
            const std::size_t bytes = 2 * static_cast<std::size_t>(subgroups_.at(id).param_count);
            grads_host_.push_back(HostBlock::allocate(bytes, true));
            std::memset(grads_host_.back().base(), 0, bytes);
            p16_host_.push_back(HostBlock::allocate(bytes, true));
        }
        aux_.assign(ring_.size(), nullptr);
        aux_ready_.assign(ring_.size(), nullptr);
        for (std::size_t b = 0; b < aux_.size(); ++b) {
            cuda_check(cudaMalloc(reinterpret_cast<void**>(&aux_[b]), 4 * ring_stride_), "cudaMalloc(staging)");
            cuda_check(cudaEventCreateWithFlags(&aux_ready_[b], cudaEventDisableTiming), "cudaEventCreate");
        }
        aux_next_ = 0;
        grads_verified_.assign(ids_.size(), 1);  // zero gradients: finite
        verified_counts_.assign(ids_.size(), 0);
    } else {
        cuda_check(cudaMalloc(&grad_arena_, std::max<std::size_t>(arena, 256)), "cudaMalloc(grads)");
        cuda_check(cudaMalloc(&p16_arena_, std::max<std::size_t>(arena, 256)), "cudaMalloc(params16)");
        cuda_check(cudaMemset(grad_arena_, 0, std::max<std::size_t>(arena, 256)), "cudaMemset(grads)");
    }
    cuda_check(cudaEventCreateWithFlags(&producer_done_, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventCreateWithFlags(&verdict_ready_, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&verdict_host_), std::max<std::size_t>(1, ids_.size()) *
                                                                          sizeof(unsigned long long),
                             cudaHostAllocDefault),
               "cudaHostAlloc(verdict)");
    cuda_check(cudaMalloc(reinterpret_cast<void**>(&counters_), 2 * sizeof(unsigned long long)), "cudaMalloc");
    cuda_check(cudaMalloc(reinterpret_cast<void**>(&sg_counts_), ids_.size() * sizeof(unsigned long long)),
               "cudaMalloc");
    hbm_slot_.assign(ids_.size(), -1);
    if (dev_.hbm_retain != 0 && dev_.zero_copy == 0 && opt_.skip_gradients) {
        int cap = retention_capacity();
        if (dev_.hbm_retain == 2 && dev_.hbm_cache_slots > 0) cap = std::min(cap, dev_.hbm_cache_slots);
        hbm_cache_.assign(static_cast<std::size_t>(cap), nullptr);
        hbm_ready_.assign(hbm_cache_.size(), nullptr);
        for (std::size_t b = 0; b < hbm_cache_.size(); ++b) {
            hbm_cache_[b] = alloc_state_buffer(ring_stride_, "cudaMalloc(hbm retention)");
            cuda_check(cudaEventCreateWithFlags(&hbm_ready_[b], cudaEventDisableTiming), "cudaEventCreate");
            hbm_free_.push_back(static_cast<int>(b));
        }
        if (dev_.hbm_retain == 2) {
            const int nwb = std::min<int>(kWritebackBlocks, std::max<int>(1, cap));
            for (int b = 0; b < nwb; ++b) {
                wb_blocks_.push_back(HostBlock::allocate(state_block_bytes_ + annex_bytes_, true));
                wb_free_.push_back(b);
            }
        }
    }
    grad_ptr_.clear();
    p16_ptr_.clear();
    arena_grad_.clear();
    events_.assign(ids_.size(), DeviceEvents{});
    grad_sources_.assign(ids_.size(), {});
    host_resident_ns_.assign(ids_.size(), 0);
    host_retired_ns_.assign(ids_.size(), 0);
    for (std::size_t k = 0; k < ids_.size(); ++k) {
        index_of_[ids_[k]] = k;
        if (dev_.host_grads) {
            grad_ptr_.push_back(reinterpret_cast<std::uint16_t*>(grads_host_[k].base()));
            p16_ptr_.push_back(reinterpret_cast<std::uint16_t*>(p16_host_[k].base()));
        } else {
            grad_ptr_.push_back(reinterpret_cast<std::uint16_t*>(static_cast<char*>(grad_arena_) + offs[k]));
            p16_ptr_.push_back(reinterpret_cast<std::uint16_t*>(static_cast<char*>(p16_arena_) + offs[k]));
        }
        arena_grad_.push_back(grad_ptr_.back());
        DeviceEvents& e = events_[k];
        for (cudaEvent_t* ev : {&e.h2d_start, &e.h2d_done, &e.k_start, &e.k_end, &e.d2h_start, &e.d2h_end})
            cuda_check(cudaEventCreate(ev), "cudaEventCreate");
        cuda_check(cudaEventCreateWithFlags(&e.d2h_half, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventCreateWithFlags(&e.h2d_half, cudaEventDisableTiming), "cudaEventCreate");
    }
    device_ready_ = true;
    completer_ = std::thread([this] { completion_loop(); });
    if (!wb_blocks_.empty()) wb_thread_ = std::thread([this] { writeback_loop(); });
}

void OffloadWorker::release_device() {
    if (!device_ready_) return;
    cudaSetDevice(dev_.device);
    for (auto& e : events_)
        for (cudaEvent_t ev : {e.h2d_start, e.h2d_done, e.k_start, e.k_end, e.d2h_start, e.d2h_end, e.d2h_half,
                               e.h2d_half})
            if (ev) cudaEventDestroy(ev);
    events_.clear();
    for (float* r : ring_) free_state_buffer(r);
    ring_.clear();
    if (phase_origin_) cudaEventDestroy(phase_origin_);
    phase_origin_ = nullptr;
    for (cudaEvent_t ev : ring_ready_)
        if (ev) cudaEventDestroy(ev);
    ring_ready_.clear();
    for (float* r : hbm_cache_) free_state_buffer(r);
    for (cudaEvent_t ev : hbm_ready_)
        if (ev) cudaEventDestroy(ev);
    hbm_cache_.clear();
    hbm_ready_.clear();
    hbm_free_.clear();
    hbm_slot_.clear();
    wb_blocks_.clear();
    wb_free_.clear();
    for (float* r : ring_grad_) cudaFree(r);
    ring_grad_.clear();
    if (grad32_dev_) cudaFree(grad32_dev_);
    grad32_dev_ = nullptr;
    for (cudaEvent_t ev : grad_stage_ready_)
        if (ev) cudaEventDestroy(ev);
    grad_stage_ready_.clear();
    grad_stages_.clear();
    grad_stage_free_.clear();
    cudaFree(grad_arena_);
    cudaFree(p16_arena_);
    for (std::uint16_t* a : aux_) cudaFree(a);
    aux_.clear();
    for (cudaEvent_t ev : aux_ready_)
        if (ev) cudaEventDestroy(ev);
    aux_ready_.clear();
    grads_host_.clear();
    p16_host_.clear();
    cudaFree(counters_);
    cudaFree(sg_counts_);
    if (producer_done_) cudaEventDestroy(producer_done_);
    producer_done_ = nullptr;
    if (verdict_ready_) cudaEventDestroy(verdict_ready_);
    verdict_ready_ = nullptr;
    if (verdict_host_) cudaFreeHost(verdict_host_);
    verdict_host_ = nullptr;
    cudaStreamDestroy(s_h2d_);
    cudaStreamDestroy(s_k_);
    cudaStreamDestroy(s_d2h_);
    cudaStreamDestroy(s_d2h2_);
    cudaStreamDestroy(s_h2d2_);
    device_ready_ = false;
}

// Host P||m||v (contiguous, stride pc) <-> device P / m / v segments (stride
// seg_stride(pc), 256-byte aligned). When the strides coincide, one copy of
// header area + payload from the block base (alloc_state_buffer); the header
// bytes that land in the host block are rewritten by every tier write.
void OffloadWorker::copy_state(float* dev_base, const HostBlock& blk, std::uint64_t pc, bool to_device,
                               cudaStream_t s) {
    const std::uint64_t ds = seg_stride(pc);
    const cudaMemcpyKind kind = to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
    float* host = blk.payload();
    if (ds == pc) {
        const StateSpan x = state_span(dev_base, blk, pc);
        cuda_check(to_device ? cudaMemcpyAsync(x.dev, x.host, x.bytes, kind, s)
                             : cudaMemcpyAsync(x.host, x.dev, x.bytes, kind, s),
                   "cudaMemcpyAsync(state)");
        return;
    }
    for (int k = 0; k < 3; ++k) {
        float* d = dev_base + k * ds;
        float* h = host + k * pc;
        cuda_check(to_device ? cudaMemcpyAsync(d, h, 4 * pc, kind, s) : cudaMemcpyAsync(h, d, 4 * pc, kind, s),
                   "cudaMemcpyAsync(state segment)");
    }
}

void OffloadWorker::init_and_flush_all(std::uint64_t seed) {
    if (ids_.empty()) throw ConfigError("worker has no subgroups");
    if (pool_) throw Error("init_and_flush_all called twice");
    std::sort(ids_.begin(), ids_.end());
    DeviceGuard dg(dev_.device);
    state_block_bytes_ = block_bytes_for(max_params_);
    annex_bytes_ = opt_.skip_gradients ? 0 : round_up(4 * static_cast<std::size_t>(max_params_), kPageBytes);
    pool_ = std::make_unique<HostBufferPool>(opt_.pool_slots, state_block_bytes_ + annex_bytes_, /*require_pinned=*/true);
    for (auto& t : tiers_) t->reserve_block_bytes(state_block_bytes_ + annex_bytes_);
    setup_device();

    const std::vector<SubgroupId> order = update_order(0, ids_, false);
    const DestinationPlan dests(order, 0, placement_bandwidths(), tier_caps());
    // Generate on the GPU into the ring, copy into a staging slot, persist.
    HostBlock staging = HostBlock::allocate(state_block_bytes_ + annex_bytes_, true);
    for (const SubgroupId id : order) {
        Subgroup& sg = subgroups_.at(id);
        const std::uint64_t pc = sg.param_count;
        const std::uint64_t ds = seg_stride(pc);
        float* d = ring_[0];
        cuda_check(launch_synthetic_state(d, d + ds, d + 2 * ds, pc, param_prefix(seed, id), s_k_),
                   "synthetic_state");
        cuda_check(cudaStreamSynchronize(s_k_), "cudaStreamSynchronize");
        copy_state(d, staging, pc, false, s_k_);
        cuda_check(cudaStreamSynchronize(s_k_), "cudaStreamSynchronize");
        const TierAssignment a = dests.assign_storage_tier(id);
        sg.begin_flush();
        tiers_[static_cast<std::size_t>(a.tier)]->write_from(id, pc, staging);
        sg.finish_flush(a.tier);
    }
}

void OffloadWorker::run_backward_sim(int iteration, std::uint64_t seed, int accum_steps) {
    if (accum_steps < 1) throw ConfigError("grad_accum_steps must be >= 1");
    if (!device_ready_) throw Error("run_backward_sim before init_and_flush_all");
    DeviceGuard dg(dev_.device);
    if (dev_.host_grads) {
        // Generated (and counted) on the device in a staging buffer, then
        // copied to the subgroup's pinned host block: the gradients a
        // ZeRO-Offload backward leaves in host memory.
        cuda_check(cudaMemsetAsync(sg_counts_, 0, ids_.size() * sizeof(unsigned long long), s_k_), "cudaMemsetAsync");
        cuda_check(cudaStreamWaitEvent(s_k_, aux_ready_[0], 0), "wait");  // staging buffer 0 is free
        for (std::size_t k = 0; k < ids_.size(); ++k) {
            const SubgroupId id = ids_[k];
            const std::uint64_t pc = subgroups_.at(id).param_count;
            std::uint16_t* g = aux_[0];
            for (int step = 0; step < accum_steps; ++step)
                cuda_check(launch_synthetic_grads(g, pc, dev_.grad_kind, grad_prefix(seed, id, iteration, step),
                                                  step > 0, s_k_),
                           "synthetic_grads");
            cuda_check(launch_count_nonfinite16(g, pc, dev_.grad_kind, sg_counts_ + k, s_k_), "count_nonfinite");
            cuda_check(cudaMemcpyAsync(grad_ptr_[k], g, 2 * pc, cudaMemcpyDeviceToHost, s_k_), "cudaMemcpyAsync(grads)");
        }
        cuda_check(cudaMemcpyAsync(verified_counts_.data(), sg_counts_, ids_.size() * sizeof(unsigned long long),
                                   cudaMemcpyDeviceToHost, s_k_),
                   "cudaMemcpyAsync(counts)");
        cuda_check(cudaStreamSynchronize(s_k_), "cudaStreamSynchronize");
        std::fill(grads_verified_.begin(), grads_verified_.end(), 1);
        return;
    }
    for (std::size_t k = 0; k < ids_.size(); ++k) {
        const SubgroupId id = ids_[k];
        const std::uint64_t pc = subgroups_.at(id).param_count;
        for (int step = 0; step < accum_steps; ++step)
            cuda_check(launch_synthetic_grads(grad_ptr_[k], pc, dev_.grad_kind, grad_prefix(seed, id, iteration, step),
                                              step > 0, s_k_),
                       "synthetic_grads");
    }
    cuda_check(cudaStreamSynchronize(s_k_), "cudaStreamSynchronize");
    if (!opt_.skip_gradients) flush_grads_to_storage();
}

// ZeRO-3 data flow (reference scheduler.hpp:377-391): widen every subgroup's
// accumulated gradient to fp32 (on the GPU here, traced as the upscale), copy
// it to the host and flush it to the subgroup's current tier (tier 0 when the
// subgroup is host-resident) through the tier's I/O queue; 4 bytes/param of
// storage writes that the engine flow avoids.
void OffloadWorker::flush_grads_to_storage() {
    std::vector<std::future<IoStats>> pending;
    for (std::size_t k = 0; k < ids_.size(); ++k) {
        const SubgroupId id = ids_[k];
        const std::uint64_t pc = subgroups_.at(id).param_count;
        int b;
        {
            std::unique_lock<std::mutex> l(mu_);
            while (grad_stage_free_.empty()) grad_stage_cv_.wait_for(l, std::chrono::milliseconds(50));
            b = grad_stage_free_.front();
            grad_stage_free_.pop_front();
        }
        float* stage = reinterpret_cast<float*>(grad_stages_[static_cast<std::size_t>(b)].base());
        const cudaEvent_t ready = grad_stage_ready_[static_cast<std::size_t>(b)];
        trace_->record(EventKind::grad_upscale_start, id_, id, kNoTier, 4 * pc);
        cuda_check(launch_widen16(grad_ptr_[k], grad32_dev_, pc, dev_.grad_kind, nullptr, s_k_), "widen16");
        cuda_check(cudaMemcpyAsync(stage, grad32_dev_, 4 * pc, cudaMemcpyDeviceToHost, s_k_), "cudaMemcpyAsync(grads)");
        cuda_check(cudaEventRecord(ready, s_k_), "cudaEventRecord");
        trace_->record(EventKind::grad_upscale_end, id_, id, kNoTier, 4 * pc);
        TierId dest;
        {
            std::lock_guard<std::mutex> g(mu_);
            const Subgroup& sg = subgroups_.at(id);
            dest = sg.residency == Residency::on_tier ? sg.tier : 0;
            grad_tier_[id] = dest;
        }
        auto tier = tiers_[static_cast<std::size_t>(dest)];
        const int device = dev_.device;
        // The write waits for the D2H on the tier's I/O thread; the stage goes
        // back to the rotation when the write completes (or fails).
        auto transfer = [tier, id, pc, stage, ready, device] {
            cudaSetDevice(device);
            cuda_check(cudaEventSynchronize(ready), "cudaEventSynchronize(grads)");
            return tier->write_grads(id, pc, stage);
        };
        auto release = [this, b](bool, const IoStats&) {
            {
                std::lock_guard<std::mutex> g(mu_);
                grad_stage_free_.push_back(b);
            }
            grad_stage_cv_.notify_all();
        };
        pending.push_back(io_[static_cast<std::size_t>(dest)]->submit(false, id, 4 * pc, std::move(transfer),
                                                                      std::move(release)));
    }
    for (auto& f : pending) {
        std::shared_future<IoStats> s = f.share();
        watchdog_wait_value(s);
    }
}

// Grad-only fetch for a host-retained subgroup (reference scheduler.hpp:746-765).
void OffloadWorker::fetch_grads_for_cached(SubgroupId id) {
    TierId gt;
    std::uint64_t pc;
    int slot;
    {
        std::lock_guard<std::mutex> g(mu_);
        gt = grad_tier_.at(id);
        pc = subgroups_.at(id).param_count;
        slot = subgroups_.at(id).slot;
    }
    auto tier = tiers_[static_cast<std::size_t>(gt)];
    float* dst = grad_annex(pool_->block(slot));
    std::shared_future<IoStats> fut =
        io_[static_cast<std::size_t>(gt)]
            ->submit(true, id, 4 * pc, [tier, id, pc, dst] { return tier->read_grads(id, pc, dst); }, nullptr)
            .share();
    const IoStats st = watchdog_wait_value(fut);
    std::lock_guard<std::mutex> g(mu_);
    account_io_locked(id, gt, st, IoDir::read, /*state_fetch=*/false);
}

void* OffloadWorker::grad_buffer(SubgroupId id) {
    if (!device_ready_) throw Error("grad_buffer before init_and_flush_all");
    const std::size_t k = index_of_.at(id);
    if (dev_.host_grads) grads_verified_.at(k) = 0;  // the caller may write it now
    return grad_ptr_.at(k);
}

void OffloadWorker::bind_grad_buffer(SubgroupId id, void* device_ptr) {
    if (!device_ready_) throw Error("bind_grad_buffer before init_and_flush_all");
    if (device_ptr == nullptr) throw ConfigError("bind_grad_buffer: null device pointer");
    const std::size_t k = index_of_.at(id);
    grad_ptr_.at(k) = static_cast<std::uint16_t*>(device_ptr);  // host_grads: a pinned host pointer
    grad_sources_.at(k).clear();
    if (dev_.host_grads) grads_verified_.at(k) = 0;
}

void OffloadWorker::bind_grad_sources(SubgroupId id, const std::vector<const void*>& sources) {
    if (!device_ready_) throw Error("bind_grad_sources before init_and_flush_all");
    if (sources.empty() || sources.size() > static_cast<std::size_t>(kMaxGradSources))
        throw ConfigError("bind_grad_sources: 1.." + std::to_string(kMaxGradSources) + " sources");
    if (!opt_.skip_gradients) throw ConfigError("bind_grad_sources: not available in the baseline gradient flow");
    if (dev_.host_grads) throw ConfigError("bind_grad_sources: the sources are device buffers (host_grads is on)");
    for (const void* s : sources)
        if (s == nullptr) throw ConfigError("bind_grad_sources: null device pointer");
    grad_sources_.at(index_of_.at(id)) = sources;
}

void OffloadWorker::set_producer_stream(cudaStream_t s) { producer_ = s; }

// Gradients are read on s_k_ (pre-check, fused kernel): order it after what
// the producer stream has queued so far, so a caller that filled or bound the
// buffers asynchronously (a reduce-scatter, a backward) needs no host sync.
void OffloadWorker::order_after_producer() {
    cuda_check(cudaEventRecord(producer_done_, producer_), "cudaEventRecord(producer)");
    cuda_check(cudaStreamWaitEvent(s_k_, producer_done_, 0), "cudaStreamWaitEvent(producer)");
}

void* OffloadWorker::params16_buffer(SubgroupId id) {
    if (!device_ready_) throw Error("params16_buffer before init_and_flush_all");
    return p16_ptr_.at(index_of_.at(id));
}

// Non-finite gradient count per subgroup (index order): of the bound buffer,
// or of the rounded fp32 sum for a subgroup fed by several sources.
// Per-subgroup non-finite gradient counts into sg_counts_, async on s_k_:
// a device buffer in place, several sources as their rounded fp32 sum. With
// host_grads, a block its producer (run_backward_sim) counted as it wrote it
// keeps that count; any other is staged through the staging ring and counted
// (2 B/param over PCIe).
void OffloadWorker::count_grads_async() {
    const std::size_t M = ids_.size();
    if (dev_.host_grads) {
        for (std::size_t k = 0; k < M; ++k) verdict_host_[k] = grads_verified_[k] ? verified_counts_[k] : 0;
        cuda_check(cudaMemcpyAsync(sg_counts_, verdict_host_, M * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                                   s_k_),
                   "cudaMemcpyAsync(counts)");
        cuda_check(cudaStreamWaitEvent(s_k_, aux_ready_[0], 0), "wait");
    } else {
        cuda_check(cudaMemsetAsync(sg_counts_, 0, M * sizeof(unsigned long long), s_k_), "cudaMemsetAsync");
    }
    for (std::size_t k = 0; k < M; ++k) {
        const std::uint64_t pc = subgroups_.at(ids_[k]).param_count;
        if (!grad_sources_[k].empty()) {
            // The contributions are reduced here, once (2(N-1) B/param over
            // NVLink for N peers), into the subgroup's own gradient buffer,
            // which the update then reads: the check sees exactly the rounded
            // sum the update uses, and a sum that overflows the 16-bit range
            // rejects the phase before any state moves.
            cuda_check(launch_reduce_sum16(grad_sources_[k].data(), static_cast<int>(grad_sources_[k].size()), pc,
                                           dev_.grad_kind, arena_grad_[k], sg_counts_ + k, s_k_),
                       "reduce_sum16");
        } else if (dev_.host_grads) {
            if (grads_verified_[k]) continue;
            cuda_check(cudaMemcpyAsync(aux_[0], grad_ptr_[k], 2 * pc, cudaMemcpyHostToDevice, s_k_),
                       "cudaMemcpyAsync(grads)");
            cuda_check(launch_count_nonfinite16(aux_[0], pc, dev_.grad_kind, sg_counts_ + k, s_k_), "count_nonfinite");
        } else {
            cuda_check(launch_count_nonfinite16(grad_ptr_[k], pc, dev_.grad_kind, sg_counts_ + k, s_k_),
                       "count_nonfinite");
        }
    }
    if (dev_.host_grads) cuda_check(cudaEventRecord(aux_ready_[0], s_k_), "cudaEventRecord");
}

std::vector<unsigned long long> OffloadWorker::nonfinite_counts() {
    count_grads_async();
    std::vector<unsigned long long> counts(ids_.size());
    cuda_check(cudaMemcpyAsync(counts.data(), sg_counts_, counts.size() * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, s_k_),
               "cudaMemcpyAsync");
    cuda_check(cudaStreamSynchronize(s_k_), "cudaStreamSynchronize");
    return counts;
}

bool OffloadWorker::gradients_finite() {
    if (!device_ready_) throw Error("gradients_finite before init_and_flush_all");
    DeviceGuard dg(dev_.device);
    order_after_producer();
    for (const auto c : nonfinite_counts())
        if (c != 0) return false;
    return true;
}

// The reference rejects non-finite gradients before mutating a subgroup
// (precision.hpp:17-25 via scheduler.hpp:467-471; its harness checks the
// whole model first, harness.hpp:218-228). The fused kernel widens and
// updates in one pass, so the whole phase is checked before the first update
// instead: one 2-byte/param count on the kernel stream (2n for n summed
// sources), its per-subgroup counts copied back asynchronously. The host
// does not wait for them before the phase's fetches start; it waits before
// issuing the first update (await_grad_verdict), by which time the count has
// long finished under the first fetch.
void OffloadWorker::launch_grad_check() {
    count_grads_async();
    cuda_check(cudaMemcpyAsync(verdict_host_, sg_counts_, ids_.size() * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, s_k_),
               "cudaMemcpyAsync(verdict)");
    cuda_check(cudaEventRecord(verdict_ready_, s_k_), "cudaEventRecord(verdict)");
}

// First subgroup with a non-finite gradient in plan order, or -1.
std::int64_t OffloadWorker::await_grad_verdict() {
    cuda_check(cudaEventSynchronize(verdict_ready_), "cudaEventSynchronize(verdict)");
    for (const SubgroupId id : order_)
        if (verdict_host_[index_of_.at(id)] != 0) return id;
    return -1;
}

// A rejected phase leaves no trace in residency: fetches it issued complete,
// then their subgroups go back to the tier they came from and the slots are
// freed, so the next phase sees exactly the cache hits of the last applied
// phase (harness.hpp:218-228: a skipped step is as if run_update was never
// called). Nothing was updated, so a directory tier's file is still current;
// a host_dram tier handed its block to the slot, so the block goes back.
void OffloadWorker::roll_back_fetches() {
    std::vector<std::shared_future<IoStats>> pending;
    {
        std::lock_guard<std::mutex> g(mu_);
        frontier_ = order_.size();  // no new fetches
        for (auto& [fid, fut] : prefetch_futures_) pending.push_back(fut);
    }
    for (auto& f : pending) {
        try {
            watchdog_wait_value(f);
        } catch (const SchedulingBugError&) {
            throw;
        } catch (...) {  // a failed fetch already left its subgroup on its tier
        }
    }
    std::lock_guard<std::mutex> g(mu_);
    for (auto& [fid, fut] : prefetch_futures_) {
        Subgroup& sg = subgroups_.at(fid);
        if (sg.residency == Residency::host_cached && sg.slot >= 0) {
            Tier& origin = *tiers_.at(static_cast<std::size_t>(sg.tier));
            if (!origin.has_subgroup(fid)) origin.write_from(fid, sg.param_count, pool_->block(sg.slot));
            pool_->evict(sg.slot);
            sg.slot = -1;
            sg.residency = Residency::on_tier;
        }
    }
    prefetch_futures_.clear();
    phase_stats_ = nullptr;
}

PhaseStats OffloadWorker::run_update(int iteration) {
    if (!pool_) throw Error("run_update before init_and_flush_all");
    DeviceGuard dg(dev_.device);
    const NvtxRange range("run_update worker %d iter %d", id_, iteration);
    const auto t0 = Clock::now();
    phase_t0_ns_ = now_ns();
    const AdamConsts c = hyper_.consts(static_cast<std::uint64_t>(iteration) + 1);

    PhaseStats stats;
    stats.tier_obs.assign(tiers_.size(), TierObservation{});
    {
        std::lock_guard<std::mutex> g(mu_);
        order_ = update_order(iteration, ids_, opt_.enable_caching);
    }
    // timeline origin: the phase start on the H2D stream
    cuda_check(cudaEventRecord(phase_origin_, s_h2d_), "cudaEventRecord");
    order_after_producer();
    launch_grad_check();
    cuda_check(cudaMemsetAsync(counters_, 0, 2 * sizeof(unsigned long long), s_k_), "cudaMemsetAsync");
    std::vector<SubgroupId> order;
    {
        std::lock_guard<std::mutex> g(mu_);
        const int cap = retention_capacity();
        dests_ = std::make_unique<DestinationPlan>(order_, cap, placement_bandwidths(), tier_caps());
        if (hbm_cache_mode()) {
            // Newly retained subgroups take HBM buffers while there are any:
            // the free ones plus those the flushed HBM-held hits release.
            int released = 0, wanted = 0;
            for (const SubgroupId sid : order_) {
                const std::size_t k = index_of_.at(sid);
                const bool keep = dests_->assign_storage_tier(sid).host_retain;
                if (hbm_slot_[k] >= 0 && !keep) ++released;
                if (hbm_slot_[k] < 0 && keep) ++wanted;
            }
            hbm_budget_ = std::min(wanted, static_cast<int>(hbm_free_.size()) + released);
        }
        stats.retained = dests_->retained_count();
        stats.flush_allocation = dests_->flush_allocation().counts;
        frontier_ = 0;
        prefetch_futures_.clear();
        flush_futures_.clear();
        cache_hits_this_phase_ = 0;
        phase_stats_ = &stats;
        io_index_.clear();
        updated_this_phase_.assign(ids_.size(), 0);
        completion_error_ = nullptr;
        order = order_;
        pump_locked();
    }

    if (const std::int64_t bad = await_grad_verdict(); bad >= 0) {
        roll_back_fetches();
        throw GradientOverflowError("subgroup " + std::to_string(bad) +
                                    ": non-finite gradients reached the update phase");
    }
    try {
        // Updates are issued as their subgroups become host-resident, scanning
        // a window of the plan ahead of the first one not yet issued: a slow
        // fetch (a directory tier) no longer idles the H2D stream while later
        // subgroups sit ready in their slots. Plan order still drives every
        // rule that has an order (fetch frontier, destinations, retention,
        // hits), and subgroups are independent, so results, cache hits and
        // per-tier fetch / flush sequences are those of the in-order loop.
        std::vector<char> issued(order.size(), 0);
        std::size_t next = 0;
        std::deque<cudaEvent_t> h2d_queued;  // h2d_done of the state copies issued and not yet drained
        auto h2d_backlog = [&] {
            while (!h2d_queued.empty()) {
                const cudaError_t q = cudaEventQuery(h2d_queued.front());
                if (q == cudaErrorNotReady) break;
                cuda_check(q, "cudaEventQuery(h2d)");
                h2d_queued.pop_front();
            }
            return static_cast<int>(h2d_queued.size());
        };
        for (std::size_t done = 0; done < order.size(); ++done) {
            while (issued[next]) ++next;
            // Hold the next state copy on the host while the H2D stream has
            // kH2dAhead queued: the choice is made as late as possible.
            while (h2d_backlog() >= kH2dAhead) {
                std::this_thread::sleep_for(std::chrono::microseconds(500));
                std::lock_guard<std::mutex> g(mu_);
                if (completion_error_) std::rethrow_exception(completion_error_);
            }
            const std::size_t j = pick_next_ready(order, issued, next);
            issued[j] = 1;
            const SubgroupId id = order[j];
            const NvtxRange sg_range("subgroup %u (plan %zu of %zu)", id, j + 1, order.size());
            const int slot = wait_host_resident(id);
            host_resident_ns_[index_of_.at(id)] = now_ns();
            const auto moved = issue_device_update(id, slot, c);
            if (moved.first > 0) h2d_queued.push_back(events_[index_of_.at(id)].h2d_done);
            std::lock_guard<std::mutex> g(mu_);
            Subgroup& sg = subgroups_.at(id);
            sg.step_count = static_cast<std::uint64_t>(iteration) + 1;
            stats.params_updated += sg.param_count;
            stats.h2d_bytes += moved.first;
            stats.d2h_bytes += moved.second;
            if (completion_error_) std::rethrow_exception(completion_error_);
        }
        // All device updates retire, then the lazy flushes drain.
        {
            std::unique_lock<std::mutex> l(mu_);
            std::uint64_t last = trace_->progress_count();
            double stalled = 0.0;
            while (in_flight_ > 0) {
                if (inflight_cv_.wait_for(l, std::chrono::milliseconds(50)) == std::cv_status::timeout) {
                    const std::uint64_t p = trace_->progress_count();
                    if (p != last) {
                        last = p;
                        stalled = 0.0;
                    } else if ((stalled += 0.05) >= opt_.deadlock_timeout_s) {
                        throw SchedulingBugError("device pipeline made no progress for " +
                                                 std::to_string(opt_.deadlock_timeout_s) + "s");
                    }
                }
            }
            if (completion_error_) std::rethrow_exception(completion_error_);
        }
        std::vector<std::pair<SubgroupId, std::shared_future<IoStats>>> pending;
        {
            std::lock_guard<std::mutex> g(mu_);
            pending = flush_futures_;
        }
        for (auto& [fid, fut] : pending) watchdog_wait_value(fut);
        // host_grads: the working params' D2H of a subgroup whose state went
        // back through the write-back lane may still be in flight; the host
        // blocks are the caller's once run_update returns.
        if (dev_.host_grads) cuda_check(cudaStreamSynchronize(s_d2h_), "cudaStreamSynchronize");
    } catch (...) {
        std::lock_guard<std::mutex> g(mu_);
        phase_stats_ = nullptr;
        throw;
    }

    unsigned long long counters[2] = {0, 0};
    cuda_check(cudaMemcpyAsync(counters, counters_, sizeof(counters), cudaMemcpyDeviceToHost, s_k_), "cudaMemcpyAsync");
    cuda_check(cudaStreamSynchronize(s_k_), "cudaStreamSynchronize");
    stats.downscale_overflows = counters[1];
    if (counters[0] != 0)
        throw SchedulingBugError("non-finite gradients reached the fused kernel after the pre-check");

    // Device timeline of the phase (CUDA events) + host retire times.
    if (!order.empty()) {
        const cudaEvent_t origin = phase_origin_;
        auto at = [&](cudaEvent_t ev) {
            float ms = 0.0f;
            return cudaEventElapsedTime(&ms, origin, ev) == cudaSuccess ? ms : -1.0f;
        };
        for (const SubgroupId id : order) {
            const std::size_t k = index_of_.at(id);
            const DeviceEvents& e = events_[k];
            DeviceSpan sp;
            sp.id = id;
            sp.h2d_start = at(e.h2d_start);
            sp.h2d_end = at(e.h2d_done);
            sp.k_start = at(e.k_start);
            sp.k_end = at(e.k_end);
            sp.d2h_end = at(e.d2h_end);
            const float d2h_start = at(e.d2h_start);
            sp.d2h_start = d2h_start;
            sp.host_resident = static_cast<float>((host_resident_ns_[k] - phase_t0_ns_) / 1e6);
            sp.host_retired = static_cast<float>((host_retired_ns_[k] - phase_t0_ns_) / 1e6);
            stats.h2d_seconds += (sp.h2d_end - sp.h2d_start) / 1e3;
            stats.kernel_seconds += (sp.k_end - sp.k_start) / 1e3;
            stats.d2h_seconds += (sp.d2h_end - d2h_start) / 1e3;
            stats.timeline.push_back(sp);
        }
        for (const DeviceSpan& sp : stats.timeline)
            stats.device_seconds = std::max(stats.device_seconds, static_cast<double>(sp.d2h_end) / 1e3);
    }
    (void)cudaGetLastError();

    {
        std::lock_guard<std::mutex> g(mu_);
        phase_stats_ = nullptr;
        stats.cache_hits = cache_hits_this_phase_;
        prefetch_futures_.clear();
        flush_futures_.clear();
    }
    if (std::getenv("TFB_DEBUG_RESIDENCY") != nullptr) {  // forensics: host-resident beyond the retained set
        std::lock_guard<std::mutex> g(mu_);
        int host = 0;
        for (const SubgroupId sid : ids_) host += subgroups_.at(sid).residency == Residency::host_cached;
        if (host != stats.retained) {
            std::fprintf(stderr, "residency: %d host-resident after the phase, %d retained;", host, stats.retained);
            for (const SubgroupId sid : ids_) {
                const Subgroup& sg = subgroups_.at(sid);
                if (sg.residency == Residency::host_cached && !dests_->assign_storage_tier(sid).host_retain)
                    std::fprintf(stderr, " %u(slot %d hbm %d wb %d)", sid, sg.slot, hbm_slot_[index_of_.at(sid)],
                                 static_cast<int>(wb_held_.count(sid)));
            }
            std::fprintf(stderr, "\n");
        }
    }
    stats.wall_seconds = std::chrono::duration<double>(Clock::now() - t0).count();
    if (fixed_ratio_.empty()) {
        // A host_dram tier moves a subgroup by exchanging pinned blocks with
        // the slot: O(1), not a bandwidth sample. Its cost is the PCIe leg of
        // the device pipeline, so Eq. 1 keeps its configured rate (set it to
        // the measured PCIe rate) instead of learning ~1e14 B/s from a swap.
        std::vector<TierObservation> ema_obs = stats.tier_obs;
        for (std::size_t i = 0; i < tiers_.size(); ++i)
            if (tiers_[i]->spec().kind == TierKind::host_dram) ema_obs[i] = TierObservation{};
        est_.update(ema_obs);
    }
    return stats;
}

// The plan position to issue next: the first one from `next` on that is
// host-resident (a hit, or its fetch has landed) or whose fetch failed
// (wait_host_resident surfaces the error); else `next` itself once it has no
// fetch in flight (wait_host_resident fetches it on demand, as the reference)
// or once nothing lands for a second (wait_host_resident's watchdog then owns
// the wait). The scan is not limited to pool_slots positions: while a slow
// directory fetch holds `next`, the slots of the subgroups issued past it
// turn over and the frontier refills them further down the plan; those must
// stay issuable, or the H2D stream idles until the slow fetch lands.
// Among the ready ones, a subgroup the plan flushes to a directory tier goes
// first: its write then overlaps the PCIe traffic of the rest of the phase
// instead of trailing it (the reference's greedy destination plan puts those
// flushes at the end of the order, and the phase waits for every flush).
// Fetch order (the frontier), cache hits and flush sets are unchanged.
std::size_t OffloadWorker::pick_next_ready(const std::vector<SubgroupId>& order, const std::vector<char>& issued,
                                           std::size_t next) {
    const std::size_t window = order.size();
    std::unique_lock<std::mutex> l(mu_);
    auto ready = [&](SubgroupId id) {
        if (subgroups_.at(id).residency == Residency::host_cached) return true;
        const auto f = prefetch_futures_.find(id);
        return f != prefetch_futures_.end() && f->second.wait_for(std::chrono::seconds(0)) == std::future_status::ready;
    };
    auto slow_dest = [&](SubgroupId id) {
        const TierAssignment a = dests_->assign_storage_tier(id);
        return !a.host_retain && a.tier != kNoTier &&
               tiers_[static_cast<std::size_t>(a.tier)]->spec().kind != TierKind::host_dram;
    };
    for (int waited_ms = 0; waited_ms < 1000; waited_ms += 5) {
        std::size_t first = window;
        for (std::size_t j = next; j < window; ++j) {
            if (issued[j] || !ready(order[j])) continue;
            if (slow_dest(order[j])) return j;
            if (first == window) first = j;
        }
        if (first != window) return first;
        if (prefetch_futures_.count(order[next]) == 0) return next;
        if (completion_error_) std::rethrow_exception(completion_error_);
        resident_cv_.wait_for(l, std::chrono::milliseconds(5));
    }
    return next;
}

// Enqueue one subgroup on the three pipeline streams (H2D -> kernel -> D2H).
std::pair<std::uint64_t, std::uint64_t> OffloadWorker::issue_device_update(SubgroupId id, int slot,
                                                                         const AdamConsts& c) {
    Subgroup& sg = subgroups_.at(id);
    const std::uint64_t pc = sg.param_count;
    const std::size_t k = index_of_.at(id);
    const std::size_t K = ring_.size();
    const DeviceEvents& e = events_[k];
    {
        std::lock_guard<std::mutex> g(mu_);
        if (slot >= 0) pool_->begin_update(slot);
        trace_->record(EventKind::update_start, id_, id, kNoTier, 12 * pc);
        updated_this_phase_[k] = 1;
        ++in_flight_;
    }
    // slot < 0 only in HBM cache mode, for a subgroup held in HBM: retained
    // again it needs no host transfer; flushed, its D2H is deferred to the
    // write-back thread (wb_pending_).
    static HostBlock no_block;
    const HostBlock& blk = slot >= 0 ? pool_->block(slot) : no_block;
    AdamLaunch a;
    // Bound sources were reduced into the subgroup's own buffer at the phase check.
    a.g = grad_sources_[k].empty() ? grad_ptr_[k] : arena_grad_[k];
    a.p16 = p16_ptr_[k];
    a.n = pc;
    a.grad_kind = dev_.grad_kind;
    a.out_kind = dev_.out_kind;
    a.c = c;
    a.counters = counters_;
    // run_update awaited the whole-phase count of exactly these gradients
    // (await_grad_verdict) before the first issue.
    a.grads_verified = true;
    if (dev_.zero_copy == 1) {
        // The kernel streams P||m||v straight from and back to the pinned
        // slot over PCIe: reads and writes interleave at cache-line grain,
        // loading both link directions evenly; no device ring, no DMA.
        float* hp = nullptr;
        cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hp), blk.payload(), 0),
                   "cudaHostGetDevicePointer");
        a.p = hp;
        a.m = hp + pc;
        a.v = hp + 2 * pc;
        if (!opt_.skip_gradients) {  // baseline flow: fp32 gradients from the slot's annex
            void* hg = nullptr;
            cuda_check(cudaHostGetDevicePointer(&hg, grad_annex(blk), 0), "cudaHostGetDevicePointer");
            a.g = hg;
            a.grad_kind = kF32;
        }
        for (cudaEvent_t ev : {e.h2d_start, e.h2d_done, e.k_start})
            cuda_check(cudaEventRecord(ev, s_k_), "cudaEventRecord");
        cuda_check(launch_spin_ns(opt_.update_pad_ns, s_k_), "spin");
        cuda_check(launch_adam_fused(a, s_k_), "adam_fused");
        for (cudaEvent_t ev : {e.k_end, e.d2h_start, e.d2h_end})
            cuda_check(cudaEventRecord(ev, s_k_), "cudaEventRecord");
        auto* ctx = new std::pair<OffloadWorker*, Completion>(this, Completion{id, slot});
        cuda_check(cudaLaunchHostFunc(s_k_, &OffloadWorker::host_done, ctx), "cudaLaunchHostFunc");
        return {(opt_.skip_gradients ? 12 : 16) * pc, 12 * pc};
    }
    // HBM retention: a subgroup whose state stayed in HBM since the last phase
    // skips the H2D; one the plan retains now skips the D2H and keeps (or
    // takes) a retention buffer. Without a free buffer it takes the host path.
    const int held = hbm_slot_[k];
    int hslot = held;
    bool keep_in_hbm = false;
    if (!hbm_cache_.empty()) {
        std::unique_lock<std::mutex> l(mu_);
        const bool retain = dests_->assign_storage_tier(id).host_retain;
        if (hbm_cache_mode()) {
            // HBM cache: a newly retained subgroup within this phase's budget
            // waits for the buffer a deferred write-back is returning; beyond
            // the budget (two-level cache) it is retained in its host slot.
            const bool take = retain && hslot < 0 && hbm_budget_ > 0;
            while (take && hbm_free_.empty() && wb_inflight_ > 0) {
                if (completion_error_) std::rethrow_exception(completion_error_);
                wb_cv_.wait_for(l, std::chrono::milliseconds(50));
            }
            if (take && !hbm_free_.empty()) {
                hslot = hbm_free_.front();
                hbm_free_.pop_front();
                --hbm_budget_;
            }
        } else if (retain && hslot < 0 && !hbm_free_.empty()) {
            // FIFO: the buffer whose write-back was queued first drains first
            hslot = hbm_free_.front();
            hbm_free_.pop_front();
        }
        keep_in_hbm = retain && hslot >= 0;
    }
    // Ring buffers go round-robin to the subgroups that stream through the
    // ring (HBM-resident ones do not), each reused once the D2H of its last
    // user has drained it (ring_ready_; a never-recorded event does not wait).
    std::size_t rb = 0;
    if (hslot < 0) {
        rb = ring_next_++ % K;
        cuda_check(cudaStreamWaitEvent(s_h2d_, ring_ready_[rb], 0), "wait");
    }
    float* d = hslot >= 0 ? hbm_cache_[static_cast<std::size_t>(hslot)] : ring_[rb];
    const std::uint64_t ds = seg_stride(pc);
    // A retention buffer taken now: its previous occupant's write-back D2H
    // must have drained. Waited before h2d_start is recorded, so every copy
    // ordered after h2d_start (the second H2D half included) is after it.
    if (held < 0 && hslot >= 0)
        cuda_check(cudaStreamWaitEvent(s_h2d_, hbm_ready_[static_cast<std::size_t>(hslot)], 0), "wait");
    cuda_check(cudaEventRecord(e.h2d_start, s_h2d_), "cudaEventRecord");
    std::uint64_t h2d_bytes = 0, d2h_bytes = 0;
    if (held < 0) {
        if (dev_.h2d_split > 1 && ds == pc) {
            // Two concurrent halves on two copy engines: the H2D side of the
            // duplex link arbitration gets a second queue, like d2h_split.
            const StateSpan x = state_span(d, blk, pc);
            const std::size_t bytes = x.bytes;
            const std::size_t half = (bytes / 2) & ~static_cast<std::size_t>(4095);
            const char* host = x.host;
            char* dev = x.dev;
            cuda_check(cudaStreamWaitEvent(s_h2d2_, e.h2d_start, 0), "wait");
            cuda_check(cudaMemcpyAsync(dev, host, half, cudaMemcpyHostToDevice, s_h2d_), "cudaMemcpyAsync");
            cuda_check(cudaMemcpyAsync(dev + half, host + half, bytes - half, cudaMemcpyHostToDevice, s_h2d2_),
                       "cudaMemcpyAsync");
            cuda_check(cudaEventRecord(e.h2d_half, s_h2d2_), "cudaEventRecord");
            cuda_check(cudaStreamWaitEvent(s_h2d_, e.h2d_half, 0), "wait");
        } else {
            copy_state(d, blk, pc, true, s_h2d_);
        }
        h2d_bytes += 12 * pc;
    }
    if (!opt_.skip_gradients) {  // baseline flow: fp32 gradients fetched with the state
        float* dg = ring_grad_[rb];
        cuda_check(cudaMemcpyAsync(dg, grad_annex(blk), 4 * pc, cudaMemcpyHostToDevice, s_h2d_),
                   "cudaMemcpyAsync(grads)");
        h2d_bytes += 4 * pc;
        a.g = dg;
        a.grad_kind = kF32;
    }
    std::size_t xb = 0;  // host_grads: the staging buffer of this update
    if (dev_.host_grads) {
        // The 16-bit gradient comes over with the state; the working params
        // go back after the kernel (below), through one staging buffer.
        xb = aux_next_++ % aux_.size();
        cuda_check(cudaStreamWaitEvent(s_h2d_, aux_ready_[xb], 0), "wait");
        cuda_check(cudaMemcpyAsync(aux_[xb], grad_ptr_[k], 2 * pc, cudaMemcpyHostToDevice, s_h2d_),
                   "cudaMemcpyAsync(grads16)");
        h2d_bytes += 2 * pc;
        a.g = aux_[xb];
        a.p16 = aux_[xb] + ring_stride_;
    }
    cuda_check(cudaEventRecord(e.h2d_done, s_h2d_), "cudaEventRecord");

    cuda_check(cudaStreamWaitEvent(s_k_, e.h2d_done, 0), "wait");
    cuda_check(cudaEventRecord(e.k_start, s_k_), "cudaEventRecord");
    cuda_check(launch_spin_ns(opt_.update_pad_ns, s_k_), "spin");
    a.p = d;
    a.m = d + ds;
    a.v = d + 2 * ds;
    if (dev_.zero_copy == 2) {
        // DMA brings the state in; the kernel's epilogue stores the updated
        // P, m, v straight into the mapped pinned slot (the D2H fused into
        // the kernel), so no copy engine serves the write-back.
        float* hp = nullptr;
        cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hp), blk.payload(), 0),
                   "cudaHostGetDevicePointer");
        a.p_out = hp;
        a.m_out = hp + pc;
        a.v_out = hp + 2 * pc;
        cuda_check(launch_adam_fused(a, s_k_), "adam_fused");
        for (cudaEvent_t ev : {e.k_end, e.d2h_start, e.d2h_end})
            cuda_check(cudaEventRecord(ev, s_k_), "cudaEventRecord");
        // The ring buffer (and, in the baseline flow, its fp32 gradient
        // segment) is free once this kernel has read it: the next H2D into
        // it waits here (there is no D2H to carry the event).
        if (hslot < 0) cuda_check(cudaEventRecord(ring_ready_[rb], s_k_), "cudaEventRecord");
        auto* ctx = new std::pair<OffloadWorker*, Completion>(this, Completion{id, slot});
        cuda_check(cudaLaunchHostFunc(s_k_, &OffloadWorker::host_done, ctx), "cudaLaunchHostFunc");
        return {h2d_bytes, 12 * pc};
    }
    cuda_check(launch_adam_fused(a, s_k_), "adam_fused");
    cuda_check(cudaEventRecord(e.k_end, s_k_), "cudaEventRecord");
    if (dev_.host_grads) {  // working params to their host block; the staging buffer is free after
        cuda_check(cudaStreamWaitEvent(s_d2h_, e.k_end, 0), "wait");
        cuda_check(cudaMemcpyAsync(p16_ptr_[k], aux_[xb] + ring_stride_, 2 * pc, cudaMemcpyDeviceToHost, s_d2h_),
                   "cudaMemcpyAsync(params16)");
        cuda_check(cudaEventRecord(aux_ready_[xb], s_d2h_), "cudaEventRecord");
        d2h_bytes += 2 * pc;
    }

    if (slot < 0 && held >= 0 && !keep_in_hbm) {  // HBM cache mode: the write-back thread takes it
        {
            std::lock_guard<std::mutex> g(mu_);
            wb_pending_.push_back(PendingWriteback{id, k, held, pc});
            ++wb_inflight_;
        }
        wb_cv_.notify_all();
        return {h2d_bytes, d2h_bytes + 12 * pc};
    }
    cuda_check(cudaStreamWaitEvent(s_d2h_, e.k_end, 0), "wait");
    cuda_check(cudaEventRecord(e.d2h_start, s_d2h_), "cudaEventRecord");
    if (keep_in_hbm) {
        // no write-back: the host slot copy is stale until the next update
    } else if (dev_.d2h_split > 1 && ds == pc) {
        // Two concurrent D2H halves on two copy engines: the write-back gets
        // a larger share of the duplex link against the H2D stream.
        const StateSpan x = state_span(d, blk, pc);
        const std::size_t bytes = x.bytes;
        const std::size_t half = (bytes / 2) & ~static_cast<std::size_t>(4095);
        char* host = x.host;
        char* dev = x.dev;
        cuda_check(cudaStreamWaitEvent(s_d2h2_, e.d2h_start, 0), "wait");
        cuda_check(cudaMemcpyAsync(host, dev, half, cudaMemcpyDeviceToHost, s_d2h_), "cudaMemcpyAsync");
        cuda_check(cudaMemcpyAsync(host + half, dev + half, bytes - half, cudaMemcpyDeviceToHost, s_d2h2_),
                   "cudaMemcpyAsync");
        cuda_check(cudaEventRecord(e.d2h_half, s_d2h2_), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(s_d2h_, e.d2h_half, 0), "wait");
    } else {
        copy_state(d, blk, pc, false, s_d2h_);
    }
    if (!keep_in_hbm) d2h_bytes += 12 * pc;
    cuda_check(cudaEventRecord(e.d2h_end, s_d2h_), "cudaEventRecord");
    if (hslot < 0) cuda_check(cudaEventRecord(ring_ready_[rb], s_d2h_), "cudaEventRecord");
    if (hslot >= 0) {
        std::lock_guard<std::mutex> g(mu_);
        if (keep_in_hbm) {
            hbm_slot_[k] = hslot;
        } else {  // written back: the buffer is free once this D2H drains
            cuda_check(cudaEventRecord(hbm_ready_[static_cast<std::size_t>(hslot)], s_d2h_), "cudaEventRecord");
            hbm_free_.push_back(hslot);
            hbm_slot_[k] = -1;
        }
    }
    auto* ctx = new std::pair<OffloadWorker*, Completion>(this, Completion{id, slot});
    cuda_check(cudaLaunchHostFunc(s_d2h_, &OffloadWorker::host_done, ctx), "cudaLaunchHostFunc");
    return {h2d_bytes, d2h_bytes};
}

// Synchronous D2H of a P/m/v buffer (segment stride seg_stride(pc)) into a
// contiguous host P||m||v. Only called with the pipeline drained.
void OffloadWorker::device_state_to_host(const float* dev, float* host, std::uint64_t pc) {
    DeviceGuard dg(dev_.device);
    const std::uint64_t ds = seg_stride(pc);
    for (int s = 0; s < 3; ++s)
        cuda_check(cudaMemcpy(host + s * pc, dev + s * ds, 4 * pc, cudaMemcpyDeviceToHost), "cudaMemcpy(state)");
}

// Refreshes the host slot of an HBM-retained subgroup and frees its buffer
// (op-level flush outside a phase). Called with mu_ held.
void OffloadWorker::writeback_hbm_copy_locked(std::size_t k, int slot) {
    const int b = hbm_slot_[k];
    if (b < 0) return;
    device_state_to_host(hbm_cache_[static_cast<std::size_t>(b)], pool_->block(slot).payload(),
                         subgroups_.at(ids_[k]).param_count);
    hbm_slot_[k] = -1;
    hbm_free_.push_back(b);
}

void CUDART_CB OffloadWorker::host_done(void* arg) {
    auto* ctx = static_cast<std::pair<OffloadWorker*, Completion>*>(arg);
    OffloadWorker* w = ctx->first;
    {
        std::lock_guard<std::mutex> g(w->cq_mu_);
        w->cq_.push_back(ctx->second);
    }
    w->cq_cv_.notify_one();
    delete ctx;
}

void OffloadWorker::completion_loop() {
    cudaSetDevice(dev_.device);
    for (;;) {
        Completion c;
        {
            std::unique_lock<std::mutex> l(cq_mu_);
            cq_cv_.wait(l, [&] { return cq_stop_ || !cq_.empty(); });
            if (cq_.empty()) return;
            c = cq_.front();
            cq_.pop_front();
        }
        std::lock_guard<std::mutex> g(mu_);
        try {
            Subgroup& sg = subgroups_.at(c.id);
            const std::size_t k = index_of_.at(c.id);
            host_retired_ns_[k] = now_ns();
            if (c.slot >= 0) pool_->end_update(c.slot);
            trace_->record(EventKind::update_end, id_, c.id, kNoTier, 12 * sg.param_count);
            const TierAssignment a = dests_->assign_storage_tier(c.id);
            if (!a.host_retain) {
                start_flush_locked(c.id, a.tier, c.slot, c.wb);
            } else if (hbm_cache_mode() && hbm_slot_[k] >= 0 && c.slot >= 0) {
                pool_->evict(c.slot);  // the state lives in HBM: the slot streams again
                sg.slot = -1;
            }
            pump_locked();
        } catch (...) {
            if (!completion_error_) completion_error_ = std::current_exception();
        }
        --in_flight_;
        inflight_cv_.notify_all();
    }
}

// Where subgroup `id` stands on its way into a host slot (mu_ held). A
// subgroup already fetching this phase is `pending`; one host-resident with no
// fetch this phase is a cache hit (reference scheduler.hpp:528-533), traced
// and counted here; one on a tier takes a free slot and its fetch is issued,
// else it is `blocked` until a slot frees. A state held in the write-back lane
// after a failed flush first moves into a slot (blocked while none is free).
OffloadWorker::HostClaim OffloadWorker::claim_host_locked(SubgroupId id) {
    if (const auto f = prefetch_futures_.find(id); f != prefetch_futures_.end())
        return {HostClaim::pending, f->second};
    Subgroup& sg = subgroups_.at(id);
    if (sg.residency != Residency::host_cached) {
        const int slot = pool_->try_reserve(id);
        if (slot < 0) return {HostClaim::blocked, {}};
        return {HostClaim::pending, start_prefetch_locked(id, slot)};
    }
    if (sg.slot < 0 && wb_held_.count(id) != 0 && adopt_wb_held_locked(id) < 0) return {HostClaim::blocked, {}};
    ++cache_hits_this_phase_;
    trace_->record(EventKind::cache_hit, id_, id, kNoTier, 0);
    return {HostClaim::hit, {}};
}

OffloadWorker::HostClaim OffloadWorker::claim_host(SubgroupId id) {
    std::unique_lock<std::mutex> l(mu_);
    HostClaim c = claim_host_locked(id);
    while (c.kind == HostClaim::blocked) {
        l.unlock();
        wait_pool_free();
        l.lock();
        c = claim_host_locked(id);
    }
    return c;
}

int OffloadWorker::wait_host_resident(SubgroupId id) {
    HostClaim c = claim_host(id);
    if (c.kind == HostClaim::pending) {
        watchdog_wait_value(c.fetch);
    } else if (!opt_.skip_gradients) {
        // Baseline flow: a cached subgroup still needs its fp32 gradients.
        bool stored;
        {
            std::lock_guard<std::mutex> g(mu_);
            stored = grad_tier_.count(id) != 0;
        }
        if (stored) fetch_grads_for_cached(id);
    }
    std::lock_guard<std::mutex> g(mu_);
    return subgroups_.at(id).slot;
}

std::shared_future<IoStats> OffloadWorker::enqueue_flush(SubgroupId id, TierId dest) {
    std::lock_guard<std::mutex> g(mu_);
    Subgroup& sg = subgroups_.at(id);
    if (sg.residency != Residency::host_cached) throw Error("enqueue_flush: subgroup not host-resident");
    if (sg.slot < 0 && wb_held_.count(id) != 0 && adopt_wb_held_locked(id) < 0)
        throw Error("enqueue_flush: no host slot free for subgroup " + std::to_string(id));
    if (sg.slot < 0 && !(hbm_cache_mode() && hbm_slot_[index_of_.at(id)] >= 0 && reserve_writeback_slot_locked(id) >= 0))
        throw Error("enqueue_flush: no host slot free for the write-back of subgroup " + std::to_string(id));
    if (!hbm_slot_.empty()) writeback_hbm_copy_locked(index_of_.at(id), sg.slot);
    return start_flush_locked(id, dest, sg.slot);
}

std::optional<std::shared_future<IoStats>> OffloadWorker::enqueue_prefetch(SubgroupId id) {
    HostClaim c = claim_host(id);
    if (c.kind == HostClaim::hit) return std::nullopt;
    return c.fetch;
}

void OffloadWorker::read_current_state(SubgroupId id, float* out) {
    TierId tier;
    std::uint64_t pc;
    {
        std::lock_guard<std::mutex> g(mu_);
        const Subgroup& sg = subgroups_.at(id);
        pc = sg.param_count;
        if (sg.residency == Residency::host_cached) {
            const int b = hbm_slot_.empty() ? -1 : hbm_slot_[index_of_.at(id)];
            const auto held = wb_held_.find(id);
            if (b >= 0)
                device_state_to_host(hbm_cache_[static_cast<std::size_t>(b)], out, pc);
            else if (sg.slot < 0 && held != wb_held_.end())
                std::memcpy(out, wb_blocks_[static_cast<std::size_t>(held->second)].payload(), 12 * pc);
            else
                std::memcpy(out, pool_->block(sg.slot).payload(), 12 * pc);
            return;
        }
        if (sg.residency != Residency::on_tier) throw Error("read_current_state: subgroup is in flight");
        tier = sg.tier;
    }
    tiers_[static_cast<std::size_t>(tier)]->read_subgroup(id, pc, out);
}

Subgroup OffloadWorker::meta(SubgroupId id) {
    std::lock_guard<std::mutex> g(mu_);
    return subgroups_.at(id);
}

std::uint64_t OffloadWorker::total_params() const {
    std::uint64_t n = 0;
    for (const auto& [id, sg] : subgroups_) n += sg.param_count;
    return n;
}

// Params per residency: host-resident (slot, HBM or write-back lane) and per
// tier; in-flight subgroups are in neither (reference scheduler.hpp:597).
std::pair<std::uint64_t, std::vector<std::uint64_t>> OffloadWorker::residency_census() {
    std::lock_guard<std::mutex> g(mu_);
    std::pair<std::uint64_t, std::vector<std::uint64_t>> census{0, std::vector<std::uint64_t>(tiers_.size(), 0)};
    for (const SubgroupId id : ids_) {
        const Subgroup& sg = subgroups_.at(id);
        std::uint64_t* bin = sg.residency == Residency::host_cached ? &census.first
                             : sg.residency == Residency::on_tier  ? &census.second.at(static_cast<std::size_t>(sg.tier))
                                                                    : nullptr;
        if (bin) *bin += sg.param_count;
    }
    return census;
}

std::vector<SubgroupId> OffloadWorker::current_order() {
    std::lock_guard<std::mutex> g(mu_);
    return order_;
}

// Advances the prefetch frontier through the plan while slots are free
// (reference scheduler.hpp:645-659). Subgroups already host-resident or
// already fetching are passed over; a state held in the write-back lane after
// a failed flush is adopted into a slot at its place in the plan. Called with
// mu_ held.
void OffloadWorker::pump_locked() {
    for (; frontier_ < order_.size(); ++frontier_) {
        const SubgroupId id = order_[frontier_];
        const Subgroup& sg = subgroups_.at(id);
        if (sg.residency == Residency::host_cached) {
            if (sg.slot < 0 && wb_held_.count(id) != 0 && adopt_wb_held_locked(id) < 0) return;
            continue;
        }
        if (sg.residency != Residency::on_tier || prefetch_futures_.count(id) != 0) continue;
        // Already updated this phase and flushed again (a hit the plan does
        // not retain, issued while the frontier was still behind it): it is
        // not fetched a second time. The reference's pump would re-fetch it
        // and hold a slot into the next phase, where it counts as a hit; that
        // only arises when C shrinks or the hits sit at the end of the order.
        if (!updated_this_phase_.empty() && updated_this_phase_[index_of_.at(id)]) continue;
        const int slot = pool_->try_reserve(id);
        if (slot < 0) return;  // resumes here when a slot frees
        start_prefetch_locked(id, slot);
    }
}

std::shared_future<IoStats> OffloadWorker::start_prefetch_locked(SubgroupId id, int slot) {
    Subgroup& sg = subgroups_.at(id);
    const TierId origin = sg.tier;
    sg.begin_prefetch();
    const std::uint64_t pc = sg.param_count;
    auto tier = tiers_[static_cast<std::size_t>(origin)];
    HostBufferPool* pool = pool_.get();
    // Baseline flow: the fp32 gradients stored with the state come along
    // (16 bytes/param; reference scheduler.hpp:667-680).
    const bool fetch_grads = !opt_.skip_gradients && grad_tier_.count(id) != 0 && grad_tier_.at(id) == origin;
    const std::size_t annex_off = state_block_bytes_;
    auto transfer = [tier, id, pc, pool, slot, fetch_grads, annex_off] {
        IoStats st = tier->read_into(id, pc, pool->block(slot));
        if (fetch_grads) {
            float* dst = reinterpret_cast<float*>(pool->block(slot).base() + annex_off);
            const IoStats gs = tier->read_grads(id, pc, dst);
            st.bytes += gs.bytes;
            st.seconds += gs.seconds;
        }
        return st;
    };
    auto completion = [this, id, slot, origin](bool ok, const IoStats& st) {
        std::lock_guard<std::mutex> g(mu_);
        Subgroup& s = subgroups_.at(id);
        if (ok) {
            s.finish_prefetch(slot);
            pool_->prefetch_done(slot);
            account_io_locked(id, origin, st, IoDir::read, /*state_fetch=*/true);
        } else {
            s.residency = Residency::on_tier;  // fetch failed: still on its tier
            s.slot = -1;
            pool_->release_failed(slot);
        }
        resident_cv_.notify_all();
    };
    auto fut = io_[static_cast<std::size_t>(origin)]
                   ->submit(true, id, 12 * pc + (fetch_grads ? 4 * pc : 0), std::move(transfer), std::move(completion))
                   .share();
    prefetch_futures_[id] = fut;
    return fut;
}

std::shared_future<IoStats> OffloadWorker::start_flush_locked(SubgroupId id, TierId dest, int slot, int wb) {
    if (dest < 0 || static_cast<std::size_t>(dest) >= tiers_.size()) throw Error("flush destination out of range");
    Subgroup& sg = subgroups_.at(id);
    const TierId origin = sg.tier;  // differs from dest when the allocation shifted
    sg.begin_flush();
    if (wb < 0) pool_->begin_flush(slot);
    const std::uint64_t pc = sg.param_count;
    auto tier = tiers_[static_cast<std::size_t>(dest)];
    HostBlock* src = wb >= 0 ? &wb_blocks_[static_cast<std::size_t>(wb)] : &pool_->block(slot);
    // The pool slot's block may be exchanged with a host_dram tier's blob by
    // write_from; a write-back block likewise (both are owned by the lane /
    // pool object, not by the pointer's referent).
    auto transfer = [tier, id, pc, src] { return tier->write_from(id, pc, *src); };
    auto completion = [this, id, slot, wb, dest, origin](bool ok, const IoStats& st) {
        std::shared_ptr<Tier> stale;
        {
            std::lock_guard<std::mutex> g(mu_);
            Subgroup& s = subgroups_.at(id);
            if (ok) {
                s.finish_flush(dest);
                if (wb >= 0) {
                    wb_free_.push_back(wb);
                    wb_cv_.notify_all();
                } else {
                    pool_->flush_done(slot);
                }
                account_io_locked(id, dest, st, IoDir::write, false);
                if (origin >= 0 && origin != dest) stale = tiers_[static_cast<std::size_t>(origin)];
                pump_locked();
            } else if (wb < 0) {
                s.residency = Residency::host_cached;  // flush failed: the state stays in its slot
                pool_->flush_failed(slot);
            } else {
                // Write-back failed: the state is only in the write-back block.
                // The subgroup stays host-cached there until a pool slot adopts
                // it (now if one is free, else in plan order by pump_locked).
                s.residency = Residency::host_cached;
                wb_held_[id] = wb;
                adopt_wb_held_locked(id);
            }
        }
        if (stale) stale->remove_subgroup(id);
    };
    auto fut = io_[static_cast<std::size_t>(dest)]
                   ->submit(false, id, 12 * pc, std::move(transfer), std::move(completion))
                   .share();
    flush_futures_.emplace_back(id, fut);
    return fut;
}

// Moves a failed write-back's block into a free pool slot (block exchange).
// Called with mu_ held; the slot, or -1 if none is free.
int OffloadWorker::adopt_wb_held_locked(SubgroupId id) {
    const auto it = wb_held_.find(id);
    if (it == wb_held_.end()) return subgroups_.at(id).slot;
    const int ps = pool_->try_reserve(id);
    if (ps < 0) return -1;
    std::swap(pool_->block(ps), wb_blocks_[static_cast<std::size_t>(it->second)]);
    pool_->prefetch_done(ps);
    subgroups_.at(id).slot = ps;
    wb_free_.push_back(it->second);
    wb_held_.erase(it);
    wb_cv_.notify_all();
    return ps;
}

// HBM cache mode write-back thread: pairs each deferred hit (kernel issued,
// state updated in its HBM buffer) with a free write-back block, issues the
// D2H on its own stream, frees the HBM buffer behind it, and hands the
// subgroup to the completion thread, which flushes it from the block.
void OffloadWorker::writeback_loop() {
    cudaSetDevice(dev_.device);
    for (;;) {
        PendingWriteback p{};
        int wb = -1;
        {
            std::unique_lock<std::mutex> l(mu_);
            wb_cv_.wait(l, [&] { return wb_stop_ || (!wb_pending_.empty() && !wb_free_.empty()); });
            if (wb_stop_) return;
            p = wb_pending_.front();
            wb_pending_.pop_front();
            wb = wb_free_.front();
            wb_free_.pop_front();
        }
        try {
            const DeviceEvents& e = events_[p.k];
            const std::uint64_t pc = p.pc;
            cuda_check(cudaStreamWaitEvent(s_d2h2_, e.k_end, 0), "wait");
            cuda_check(cudaEventRecord(e.d2h_start, s_d2h2_), "cudaEventRecord");
            copy_state(hbm_cache_[static_cast<std::size_t>(p.hslot)], wb_blocks_[static_cast<std::size_t>(wb)], pc,
                       false, s_d2h2_);
            cuda_check(cudaEventRecord(e.d2h_end, s_d2h2_), "cudaEventRecord");
            cuda_check(cudaEventRecord(hbm_ready_[static_cast<std::size_t>(p.hslot)], s_d2h2_), "cudaEventRecord");
            {
                std::lock_guard<std::mutex> g(mu_);
                hbm_free_.push_back(p.hslot);
                hbm_slot_[p.k] = -1;
                --wb_inflight_;
            }
            wb_cv_.notify_all();
            auto* ctx = new std::pair<OffloadWorker*, Completion>(this, Completion{p.id, -1, wb});
            cuda_check(cudaLaunchHostFunc(s_d2h2_, &OffloadWorker::host_done, ctx), "cudaLaunchHostFunc");
        } catch (...) {
            std::lock_guard<std::mutex> g(mu_);
            if (!completion_error_) completion_error_ = std::current_exception();
            --wb_inflight_;
            --in_flight_;
            inflight_cv_.notify_all();
            wb_cv_.notify_all();
        }
    }
}

// One finished transfer into this phase's observations: the tier's totals
// (the EMA input, reference scheduler.hpp:767-797) and the subgroup's own
// read/write times (the effective-I/O metric). Outside a phase (op-level
// calls) nothing is recorded. Called with mu_ held.
void OffloadWorker::account_io_locked(SubgroupId id, TierId tier, const IoStats& st, IoDir dir, bool state_fetch) {
    if (phase_stats_ == nullptr) return;
    TierObservation& obs = phase_stats_->tier_obs.at(static_cast<std::size_t>(tier));
    auto [slot, fresh] = io_index_.try_emplace(id, phase_stats_->subgroup_io.size());
    if (fresh) {
        SubgroupIoTimes e;
        e.id = id;
        e.state_bytes = 12 * subgroups_.at(id).param_count;
        phase_stats_->subgroup_io.push_back(e);
    }
    SubgroupIoTimes& io = phase_stats_->subgroup_io[slot->second];
    const double bytes = static_cast<double>(st.bytes);
    if (dir == IoDir::read) {
        obs.read_transfers += 1;
        obs.read_bytes += bytes;
        obs.read_seconds += st.seconds;
        io.read_seconds += st.seconds;
        io.fetched = io.fetched || state_fetch;
    } else {
        obs.write_transfers += 1;
        obs.write_bytes += bytes;
        obs.write_seconds += st.seconds;
        io.write_seconds += st.seconds;
        io.flushed = true;
    }
}

void OffloadWorker::wait_pool_free() {
    const std::uint64_t start = trace_->progress_count();
    double waited = 0.0;
    while (!pool_->wait_for_free(std::chrono::milliseconds(50))) {
        waited += 0.05;
        if (trace_->progress_count() != start) return;  // progress elsewhere: re-examine
        if (waited >= opt_.deadlock_timeout_s)
            throw SchedulingBugError("host buffer pool made no progress (all slots busy) for " +
                                     std::to_string(opt_.deadlock_timeout_s) + "s");
    }
}

IoStats OffloadWorker::watchdog_wait_value(std::shared_future<IoStats>& fut) {
    std::uint64_t last = trace_->progress_count();
    double stalled = 0.0;
    while (fut.wait_for(std::chrono::milliseconds(50)) != std::future_status::ready) {
        const std::uint64_t p = trace_->progress_count();
        if (p != last) {
            last = p;
            stalled = 0.0;
        } else if ((stalled += 0.05) >= opt_.deadlock_timeout_s) {
            throw SchedulingBugError("pipeline made no trace progress for " + std::to_string(opt_.deadlock_timeout_s) +
                                     "s");
        }
    }
    return fut.get();
}

}  // namespace tfb
