// extern "C" boundary (include/tierflow_b200.h). Exceptions stop here and
// become tfg_status codes; the message is kept per thread for tfg_last_error.
#include "../../include/tierflow_b200.h"

#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "capi_internal.hpp"
#include "pacer.hpp"
#include "engine.hpp"
#include "kernels.hpp"
#include "placement.hpp"
#include "tier.hpp"
#include "tier_lock.hpp"
#include "trace.hpp"

struct tfg_tier {
    std::shared_ptr<tfb::Tier> t;
};
struct tfg_trace {
    std::shared_ptr<tfb::EventTrace> t;
};
struct tfg_engine {
    std::unique_ptr<tfb::OffloadWorker> w;
    std::vector<tfb::SubgroupIoTimes> last_io;
    std::vector<tfb::DeviceSpan> last_timeline;
    std::mutex mu;
    std::map<std::uint64_t, std::shared_future<tfb::IoStats>> tickets;
    std::uint64_t next_ticket = 1;
};

namespace {

thread_local std::string g_last_error;

}  // namespace

void tfb::set_last_error(const std::string& msg) { g_last_error = msg; }

namespace {

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return TFG_OK;
    } catch (const tfb::Error& e) {
        g_last_error = e.what();
        return e.code();
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return TFG_ERROR;
    } catch (...) {
        g_last_error = "unknown exception";
        return TFG_ERROR;
    }
}

void need(const void* p, const char* what) {
    if (p == nullptr) throw tfb::ConfigError(std::string(what) + " must not be NULL");
}

void check_dtype(int d) {
    if (d != TFG_F16 && d != TFG_BF16) throw tfb::ConfigError("unknown 16-bit dtype " + std::to_string(d));
}

void check_grad_dtype(int d) {
    if (d != TFG_F16 && d != TFG_BF16 && d != TFG_F32) throw tfb::ConfigError("unknown gradient dtype " + std::to_string(d));
}

tfb::AdamHyper to_hyper(const tfg_adam_hyper* h) {
    need(h, "hyper");
    tfb::AdamHyper a;
    a.lr = h->lr;
    a.beta1 = h->beta1;
    a.beta2 = h->beta2;
    a.eps = h->eps;
    a.weight_decay = h->weight_decay;
    return a;
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

tfb::AdamLaunch adam_launch(float* p, float* m, float* v, const void* g, int gk, uint16_t* p16, int ok,
                            uint64_t n, const tfg_adam_hyper* hyper, uint64_t t, unsigned long long* counters) {
    check_grad_dtype(gk);
    check_dtype(ok);
    if (n > 0) {
        need(p, "p");
        need(m, "m");
        need(v, "v");
        need(g, "grad");
        need(p16, "param16");
    }
    tfb::AdamLaunch a;
    a.p = p;
    a.m = m;
    a.v = v;
    a.g = g;
    a.p16 = p16;
    a.n = n;
    a.grad_kind = gk;
    a.out_kind = ok;
    a.c = to_hyper(hyper).consts(t);
    a.counters = counters;
    return a;
}

}  // namespace

extern "C" {

const char* tfg_last_error(void) { return g_last_error.c_str(); }

int tfg_abi_version(void) { return TFG_ABI_VERSION; }

int tfg_device_count(int* count) {
    return guarded([&] {
        need(count, "count");
        int n = 0;
        const cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            n = 0;
        }
        *count = n;
    });
}

// ---- peer memory ---------------------------------------------------------------

namespace {
struct DeviceScope {
    int prev = 0;
    explicit DeviceScope(int d) {
        tfb::cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
        tfb::cuda_check(cudaSetDevice(d), "cudaSetDevice");
    }
    ~DeviceScope() { cudaSetDevice(prev); }
};
static_assert(sizeof(cudaIpcMemHandle_t) == TFG_IPC_HANDLE_BYTES, "IPC handle size");
}  // namespace

int tfg_device_alloc(int device, uint64_t bytes, void** out) {
    return guarded([&] {
        need(out, "out");
        if (bytes == 0) throw tfb::ConfigError("device_alloc: zero bytes");
        DeviceScope ds(device);
        tfb::cuda_check(cudaMalloc(out, bytes), "cudaMalloc");
    });
}

int tfg_device_free(int device, void* ptr) {
    return guarded([&] {
        DeviceScope ds(device);
        tfb::cuda_check(cudaFree(ptr), "cudaFree");
    });
}

int tfg_ipc_get_handle(int device, void* ptr, unsigned char* handle_out) {
    return guarded([&] {
        need(ptr, "ptr");
        need(handle_out, "handle_out");
        DeviceScope ds(device);
        cudaIpcMemHandle_t h;
        tfb::cuda_check(cudaIpcGetMemHandle(&h, ptr), "cudaIpcGetMemHandle");
        std::memcpy(handle_out, &h, sizeof(h));
    });
}

int tfg_ipc_open_handle(int device, const unsigned char* handle, void** out) {
    return guarded([&] {
        need(handle, "handle");
        need(out, "out");
        DeviceScope ds(device);
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof(h));
        tfb::cuda_check(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    });
}

int tfg_ipc_close_handle(int device, void* ptr) {
    return guarded([&] {
        need(ptr, "ptr");
        DeviceScope ds(device);
        tfb::cuda_check(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle");
    });
}

// ---- kernels -------------------------------------------------------------------

int tfg_adam_fused(float* p, float* m, float* v, const void* grad, int grad_dtype, uint16_t* param16,
                   int param_dtype, uint64_t n, const tfg_adam_hyper* hyper, uint64_t t,
                   unsigned long long* counters, void* stream) {
    return guarded([&] {
        const auto a = adam_launch(p, m, v, grad, grad_dtype, param16, param_dtype, n, hyper, t, counters);
        tfb::cuda_check(tfb::launch_adam_fused(a, as_stream(stream)), "adam_fused");
    });
}

int tfg_adam_fused_gated(float* p, float* m, float* v, const void* grad, int grad_dtype, uint16_t* param16,
                         int param_dtype, uint64_t n, const tfg_adam_hyper* hyper, uint64_t t,
                         unsigned long long* counters, const unsigned long long* gate, void* stream) {
    return guarded([&] {
        auto a = adam_launch(p, m, v, grad, grad_dtype, param16, param_dtype, n, hyper, t, counters);
        a.gate = gate;
        tfb::cuda_check(tfb::launch_adam_fused(a, as_stream(stream)), "adam_fused_gated");
    });
}

int tfg_adam_fused_multi(float* p, float* m, float* v, const void* const* grads, int n_sources, int grad_dtype,
                         uint16_t* param16, int param_dtype, uint64_t n, const tfg_adam_hyper* hyper, uint64_t t,
                         unsigned long long* counters, void* stream) {
    return guarded([&] {
        check_dtype(grad_dtype);
        if (n_sources < 1 || n_sources > tfb::kMaxGradSources)
            throw tfb::ConfigError("n_sources must be in [1, " + std::to_string(tfb::kMaxGradSources) + "]");
        need(grads, "grads");
        for (int s = 0; s < n_sources; ++s) need(grads[s], "grads[s]");
        auto a = adam_launch(p, m, v, grads[0], grad_dtype, param16, param_dtype, n, hyper, t, counters);
        for (int s = 0; s < n_sources; ++s) a.peers[s] = grads[s];
        a.n_peers = n_sources;
        tfb::cuda_check(tfb::launch_adam_fused(a, as_stream(stream)), "adam_fused_multi");
    });
}

int tfg_adam_fused_contiguous(float* state, uint64_t n, const void* grad, int grad_dtype, uint16_t* param16,
                              int param_dtype, const tfg_adam_hyper* hyper, uint64_t t,
                              unsigned long long* counters, void* stream) {
    return guarded([&] {
        if (n > 0) need(state, "state");
        const auto a = adam_launch(state, state + n, state + 2 * n, grad, grad_dtype, param16, param_dtype, n, hyper,
                                   t, counters);
        tfb::cuda_check(tfb::launch_adam_fused(a, as_stream(stream)), "adam_fused");
    });
}

int tfg_adam_step(float* p, float* m, float* v, const uint16_t* grad, int grad_dtype, uint16_t* param16,
                  int param_dtype, uint64_t n, const tfg_adam_hyper* hyper, uint64_t t, uint64_t* overflows_out,
                  void* stream) {
    return guarded([&] {
        check_dtype(grad_dtype);  // the pre-check counts 16-bit patterns
        auto a = adam_launch(p, m, v, grad, grad_dtype, param16, param_dtype, n, hyper, t, nullptr);
        cudaStream_t s = as_stream(stream);
        unsigned long long* dc = nullptr;
        tfb::cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&dc), 2 * sizeof(unsigned long long), s),
                        "cudaMallocAsync");
        struct Free {
            unsigned long long* p;
            cudaStream_t s;
            ~Free() { cudaFreeAsync(p, s); }
        } guard{dc, s};
        tfb::cuda_check(cudaMemsetAsync(dc, 0, 2 * sizeof(unsigned long long), s), "cudaMemsetAsync");
        tfb::cuda_check(tfb::launch_count_nonfinite16(grad, n, grad_dtype, dc, s), "count_nonfinite");
        unsigned long long h[2] = {0, 0};
        tfb::cuda_check(cudaMemcpyAsync(h, dc, sizeof(h), cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync");
        tfb::cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        if (h[0] != 0) throw tfb::GradientOverflowError("adam_step: non-finite gradients");
        a.counters = dc;
        a.grads_verified = true;  // counted above
        tfb::cuda_check(tfb::launch_adam_fused(a, s), "adam_fused");
        tfb::cuda_check(cudaMemcpyAsync(h, dc, sizeof(h), cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync");
        tfb::cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        if (overflows_out) *overflows_out = h[1];
    });
}

int tfg_selftest_div_const(double divisor, uint64_t n, uint64_t seed, int exp_lo, int exp_span, uint64_t* mismatches,
                           double* first_bad) {
    return guarded([&] {
        if (!(divisor > 0.0)) throw tfb::ConfigError("divisor must be > 0");
        if (exp_span < 1) throw tfb::ConfigError("exp_span must be >= 1");
        unsigned long long* d = nullptr;
        tfb::cuda_check(cudaMalloc(reinterpret_cast<void**>(&d), 16), "cudaMalloc");
        tfb::cuda_check(cudaMemset(d, 0, 16), "cudaMemset");
        const cudaError_t e = tfb::launch_divtest(divisor, 1.0 / divisor, n, seed, exp_lo, exp_span, d,
                                                  reinterpret_cast<double*>(d + 1), nullptr);
        unsigned long long h[2] = {0, 0};
        const cudaError_t e2 = e == cudaSuccess ? cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost) : e;
        cudaFree(d);
        tfb::cuda_check(e2, "divtest");
        if (mismatches) *mismatches = h[0];
        if (first_bad) std::memcpy(first_bad, &h[1], sizeof(double));
    });
}

int tfg_upscale16(const uint16_t* src, float* dst, uint64_t n, int dtype, unsigned long long* nonfinite,
                  void* stream) {
    return guarded([&] {
        check_dtype(dtype);
        tfb::cuda_check(tfb::launch_widen16(src, dst, n, dtype, nonfinite, as_stream(stream)), "upscale16");
    });
}

int tfg_downscale16(const float* src, uint16_t* dst, uint64_t n, int dtype, unsigned long long* overflows,
                    void* stream) {
    return guarded([&] {
        check_dtype(dtype);
        tfb::cuda_check(tfb::launch_narrow16(src, dst, n, dtype, overflows, as_stream(stream)), "downscale16");
    });
}

int tfg_count_nonfinite16(const uint16_t* src, uint64_t n, int dtype, unsigned long long* count, void* stream) {
    return guarded([&] {
        check_dtype(dtype);
        need(count, "count");
        tfb::cuda_check(tfb::launch_count_nonfinite16(src, n, dtype, count, as_stream(stream)), "count_nonfinite16");
    });
}

int tfg_synthetic_grads(uint16_t* out, uint64_t n, int dtype, uint64_t seed, uint32_t subgroup, int iteration,
                        int step, int accumulate, void* stream) {
    return guarded([&] {
        check_dtype(dtype);
        tfb::cuda_check(tfb::launch_synthetic_grads(out, n, dtype, tfb::grad_prefix(seed, subgroup, iteration, step),
                                                    accumulate != 0, as_stream(stream)),
                        "synthetic_grads");
    });
}

int tfg_synthetic_state(float* p, float* m, float* v, uint64_t n, uint64_t seed, uint32_t subgroup, void* stream) {
    return guarded([&] {
        const uint64_t prefix = tfb::param_prefix(seed, subgroup);
        tfb::cuda_check(tfb::launch_synthetic_state(p, m, v, n, prefix, as_stream(stream)), "synthetic_state");
    });
}

// ---- placement -------------------------------------------------------------------

int tfg_host_blocks_live(int64_t* blocks_out, int64_t* bytes_out, int64_t* free_failures_out) {
    return guarded([&] {
        if (blocks_out) *blocks_out = tfb::g_host_blocks_live.load();
        if (bytes_out) *bytes_out = tfb::g_host_bytes_live.load();
        if (free_failures_out) *free_failures_out = tfb::g_host_free_failures.load();
    });
}

int tfg_assign_subgroups(int M, const double* bandwidths, int n_tiers, int* counts_out) {
    return guarded([&] {
        if (n_tiers > 0) {
            need(bandwidths, "bandwidths");
            need(counts_out, "counts_out");
        }
        const std::vector<double> b(bandwidths, bandwidths + std::max(n_tiers, 0));
        const auto a = tfb::assign_subgroups(M, b);
        for (int i = 0; i < n_tiers; ++i) counts_out[i] = a.counts[static_cast<std::size_t>(i)];
    });
}

int tfg_assign_subgroups_capped(int M, const double* bandwidths, const int* caps, int n_tiers, int* counts_out) {
    return guarded([&] {
        if (n_tiers > 0) {
            need(bandwidths, "bandwidths");
            need(caps, "caps");
            need(counts_out, "counts_out");
        }
        const std::vector<double> b(bandwidths, bandwidths + std::max(n_tiers, 0));
        const std::vector<int> c(caps, caps + std::max(n_tiers, 0));
        const auto a = tfb::assign_subgroups_capped(M, b, c);
        for (int i = 0; i < n_tiers; ++i) counts_out[i] = a.counts[static_cast<std::size_t>(i)];
    });
}

int tfg_destination_plan(const uint32_t* order, int M, int capacity, const double* bandwidths, int n_tiers,
                         int* retain_out, int* tier_out, int* flush_allocation_out) {
    return guarded([&] {
        if (M < 0 || n_tiers < 0) throw tfb::ConfigError("negative size");
        const std::vector<tfb::SubgroupId> ord(order, order + M);
        const std::vector<double> b(bandwidths, bandwidths + n_tiers);
        const tfb::DestinationPlan plan(ord, capacity, b);
        for (int k = 0; k < M; ++k) {
            const auto a = plan.assign_storage_tier(ord[static_cast<std::size_t>(k)]);
            if (retain_out) retain_out[k] = a.host_retain ? 1 : 0;
            if (tier_out) tier_out[k] = a.tier;
        }
        if (flush_allocation_out)
            for (int i = 0; i < n_tiers; ++i)
                flush_allocation_out[i] = plan.flush_allocation().counts[static_cast<std::size_t>(i)];
    });
}

int tfg_update_order(int iteration, const uint32_t* sorted_ids, int M, int alternate, uint32_t* order_out) {
    return guarded([&] {
        if (M < 0) throw tfb::ConfigError("negative size");
        const auto o = tfb::update_order(iteration, std::vector<tfb::SubgroupId>(sorted_ids, sorted_ids + M),
                                         alternate != 0);
        std::copy(o.begin(), o.end(), order_out);
    });
}

int tfg_retention_capacity(int enable_caching, int pool_slots, int cache_slots, int subgroup_count, int* out) {
    return guarded([&] {
        need(out, "out");
        *out = tfb::retention_capacity(enable_caching != 0, pool_slots, cache_slots, subgroup_count);
    });
}

int tfg_update_bandwidth_estimates(double* read_bw, double* write_bw, uint64_t* sample_count, int n_tiers,
                                   double alpha, const tfg_tier_observation* observed, int n_observed) {
    return guarded([&] {
        std::vector<double> r(read_bw, read_bw + n_tiers), w(write_bw, write_bw + n_tiers);
        auto est = tfb::BandwidthEstimate::init(r, w, alpha);
        for (int i = 0; i < n_tiers; ++i) est.tiers[static_cast<std::size_t>(i)].sample_count = sample_count ? sample_count[i] : 0;
        std::vector<tfb::TierObservation> obs;
        for (int i = 0; i < n_observed; ++i) {
            tfb::TierObservation o;
            o.read_transfers = observed[i].read_transfers;
            o.read_bytes = observed[i].read_bytes;
            o.read_seconds = observed[i].read_seconds;
            o.write_transfers = observed[i].write_transfers;
            o.write_bytes = observed[i].write_bytes;
            o.write_seconds = observed[i].write_seconds;
            obs.push_back(o);
        }
        est.update(obs);
        for (int i = 0; i < n_tiers; ++i) {
            read_bw[i] = est.tiers[static_cast<std::size_t>(i)].read_bw;
            write_bw[i] = est.tiers[static_cast<std::size_t>(i)].write_bw;
            if (sample_count) sample_count[i] = est.tiers[static_cast<std::size_t>(i)].sample_count;
        }
    });
}

// ---- trace -----------------------------------------------------------------------

int tfg_trace_create(tfg_trace** out) {
    return guarded([&] {
        need(out, "out");
        *out = new tfg_trace{std::make_shared<tfb::EventTrace>()};
    });
}

int tfg_trace_destroy(tfg_trace* trace) {
    delete trace;
    return TFG_OK;
}

int tfg_trace_size(tfg_trace* trace, uint64_t* size_out) {
    return guarded([&] {
        need(trace, "trace");
        *size_out = trace->t->size();
    });
}

int tfg_trace_copy(tfg_trace* trace, uint64_t begin, tfg_event* out, uint64_t max_n, uint64_t* n_out) {
    static_assert(sizeof(tfg_event) == sizeof(tfb::Event), "event layout");
    return guarded([&] {
        need(trace, "trace");
        const std::size_t n = trace->t->copy_out(begin, reinterpret_cast<tfb::Event*>(out), max_n);
        if (n_out) *n_out = n;
    });
}

int tfg_trace_record(tfg_trace* trace, int kind, int worker, int64_t subgroup, int tier, uint64_t bytes) {
    return guarded([&] {
        need(trace, "trace");
        trace->t->record(static_cast<tfb::EventKind>(kind), worker, subgroup, tier, bytes);
    });
}

struct tfg_pacer {
    tfb::DevicePacer pacer{1.0};  // books device-seconds: bytes / rate
    std::atomic<double> rate{0.0};
};

int tfg_pacer_create(double bytes_per_second, tfg_pacer** out) {
    return guarded([&] {
        need(out, "out");
        if (!(bytes_per_second > 0.0)) throw tfb::ConfigError("token bucket rate must be > 0");
        auto p = std::make_unique<tfg_pacer>();
        p->rate = bytes_per_second;
        *out = p.release();
    });
}

int tfg_pacer_destroy(tfg_pacer* pacer) {
    delete pacer;
    return TFG_OK;
}

int tfg_pacer_set_rate(tfg_pacer* pacer, double bytes_per_second) {
    return guarded([&] {
        need(pacer, "pacer");
        if (!(bytes_per_second > 0.0)) throw tfb::ConfigError("token bucket rate must be > 0");
        pacer->rate = bytes_per_second;
    });
}

int tfg_pacer_rate(tfg_pacer* pacer, double* out) {
    return guarded([&] {
        need(pacer, "pacer");
        need(out, "out");
        *out = pacer->rate.load();
    });
}

int tfg_pacer_acquire(tfg_pacer* pacer, double bytes) {
    return guarded([&] {
        need(pacer, "pacer");
        pacer->pacer.book(bytes / pacer->rate.load());
    });
}

int tfg_file_header_encode(const tfg_file_header* h, uint8_t out[32]) {
    return guarded([&] {
        need(h, "header");
        need(out, "out");
        tfb::SubgroupFileHeader f;
        f.magic = h->magic;
        f.version = h->version;
        f.element_kind = h->element_kind;
        f.subgroup_id = h->subgroup_id;
        f.param_count = h->param_count;
        f.encode(out);
    });
}

int tfg_file_header_decode(const uint8_t in[32], tfg_file_header* out) {
    return guarded([&] {
        need(in, "in");
        need(out, "out");
        const auto f = tfb::SubgroupFileHeader::decode(in);
        *out = tfg_file_header{f.magic, f.version, f.element_kind, f.subgroup_id, f.param_count};
    });
}

int tfg_file_header_validate(const tfg_file_header* h, uint32_t expected_id, uint64_t expected_params) {
    return guarded([&] {
        need(h, "header");
        tfb::SubgroupFileHeader f;
        f.magic = h->magic;
        f.version = h->version;
        f.element_kind = h->element_kind;
        f.subgroup_id = h->subgroup_id;
        f.param_count = h->param_count;
        f.validate(expected_id, expected_params);
    });
}

int tfg_subgroup_file_name(uint32_t id, char* out, uint64_t out_len) {
    return guarded([&] {
        need(out, "out");
        const std::string name = tfb::subgroup_file_name(id);
        if (out_len < name.size() + 1) throw tfb::ConfigError("subgroup_file_name: buffer too small");
        std::memcpy(out, name.c_str(), name.size() + 1);
    });
}

int tfg_trace_record_at(tfg_trace* trace, int64_t timestamp_ns, int kind, int worker, int64_t subgroup, int tier,
                        uint64_t bytes) {
    return guarded([&] {
        need(trace, "trace");
        trace->t->append(tfb::Event{timestamp_ns, worker, kind, subgroup, tier, 0, bytes});
    });
}

int tfg_trace_write(tfg_trace* trace, const char* path) {
    return guarded([&] {
        need(trace, "trace");
        need(path, "path");
        std::ofstream os(path, std::ios::trunc);
        if (!os) throw tfb::IoError(std::string("cannot write trace to ") + path);
        const std::string p(path);
        if (p.size() >= 6 && p.compare(p.size() - 6, 6, ".jsonl") == 0)
            trace->t->write_jsonl(os);
        else
            trace->t->write_csv(os);
    });
}

int tfg_trace_clear(tfg_trace* trace) {
    return guarded([&] {
        need(trace, "trace");
        trace->t->clear();
    });
}

// ---- tiers -------------------------------------------------------------------------

int tfg_tier_create(const tfg_tier_spec* spec, tfg_tier** out) {
    return guarded([&] {
        need(spec, "spec");
        need(out, "out");
        tfb::TierSpec s;
        s.tier_id = spec->tier_id;
        if (spec->kind < 0 || spec->kind > 3) throw tfb::ConfigError("unknown tier kind");
        s.kind = static_cast<tfb::TierKind>(spec->kind);
        s.root = spec->root ? spec->root : "";
        s.read_bw = spec->read_bw;
        s.write_bw = spec->write_bw;
        s.io_parallelism = spec->io_parallelism;
        s.persistent = spec->persistent != 0;
        s.lock_width = spec->lock_width;
        s.direct_io = spec->direct_io != 0;
        if (spec->lock_device < 0) throw tfb::ConfigError("lock_device must be >= 0");
        s.lock_device = spec->lock_device;
        s.capacity_bytes = spec->capacity_bytes;
        if ((s.kind == tfb::TierKind::local_dir || s.kind == tfb::TierKind::remote_dir) && s.root.empty())
            throw tfb::ConfigError("directory tiers need a root path");
        *out = new tfg_tier{std::make_shared<tfb::Tier>(s)};
    });
}

int tfg_tier_destroy(tfg_tier* tier) {
    delete tier;
    return TFG_OK;
}

int tfg_tier_bandwidths(tfg_tier* tier, double* read_bw, double* write_bw) {
    return guarded([&] {
        need(tier, "tier");
        if (read_bw) *read_bw = tier->t->spec().read_bw;
        if (write_bw) *write_bw = tier->t->spec().write_bw;
    });
}

int tfg_tier_set_throttle_rates(tfg_tier* tier, double read_bps, double write_bps) {
    return guarded([&] {
        need(tier, "tier");
        tier->t->set_throttle_rates(read_bps, write_bps);
    });
}

int tfg_tier_write_subgroup(tfg_tier* tier, uint32_t id, uint64_t params, const float* state, uint64_t* bytes_out,
                            double* seconds_out) {
    return guarded([&] {
        need(tier, "tier");
        need(state, "state");
        const auto st = tier->t->write_subgroup(id, params, state);
        if (bytes_out) *bytes_out = st.bytes;
        if (seconds_out) *seconds_out = st.seconds;
    });
}

int tfg_tier_read_subgroup(tfg_tier* tier, uint32_t id, uint64_t params, float* state, uint64_t* bytes_out,
                           double* seconds_out) {
    return guarded([&] {
        need(tier, "tier");
        need(state, "state");
        const auto st = tier->t->read_subgroup(id, params, state);
        if (bytes_out) *bytes_out = st.bytes;
        if (seconds_out) *seconds_out = st.seconds;
    });
}

int tfg_tier_write_grads(tfg_tier* tier, uint32_t id, uint64_t params, const float* grads) {
    return guarded([&] {
        need(tier, "tier");
        tier->t->write_grads(id, params, grads);
    });
}

int tfg_tier_read_grads(tfg_tier* tier, uint32_t id, uint64_t params, float* grads) {
    return guarded([&] {
        need(tier, "tier");
        tier->t->read_grads(id, params, grads);
    });
}

int tfg_tier_has_subgroup(tfg_tier* tier, uint32_t id, int* out) {
    return guarded([&] {
        need(tier, "tier");
        *out = tier->t->has_subgroup(id) ? 1 : 0;
    });
}

int tfg_tier_remove_subgroup(tfg_tier* tier, uint32_t id) {
    return guarded([&] {
        need(tier, "tier");
        tier->t->remove_subgroup(id);
    });
}

int tfg_tier_probe(tfg_tier* tier, uint64_t probe_bytes, int repetitions, double* read_bw, double* write_bw,
                   int* low_confidence) {
    return guarded([&] {
        need(tier, "tier");
        const auto r = tier->t->probe_bandwidth(probe_bytes, repetitions);
        if (read_bw) *read_bw = r.read_bw;
        if (write_bw) *write_bw = r.write_bw;
        if (low_confidence) *low_confidence = r.low_confidence ? 1 : 0;
    });
}

int tfg_tier_available_bytes(tfg_tier* tier, uint64_t* out) {
    return guarded([&] {
        need(tier, "tier");
        *out = tier->t->available_bytes();
    });
}

int tfg_tier_lock_acquire(const char* lock_dir, int tier, int worker, tfg_trace* trace, int width, void** token) {
    return guarded([&] {
        need(lock_dir, "lock_dir");
        need(token, "token");
        *token = new tfb::TierLockGuard(lock_dir, tier, worker, trace ? trace->t.get() : nullptr, width);
    });
}

int tfg_tier_lock_release(void* token) {
    return guarded([&] { delete static_cast<tfb::TierLockGuard*>(token); });
}

// ---- engine --------------------------------------------------------------------------

int tfg_engine_create(int worker_id, tfg_tier* const* tiers, int n_tiers, const tfg_schedule_options* options,
                      const tfg_adam_hyper* hyper, tfg_trace* trace, const tfg_device_options* device,
                      tfg_engine** out) {
    return guarded([&] {
        need(out, "out");
        need(options, "options");
        if (n_tiers < 1 || n_tiers > TFG_MAX_TIERS) throw tfb::ConfigError("engine needs 1..8 tiers");
        std::vector<std::shared_ptr<tfb::Tier>> ts;
        for (int i = 0; i < n_tiers; ++i) {
            need(tiers[i], "tier");
            ts.push_back(tiers[i]->t);
        }
        tfb::ScheduleOptions o;
        o.pool_slots = options->pool_slots;
        o.cache_slots = options->cache_slots;
        o.enable_caching = options->enable_caching != 0;
        o.skip_gradients = options->skip_gradients != 0;
        o.atomic_rw = options->atomic_rw != 0;
        o.multi_path = options->multi_path != 0;
        o.lock_dir = options->lock_dir ? options->lock_dir : "";
        o.update_threads = options->update_threads;
        o.deadlock_timeout_s = options->deadlock_timeout_s;
        o.update_pad_ns = options->update_pad_ns;
        tfb::DeviceOptions d;
        if (device) {
            d.device = device->device;
            d.grad_kind = device->grad_dtype;
            d.out_kind = device->param_dtype;
            d.device_buffers = device->device_buffers;
            d.zero_copy = device->zero_copy;
            d.d2h_split = device->d2h_split;
            d.h2d_split = device->h2d_split > 1 ? 2 : 1;
            if (device->hbm_cache_slots < 0) throw tfb::ConfigError("hbm_cache_slots must be >= 0");
            d.hbm_cache_slots = device->hbm_cache_slots;
            d.hbm_retain = device->hbm_retain;
            d.host_grads = device->host_grads != 0;
        }
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= d.device || d.device < 0) {
            (void)cudaGetLastError();
            throw tfb::CudaError("no usable CUDA device " + std::to_string(d.device) +
                                 " (the update engine runs only on the GPU)");
        }
        auto e = std::make_unique<tfg_engine>();
        e->w = std::make_unique<tfb::OffloadWorker>(worker_id, std::move(ts), o, to_hyper(hyper),
                                                    trace ? trace->t : nullptr, d);
        *out = e.release();
    });
}

int tfg_engine_destroy(tfg_engine* engine) {
    return guarded([&] { delete engine; });
}

int tfg_engine_set_alpha(tfg_engine* engine, double alpha) {
    return guarded([&] {
        need(engine, "engine");
        engine->w->set_alpha(alpha);
    });
}

int tfg_engine_set_fixed_ratio(tfg_engine* engine, const double* ratio, int n) {
    return guarded([&] {
        need(engine, "engine");
        engine->w->set_fixed_ratio(std::vector<double>(ratio, ratio + std::max(n, 0)));
    });
}

int tfg_engine_add_subgroup(tfg_engine* engine, uint32_t id, uint64_t param_count) {
    return guarded([&] {
        need(engine, "engine");
        engine->w->add_subgroup(id, param_count);
    });
}

int tfg_engine_init_and_flush_all(tfg_engine* engine, uint64_t seed) {
    return guarded([&] {
        need(engine, "engine");
        engine->w->init_and_flush_all(seed);
    });
}

int tfg_engine_run_backward_sim(tfg_engine* engine, int iteration, uint64_t seed, int accum_steps) {
    return guarded([&] {
        need(engine, "engine");
        engine->w->run_backward_sim(iteration, seed, accum_steps);
    });
}

int tfg_engine_gradients_finite(tfg_engine* engine, int* out) {
    return guarded([&] {
        need(engine, "engine");
        *out = engine->w->gradients_finite() ? 1 : 0;
    });
}

int tfg_engine_grad_buffer(tfg_engine* engine, uint32_t id, void** device_ptr) {
    return guarded([&] {
        need(engine, "engine");
        *device_ptr = engine->w->grad_buffer(id);
    });
}

int tfg_engine_bind_grad_buffer(tfg_engine* engine, uint32_t id, void* device_ptr) {
    return guarded([&] {
        need(engine, "engine");
        engine->w->bind_grad_buffer(id, device_ptr);
    });
}

int tfg_engine_set_cache_slots(tfg_engine* engine, int cache_slots) {
    return guarded([&] {
        need(engine, "engine");
        engine->w->set_cache_slots(cache_slots);
    });
}

int tfg_engine_set_producer_stream(tfg_engine* engine, void* stream) {
    return guarded([&] {
        need(engine, "engine");
        engine->w->set_producer_stream(stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy);
    });
}

int tfg_engine_bind_grad_sources(tfg_engine* engine, uint32_t id, const void* const* device_ptrs, int n) {
    return guarded([&] {
        need(engine, "engine");
        if (n < 0 || (n > 0 && device_ptrs == nullptr)) throw tfb::ConfigError("bind_grad_sources: bad source list");
        engine->w->bind_grad_sources(id, std::vector<const void*>(device_ptrs, device_ptrs + n));
    });
}

int tfg_engine_params16_buffer(tfg_engine* engine, uint32_t id, void** device_ptr) {
    return guarded([&] {
        need(engine, "engine");
        *device_ptr = engine->w->params16_buffer(id);
    });
}

int tfg_engine_run_update(tfg_engine* engine, int iteration, tfg_phase_stats* stats) {
    return guarded([&] {
        need(engine, "engine");
        const tfb::PhaseStats st = engine->w->run_update(iteration);
        engine->last_io = st.subgroup_io;
        engine->last_timeline = st.timeline;
        if (stats == nullptr) return;
        std::memset(stats, 0, sizeof(*stats));
        stats->wall_seconds = st.wall_seconds;
        stats->params_updated = st.params_updated;
        stats->cache_hits = st.cache_hits;
        stats->downscale_overflows = st.downscale_overflows;
        stats->retained = st.retained;
        stats->n_tiers = static_cast<int32_t>(st.tier_obs.size());
        for (std::size_t i = 0; i < st.flush_allocation.size() && i < TFG_MAX_TIERS; ++i)
            stats->flush_allocation[i] = st.flush_allocation[i];
        for (std::size_t i = 0; i < st.tier_obs.size() && i < TFG_MAX_TIERS; ++i) {
            const auto& o = st.tier_obs[i];
            stats->tier_obs[i] = tfg_tier_observation{o.read_transfers, o.read_bytes, o.read_seconds,
                                                      o.write_transfers, o.write_bytes, o.write_seconds};
        }
        stats->n_subgroup_io = st.subgroup_io.size();
        stats->device_seconds = st.device_seconds;
        stats->kernel_seconds = st.kernel_seconds;
        stats->h2d_seconds = st.h2d_seconds;
        stats->d2h_seconds = st.d2h_seconds;
        stats->h2d_bytes = st.h2d_bytes;
        stats->d2h_bytes = st.d2h_bytes;
    });
}

int tfg_engine_last_subgroup_io(tfg_engine* engine, tfg_subgroup_io* out, uint64_t max_n, uint64_t* n_out) {
    return guarded([&] {
        need(engine, "engine");
        const std::size_t n = std::min<std::size_t>(max_n, engine->last_io.size());
        for (std::size_t i = 0; i < n; ++i) {
            const auto& e = engine->last_io[i];
            out[i] = tfg_subgroup_io{e.id, e.fetched ? 1u : 0u, e.flushed ? 1u : 0u, 0u, e.state_bytes, e.read_seconds,
                                     e.write_seconds};
        }
        if (n_out) *n_out = n;
    });
}

int tfg_engine_last_timeline(tfg_engine* engine, tfg_device_span* out, uint64_t max_n, uint64_t* n_out) {
    static_assert(sizeof(tfg_device_span) == sizeof(tfb::DeviceSpan), "span layout");
    return guarded([&] {
        need(engine, "engine");
        const std::size_t n = std::min<std::size_t>(max_n, engine->last_timeline.size());
        if (n > 0) need(out, "out");
        std::memcpy(out, engine->last_timeline.data(), n * sizeof(tfg_device_span));
        if (n_out) *n_out = n;
    });
}

int tfg_engine_wait_host_resident(tfg_engine* engine, uint32_t id, int* slot_out) {
    return guarded([&] {
        need(engine, "engine");
        const int s = engine->w->wait_host_resident(id);
        if (slot_out) *slot_out = s;
    });
}

int tfg_engine_enqueue_prefetch(tfg_engine* engine, uint32_t id, uint64_t* ticket_out) {
    return guarded([&] {
        need(engine, "engine");
        auto f = engine->w->enqueue_prefetch(id);
        std::uint64_t ticket = 0;
        if (f) {
            std::lock_guard<std::mutex> g(engine->mu);
            ticket = engine->next_ticket++;
            engine->tickets[ticket] = *f;
        }
        if (ticket_out) *ticket_out = ticket;
    });
}

int tfg_engine_enqueue_flush(tfg_engine* engine, uint32_t id, int dest, uint64_t* ticket_out) {
    return guarded([&] {
        need(engine, "engine");
        auto f = engine->w->enqueue_flush(id, dest);
        std::lock_guard<std::mutex> g(engine->mu);
        const std::uint64_t ticket = engine->next_ticket++;
        engine->tickets[ticket] = f;
        if (ticket_out) *ticket_out = ticket;
    });
}

int tfg_engine_wait_ticket(tfg_engine* engine, uint64_t ticket, uint64_t* bytes_out, double* seconds_out) {
    return guarded([&] {
        need(engine, "engine");
        if (ticket == 0) {  // cache hit: nothing was queued
            if (bytes_out) *bytes_out = 0;
            if (seconds_out) *seconds_out = 0.0;
            return;
        }
        std::shared_future<tfb::IoStats> f;
        {
            std::lock_guard<std::mutex> g(engine->mu);
            auto it = engine->tickets.find(ticket);
            if (it == engine->tickets.end()) throw tfb::Error("unknown ticket " + std::to_string(ticket));
            f = it->second;
            engine->tickets.erase(it);
        }
        const tfb::IoStats st = engine->w->watchdog_wait_value(f);
        if (bytes_out) *bytes_out = st.bytes;
        if (seconds_out) *seconds_out = st.seconds;
    });
}

int tfg_engine_read_state(tfg_engine* engine, uint32_t id, float* out_3n) {
    return guarded([&] {
        need(engine, "engine");
        need(out_3n, "out");
        engine->w->read_current_state(id, out_3n);
    });
}

int tfg_engine_read_params16(tfg_engine* engine, uint32_t id, uint16_t* out_n) {
    return guarded([&] {
        need(engine, "engine");
        need(out_n, "out");
        const auto meta = engine->w->meta(id);
        tfb::cuda_check(cudaSetDevice(engine->w->device_options().device), "cudaSetDevice");
        tfb::cuda_check(cudaMemcpy(out_n, engine->w->params16_buffer(id), 2 * meta.param_count, cudaMemcpyDefault),
                        "cudaMemcpy(params16)");
    });
}

int tfg_engine_read_grads16(tfg_engine* engine, uint32_t id, uint16_t* out_n) {
    return guarded([&] {
        need(engine, "engine");
        need(out_n, "out");
        const auto meta = engine->w->meta(id);
        tfb::cuda_check(cudaSetDevice(engine->w->device_options().device), "cudaSetDevice");
        tfb::cuda_check(cudaMemcpy(out_n, engine->w->grad_buffer(id), 2 * meta.param_count, cudaMemcpyDefault),
                        "cudaMemcpy(grads16)");
    });
}

int tfg_engine_write_grads16(tfg_engine* engine, uint32_t id, const uint16_t* in_n) {
    return guarded([&] {
        need(engine, "engine");
        need(in_n, "in");
        const auto meta = engine->w->meta(id);
        tfb::cuda_check(cudaSetDevice(engine->w->device_options().device), "cudaSetDevice");
        tfb::cuda_check(cudaMemcpy(engine->w->grad_buffer(id), in_n, 2 * meta.param_count, cudaMemcpyDefault),
                        "cudaMemcpy(grads16)");
    });
}

int tfg_engine_meta(tfg_engine* engine, uint32_t id, tfg_subgroup_meta* out) {
    return guarded([&] {
        need(engine, "engine");
        need(out, "out");
        const auto m = engine->w->meta(id);
        *out = tfg_subgroup_meta{m.id, static_cast<int32_t>(m.residency), m.tier, m.slot, m.param_count, m.step_count};
    });
}

int tfg_engine_residency_census(tfg_engine* engine, uint64_t* host_params, uint64_t* per_tier, int n_tiers) {
    return guarded([&] {
        need(engine, "engine");
        const auto [h, t] = engine->w->residency_census();
        if (host_params) *host_params = h;
        for (int i = 0; i < n_tiers && static_cast<std::size_t>(i) < t.size(); ++i) per_tier[i] = t[static_cast<std::size_t>(i)];
    });
}

int tfg_engine_current_order(tfg_engine* engine, uint32_t* out, int max_n, int* n_out) {
    return guarded([&] {
        need(engine, "engine");
        const auto o = engine->w->current_order();
        const int n = std::min<int>(max_n, static_cast<int>(o.size()));
        for (int i = 0; i < n; ++i) out[i] = o[static_cast<std::size_t>(i)];
        if (n_out) *n_out = static_cast<int>(o.size());
    });
}

int tfg_engine_estimates(tfg_engine* engine, double* read_bw, double* write_bw, int n_tiers) {
    return guarded([&] {
        need(engine, "engine");
        const auto& est = engine->w->estimates();
        for (int i = 0; i < n_tiers && static_cast<std::size_t>(i) < est.tiers.size(); ++i) {
            if (read_bw) read_bw[i] = est.tiers[static_cast<std::size_t>(i)].read_bw;
            if (write_bw) write_bw[i] = est.tiers[static_cast<std::size_t>(i)].write_bw;
        }
    });
}

int tfg_engine_pool_state(tfg_engine* engine, int slot, int* state_out, uint32_t* owner_out) {
    return guarded([&] {
        need(engine, "engine");
        if (state_out) *state_out = static_cast<int>(engine->w->pool().state(slot));
        if (owner_out) *owner_out = engine->w->pool().owner(slot);
    });
}

}  // extern "C"
