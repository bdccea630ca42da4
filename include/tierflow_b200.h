/*
 * tierflow_b200.h — C ABI of the B200-native MLP-Offload update phase.
 *
 * The reference ("tierflow", /root/reference/proj) is a header-only C++20
 * library with no FFI layer; its drop-in boundary is the C++ API the harness
 * and tests call. Every entry point below replaces one of those calls and
 * cites it as reference-file:line (paths relative to proj/include/tierflow/).
 * Plain C types only: opaque handles, pointers and sizes; device pointers are
 * `void*` / typed pointers into CUDA device memory; streams are
 * `cudaStream_t` passed as `void*` (NULL = legacy default stream).
 *
 * Errors: every function returns a tfg_status. The C++ exception hierarchy of
 * the reference (common.hpp:36-78) maps one to one onto the codes; the message
 * of the last failure on the calling thread is returned by tfg_last_error().
 * No exception crosses this boundary.
 *
 * Library: paper_2509_02480_b200/lib/libtierflow_b200.so (sm_100a).
 */
#ifndef TIERFLOW_B200_H
#define TIERFLOW_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TFG_ABI_VERSION 5  /* 5: tfg_device_span.d2h_start */
#define TFG_MAX_TIERS 8

typedef enum tfg_status {
    TFG_OK = 0,
    TFG_ERROR = 1,                   /* tierflow::Error                       common.hpp:36  */
    TFG_IO_ERROR = 2,                /* tierflow::IoError                     common.hpp:42  */
    TFG_FORMAT_ERROR = 3,            /* tierflow::FormatError                 common.hpp:48  */
    TFG_CONFIG_ERROR = 4,            /* tierflow::ConfigError                 common.hpp:54  */
    TFG_PLACEMENT_INCONSISTENCY = 5, /* tierflow::PlacementInconsistencyError common.hpp:61  */
    TFG_SCHEDULING_BUG = 6,          /* tierflow::SchedulingBugError          common.hpp:67  */
    TFG_GRADIENT_OVERFLOW = 7,       /* tierflow::GradientOverflowError       common.hpp:73  */
    TFG_CUDA_ERROR = 8               /* CUDA runtime failure (no reference counterpart)      */
} tfg_status;

/* Element kinds: gradients F16 / BF16 / F32 (F32 = the ZeRO-3 baseline flow's
 * stored fp32 gradients); working parameters F16 / BF16. */
typedef enum tfg_dtype { TFG_F16 = 0, TFG_BF16 = 1, TFG_F32 = 2 } tfg_dtype;

/* Tier kinds: tier.hpp:32 plus TFG_HOST_DRAM (pinned host blobs, zero-copy). */
typedef enum tfg_tier_kind {
    TFG_LOCAL_DIR = 0,
    TFG_REMOTE_DIR = 1,
    TFG_MEM_THROTTLED = 2,
    TFG_HOST_DRAM = 3
} tfg_tier_kind;

/* AdamHyper, optimizer.hpp:17-31. */
typedef struct tfg_adam_hyper {
    double lr;
    double beta1;
    double beta2;
    double eps;
    double weight_decay;
} tfg_adam_hyper;

/* TierSpec, tier.hpp:43-51 (+ lock_width, direct_io). */
typedef struct tfg_tier_spec {
    int32_t tier_id;
    int32_t kind;            /* tfg_tier_kind */
    const char* root;        /* directory for *_DIR kinds, a label otherwise */
    double read_bw;          /* bytes/s, configured (or 0 and probe) */
    double write_bw;
    int32_t io_parallelism;  /* >= 1 */
    int32_t persistent;
    int32_t lock_width;      /* tier semaphore width; 1 = exclusive flock (the reference) */
    int32_t direct_io;       /* O_DIRECT on the engine path when the filesystem allows */
    int32_t lock_device;     /* 0: the tier's own semaphore (the reference); k > 0: one semaphore
                                shared by every tier with the same k, i.e. per physical device,
                                so tiers on one disk do not contend with concurrent transfers */
    uint64_t capacity_bytes; /* 0: unlimited (the reference); else the state bytes the tier may hold:
                                Eq. 1 is capped at capacity / state block bytes subgroups per tier */
} tfg_tier_spec;

/* ScheduleOptions, scheduler.hpp:32-50. */
typedef struct tfg_schedule_options {
    int32_t pool_slots;
    int32_t cache_slots;     /* -1 derives pool_slots - 3 */
    int32_t enable_caching;
    int32_t skip_gradients;  /* must be 1 on the GPU engine (fused widening) */
    int32_t atomic_rw;
    int32_t multi_path;
    const char* lock_dir;    /* NULL/"" = <tmp>/tierflow-locks */
    int32_t update_threads;  /* accepted for parity, unused (update runs on the GPU) */
    double deadlock_timeout_s;
    uint64_t update_pad_ns;
} tfg_schedule_options;

/* GPU placement of one engine (no reference counterpart). */
typedef struct tfg_device_options {
    int32_t device;          /* CUDA ordinal */
    int32_t grad_dtype;      /* tfg_dtype of the device gradient buffers */
    int32_t param_dtype;     /* tfg_dtype of the device working-parameter buffers */
    int32_t device_buffers;  /* depth of the H2D -> kernel -> D2H ring (>= 1) */
    int32_t zero_copy;       /* 0: copy engines via the device ring; 1: the fused kernel streams the
                                pinned slot over PCIe both ways; 2: DMA in, the kernel's epilogue
                                writes the updated state back into the pinned slot */
    int32_t d2h_split;       /* copy mode: concurrent D2H streams per subgroup (1 or 2) */
    int32_t hbm_retain;      /* copy mode, 16-bit gradients: retained subgroups keep their state in
                                HBM between phases (no D2H now, no H2D at the next update).
                                1: the host slot stays reserved, C = min(cache_slots, pool_slots-3)
                                as in the reference; 2 (HBM cache): the slot streams again and
                                C = cache_slots (or pool_slots-3 if < 0), bounded by HBM only */
    int32_t h2d_split;       /* copy mode: concurrent H2D streams per subgroup (0 or 1: one; 2: two) */
    int32_t hbm_cache_slots; /* hbm_retain 2: HBM buffers for retained subgroups; 0 = all of C. Fewer
                                than C makes a two-level cache: the rest keep their host slots, and
                                C = min(cache_slots, hbm_cache_slots + pool_slots - 3) */
    int32_t host_grads;      /* (ABI 3) 1: the 16-bit gradients and working params live in pinned host
                                memory per subgroup and stream with the state (2 B/param more each
                                way) instead of 4 B/param of HBM for the whole shard; grad_buffer /
                                params16_buffer / bind_grad_buffer then take host pointers. Copy
                                pipeline and 16-bit gradient flow only */
} tfg_device_options;

typedef struct tfg_tier_observation { /* placement.hpp:138-145 */
    uint64_t read_transfers;
    double read_bytes;
    double read_seconds;
    uint64_t write_transfers;
    double write_bytes;
    double write_seconds;
} tfg_tier_observation;

typedef struct tfg_subgroup_io { /* scheduler.hpp:114-121 */
    uint32_t id;
    uint32_t fetched;
    uint32_t flushed;
    uint32_t pad;
    uint64_t state_bytes;
    double read_seconds;
    double write_seconds;
} tfg_subgroup_io;

/* PhaseStats, scheduler.hpp:123-132, plus the device timeline. */
typedef struct tfg_phase_stats {
    double wall_seconds;
    uint64_t params_updated;
    uint64_t cache_hits;
    uint64_t downscale_overflows;
    int32_t retained;
    int32_t n_tiers;
    int32_t flush_allocation[TFG_MAX_TIERS];
    tfg_tier_observation tier_obs[TFG_MAX_TIERS];
    uint64_t n_subgroup_io;  /* entries available via tfg_engine_last_subgroup_io */
    double device_seconds;   /* phase start -> last D2H end (CUDA events) */
    double kernel_seconds;   /* sum of fused-kernel durations */
    double h2d_seconds;
    double d2h_seconds;
    uint64_t h2d_bytes;
    uint64_t d2h_bytes;
} tfg_phase_stats;

/* Event, trace.hpp:65-72 (POD layout). */
typedef struct tfg_event {
    int64_t timestamp_ns;
    int32_t worker_id;
    int32_t kind;  /* EventKind order of trace.hpp:19-33 */
    int64_t subgroup_id;
    int32_t tier_id;
    int32_t pad;
    uint64_t bytes;
} tfg_event;

/* One subgroup's pass through the pipeline in the last phase (no reference
 * counterpart): device times from CUDA events, ms from the phase start;
 * host times ms from run_update entry. */
typedef struct tfg_device_span {
    uint32_t id;
    float h2d_start, h2d_end, k_start, k_end, d2h_end;
    float host_resident, host_retired;
    float d2h_start;
} tfg_device_span;

typedef struct tfg_subgroup_meta { /* Subgroup, optimizer.hpp:39-73 */
    uint32_t id;
    int32_t residency;  /* 0 host_cached, 1 in_flight, 2 on_tier */
    int32_t tier;
    int32_t slot;
    uint64_t param_count;
    uint64_t step_count;
} tfg_subgroup_meta;

typedef struct tfg_tier tfg_tier;
typedef struct tfg_trace tfg_trace;
typedef struct tfg_engine tfg_engine;

/* ---- library ------------------------------------------------------------ */
const char* tfg_last_error(void);
int tfg_abi_version(void);
int tfg_device_count(int* count);

/* ---- peer memory (fused data-parallel gradient exchange) ----------------- */
/* Device buffers that other ranks map over NVLink: cudaMalloc'd (whole
 * allocations, so an IPC handle maps exactly this buffer), shared as the
 * 64-byte cudaIpcMemHandle_t. Opening maps the peer's buffer with lazy peer
 * access; a rank never opens its own handle. No reference counterpart: they
 * replace the NCCL reduce in front of the update. */
#define TFG_IPC_HANDLE_BYTES 64
int tfg_device_alloc(int device, uint64_t bytes, void** out);
int tfg_device_free(int device, void* ptr);
int tfg_ipc_get_handle(int device, void* ptr, unsigned char* handle_out);
int tfg_ipc_open_handle(int device, const unsigned char* handle, void** out);
int tfg_ipc_close_handle(int device, void* ptr);

/* ---- kernels (device pointers, async on `stream`) ------------------------ */
/* Fused upscale_f16_to_f32 -> adam_step -> downscale_f32_to_f16
 * (precision.hpp:17, optimizer.hpp:116, precision.hpp:29; composed at
 * scheduler.hpp:467-490). t >= 1 is the Adam timestep; bc1/bc2 are computed on
 * the host with pow() as optimizer.hpp:129-130. counters (device, 2 x u64) are
 * accumulated: [0] += non-finite gradients, [1] += +-Inf 16-bit outputs. */
int tfg_adam_fused(float* p, float* m, float* v, const void* grad, int grad_dtype, uint16_t* param16,
                   int param_dtype, uint64_t n, const tfg_adam_hyper* hyper, uint64_t t,
                   unsigned long long* counters, void* stream);
/* tfg_adam_fused behind a device-side gate: when *gate (device memory) is
 * nonzero when the kernel starts, it writes nothing. A whole-phase non-finite
 * count accumulated into the gate on the same stream (tfg_count_nonfinite16)
 * rejects the phase's updates with no host round trip: the reference's
 * check-before-mutate (harness.hpp:218-228, optimizer.hpp:123-127). The gate
 * is taken as that count of this launch's gradients: a gated launch does not
 * count non-finite gradients again (counters[0] is left alone; [1] still
 * counts overflows). */
int tfg_adam_fused_gated(float* p, float* m, float* v, const void* grad, int grad_dtype, uint16_t* param16,
                         int param_dtype, uint64_t n, const tfg_adam_hyper* hyper, uint64_t t,
                         unsigned long long* counters, const unsigned long long* gate, void* stream);
/* Reduce + update in one pass: the gradient is the fp32 sum, in source order,
 * of n_sources (<= 8) 16-bit buffers — e.g. every data-parallel peer's
 * contribution to this rank's subgroup, read over NVLink through mapped peer
 * pointers — rounded once to grad_dtype, then the fused Adam step. Replaces a
 * reduce-scatter followed by tfg_adam_fused. */
int tfg_adam_fused_multi(float* p, float* m, float* v, const void* const* grads, int n_sources, int grad_dtype,
                         uint16_t* param16, int param_dtype, uint64_t n, const tfg_adam_hyper* hyper, uint64_t t,
                         unsigned long long* counters, void* stream);
/* Same on one contiguous P||m||v state (StateView::from_contiguous, optimizer.hpp:82-86). */
int tfg_adam_fused_contiguous(float* state, uint64_t n, const void* grad, int grad_dtype, uint16_t* param16,
                              int param_dtype, const tfg_adam_hyper* hyper, uint64_t t,
                              unsigned long long* counters, void* stream);
/* Reference-semantics synchronous step (adam_step, optimizer.hpp:116-157):
 * validates, rejects non-finite gradients with TFG_GRADIENT_OVERFLOW before
 * mutating state, then runs the fused kernel and synchronizes.
 * overflows_out (host, may be NULL) receives the narrowing overflow count. */
int tfg_adam_step(float* p, float* m, float* v, const uint16_t* grad, int grad_dtype, uint16_t* param16,
                  int param_dtype, uint64_t n, const tfg_adam_hyper* hyper, uint64_t t, uint64_t* overflows_out,
                  void* stream);
/* The kernel's tuning variants live in a separate library (include/tierflow_b200_tuning.h). */
/* Self-test of the constant-divisor quotient used for m/bc1, v/bc2 against
 * div.rn.f64 on n generated numerators (synchronous; host outputs). */
int tfg_selftest_div_const(double divisor, uint64_t n, uint64_t seed, int exp_lo, int exp_span,
                           uint64_t* mismatches, double* first_bad);
/* upscale_f16_to_f32, precision.hpp:17-25 (nonfinite: device u64, accumulated). */
int tfg_upscale16(const uint16_t* src, float* dst, uint64_t n, int dtype, unsigned long long* nonfinite,
                  void* stream);
/* downscale_f32_to_f16, precision.hpp:29-37 (overflows: device u64, accumulated). */
int tfg_downscale16(const float* src, uint16_t* dst, uint64_t n, int dtype, unsigned long long* overflows,
                    void* stream);
/* all_finite, precision.hpp:39-43 (count: device u64, accumulated). */
int tfg_count_nonfinite16(const uint16_t* src, uint64_t n, int dtype, unsigned long long* count, void* stream);
/* SyntheticGradSource::fill (+ GradBufferF16::accumulate when accumulate != 0),
 * scheduler.hpp:85-102, precision.hpp:66-75. */
int tfg_synthetic_grads(uint16_t* out, uint64_t n, int dtype, uint64_t seed, uint32_t subgroup, int iteration,
                        int step, int accumulate, void* stream);
/* synthetic_param_init into P, zeros into m and v (scheduler.hpp:104-110, 352). */
int tfg_synthetic_state(float* p, float* m, float* v, uint64_t n, uint64_t seed, uint32_t subgroup, void* stream);

/* ---- placement (host, pure) --------------------------------------------- */
/* assign_subgroups, placement.hpp:30-100. counts_out[n_tiers]. */
int tfg_assign_subgroups(int M, const double* bandwidths, int n_tiers, int* counts_out);
/* Host blocks (pinned slots, tier blobs, staging) alive in the process: leak accounting. */
int tfg_host_blocks_live(int64_t* blocks_out, int64_t* bytes_out, int64_t* free_failures_out);
/* Capacity-aware Eq. 1 (beyond the reference): caps[i] < 0 unlimited; the
   reference allocation whenever it fits every cap, else the min-max of T_i/B_i
   subject to T_i <= caps[i] (water filling). ConfigError if the caps cannot hold M. */
int tfg_assign_subgroups_capped(int M, const double* bandwidths, const int* caps, int n_tiers, int* counts_out);
/* DestinationPlan, placement.hpp:178-225: per order position, retain flag and tier. */
int tfg_destination_plan(const uint32_t* order, int M, int capacity, const double* bandwidths, int n_tiers,
                         int* retain_out, int* tier_out, int* flush_allocation_out);
/* UpdatePlan::make, scheduler.hpp:60-67 (sorted_ids ascending). */
int tfg_update_order(int iteration, const uint32_t* sorted_ids, int M, int alternate, uint32_t* order_out);
/* ScheduleOptions::retention_capacity, scheduler.hpp:44-49. */
int tfg_retention_capacity(int enable_caching, int pool_slots, int cache_slots, int subgroup_count, int* out);
/* update_bandwidth_estimates, placement.hpp:149-162, on arrays of n_tiers. */
int tfg_update_bandwidth_estimates(double* read_bw, double* write_bw, uint64_t* sample_count, int n_tiers,
                                   double alpha, const tfg_tier_observation* observed, int n_observed);

/* ---- trace --------------------------------------------------------------- */
int tfg_trace_create(tfg_trace** out);                       /* EventTrace, trace.hpp:77 */
int tfg_trace_destroy(tfg_trace* trace);
int tfg_trace_size(tfg_trace* trace, uint64_t* size_out);
int tfg_trace_copy(tfg_trace* trace, uint64_t begin, tfg_event* out, uint64_t max_n, uint64_t* n_out);
int tfg_trace_record(tfg_trace* trace, int kind, int worker, int64_t subgroup, int tier, uint64_t bytes);
int tfg_trace_record_at(tfg_trace* trace, int64_t timestamp_ns, int kind, int worker, int64_t subgroup, int tier,
                        uint64_t bytes);                      /* EventTrace::append, trace.hpp:79 */
int tfg_trace_write(tfg_trace* trace, const char* path);     /* .jsonl or CSV, trace.hpp:119-134 */
int tfg_trace_clear(tfg_trace* trace);

/* ---- tiers ---------------------------------------------------------------- */
int tfg_tier_create(const tfg_tier_spec* spec, tfg_tier** out);            /* Tier(TierSpec), tier.hpp:159 */
int tfg_tier_destroy(tfg_tier* tier);
int tfg_tier_bandwidths(tfg_tier* tier, double* read_bw, double* write_bw);
int tfg_tier_set_throttle_rates(tfg_tier* tier, double read_bps, double write_bps);   /* tier.hpp:181 */
int tfg_tier_write_subgroup(tfg_tier* tier, uint32_t id, uint64_t params, const float* state,
                            uint64_t* bytes_out, double* seconds_out);                 /* tier.hpp:192 */
int tfg_tier_read_subgroup(tfg_tier* tier, uint32_t id, uint64_t params, float* state,
                           uint64_t* bytes_out, double* seconds_out);                  /* tier.hpp:199 */
int tfg_tier_write_grads(tfg_tier* tier, uint32_t id, uint64_t params, const float* grads);  /* tier.hpp:204 */
int tfg_tier_read_grads(tfg_tier* tier, uint32_t id, uint64_t params, float* grads);         /* tier.hpp:209 */
int tfg_tier_has_subgroup(tfg_tier* tier, uint32_t id, int* out);                            /* tier.hpp:214 */
int tfg_tier_remove_subgroup(tfg_tier* tier, uint32_t id);                                   /* tier.hpp:216 */
int tfg_tier_probe(tfg_tier* tier, uint64_t probe_bytes, int repetitions, double* read_bw, double* write_bw,
                   int* low_confidence);                                                     /* tier.hpp:223 */
int tfg_tier_available_bytes(tfg_tier* tier, uint64_t* out);                                 /* tier.hpp:244 */

/* TierLockGuard, tier_lock.hpp:36-106: acquire returns an opaque token. */
/* TokenBucket (token_bucket.hpp:23-70): byte-rate pacing, served by the
   library's device pacer (a virtual-clock schedule with the bucket's 1 ms
   burst). TFG_CONFIG_ERROR for a rate <= 0. */
typedef struct tfg_pacer tfg_pacer;
int tfg_pacer_create(double bytes_per_second, tfg_pacer** out);
int tfg_pacer_destroy(tfg_pacer* pacer);
int tfg_pacer_set_rate(tfg_pacer* pacer, double bytes_per_second);
int tfg_pacer_rate(tfg_pacer* pacer, double* out);
int tfg_pacer_acquire(tfg_pacer* pacer, double bytes);          /* blocks until the bytes are due */
/* v1 subgroup file header (tier.hpp:92-134): encode the 32 bytes from the
   fields, decode them back, validate against an expected id and size
   (TFG_FORMAT_ERROR with the reference's messages). */
typedef struct tfg_file_header {
    uint32_t magic;
    uint16_t version;
    uint16_t element_kind;
    uint32_t subgroup_id;
    uint64_t param_count;
} tfg_file_header;
int tfg_file_header_encode(const tfg_file_header* h, uint8_t out[32]);
int tfg_file_header_decode(const uint8_t in[32], tfg_file_header* out);
int tfg_file_header_validate(const tfg_file_header* h, uint32_t expected_id, uint64_t expected_params);
/* subgroup_file_name (tier.hpp:136-140) into out (>= 32 bytes). */
int tfg_subgroup_file_name(uint32_t id, char* out, uint64_t out_len);
int tfg_tier_lock_acquire(const char* lock_dir, int tier, int worker, tfg_trace* trace, int width, void** token);
int tfg_tier_lock_release(void* token);

/* ---- engine (OffloadWorker, scheduler.hpp:286-864) ------------------------ */
int tfg_engine_create(int worker_id, tfg_tier* const* tiers, int n_tiers, const tfg_schedule_options* options,
                      const tfg_adam_hyper* hyper, tfg_trace* trace, const tfg_device_options* device,
                      tfg_engine** out);                                                    /* :288-304 */
int tfg_engine_destroy(tfg_engine* engine);
int tfg_engine_set_alpha(tfg_engine* engine, double alpha);                                 /* :315 */
int tfg_engine_set_fixed_ratio(tfg_engine* engine, const double* ratio, int n);             /* :322 */
/* ScheduleOptions::cache_slots (scheduler.hpp:44-49) for the following phases;
 * between phases only. HBM cache mode: at most the buffers allocated at init. */
int tfg_engine_set_cache_slots(tfg_engine* engine, int cache_slots);
int tfg_engine_add_subgroup(tfg_engine* engine, uint32_t id, uint64_t param_count);         /* :324 */
int tfg_engine_init_and_flush_all(tfg_engine* engine, uint64_t seed);                       /* :339 */
int tfg_engine_run_backward_sim(tfg_engine* engine, int iteration, uint64_t seed, int accum_steps); /* :365 */
int tfg_engine_gradients_finite(tfg_engine* engine, int* out);                              /* :395 */
int tfg_engine_grad_buffer(tfg_engine* engine, uint32_t id, void** device_ptr);             /* :401 */
int tfg_engine_bind_grad_buffer(tfg_engine* engine, uint32_t id, void* device_ptr);
/* The CUDA stream that produces the gradients (backward, reduce-scatter).
 * run_update and gradients_finite order the engine's streams after the work
 * queued on it at call time, so no host sync is needed between producing the
 * gradients and the update. NULL (the default) = the legacy default stream.
 * (No reference counterpart: the reference's gradients are host memory.) */
int tfg_engine_set_producer_stream(tfg_engine* engine, void* stream);
/* Data-parallel reduction in the engine: the update of `id` consumes the fp32
 * sum (in order, rounded once to grad_kind) of n (1..8) 16-bit device
 * buffers, e.g. every peer's contribution mapped over NVLink (CUDA IPC). Each
 * phase's gradient check reads every source once, writes the rounded sum to
 * the subgroup's own buffer and counts non-finite results (a sum that
 * overflows rejects the phase before any state moves); the update reads the
 * reduced buffer: 2(N-1) B/param over NVLink. Replaces the
 * reduce_grads_to_owners step in front of run_update.
 * TFG_ERR_CONFIG in the baseline gradient flow (skip_gradients = 0) and with
 * host_grads. */
int tfg_engine_bind_grad_sources(tfg_engine* engine, uint32_t id, const void* const* device_ptrs, int n);
int tfg_engine_params16_buffer(tfg_engine* engine, uint32_t id, void** device_ptr);         /* shadow_, :861 */
int tfg_engine_run_update(tfg_engine* engine, int iteration, tfg_phase_stats* stats);      /* :405 */
int tfg_engine_last_subgroup_io(tfg_engine* engine, tfg_subgroup_io* out, uint64_t max_n, uint64_t* n_out);
int tfg_engine_last_timeline(tfg_engine* engine, tfg_device_span* out, uint64_t max_n, uint64_t* n_out);
int tfg_engine_wait_host_resident(tfg_engine* engine, uint32_t id, int* slot_out);         /* :514 */
/* enqueue_* return a ticket (0 = cache hit, nothing queued) to wait on. */
int tfg_engine_enqueue_prefetch(tfg_engine* engine, uint32_t id, uint64_t* ticket_out);    /* :563 */
int tfg_engine_enqueue_flush(tfg_engine* engine, uint32_t id, int dest, uint64_t* ticket_out); /* :553 */
int tfg_engine_wait_ticket(tfg_engine* engine, uint64_t ticket, uint64_t* bytes_out, double* seconds_out);
int tfg_engine_read_state(tfg_engine* engine, uint32_t id, float* out_3n);                  /* :611 */
int tfg_engine_read_params16(tfg_engine* engine, uint32_t id, uint16_t* out_n);
int tfg_engine_read_grads16(tfg_engine* engine, uint32_t id, uint16_t* out_n);              /* grad_buffer(id).values(), :401 */
/* Writes a host array back into the subgroup's 16-bit gradient buffer (a
   caller that edited grad_buffer(id).mutable_values(), :401). */
int tfg_engine_write_grads16(tfg_engine* engine, uint32_t id, const uint16_t* in_n);
int tfg_engine_meta(tfg_engine* engine, uint32_t id, tfg_subgroup_meta* out);               /* :587 */
int tfg_engine_residency_census(tfg_engine* engine, uint64_t* host_params, uint64_t* per_tier, int n_tiers); /* :597 */
int tfg_engine_current_order(tfg_engine* engine, uint32_t* out, int max_n, int* n_out);     /* :582 */
int tfg_engine_estimates(tfg_engine* engine, double* read_bw, double* write_bw, int n_tiers); /* :583 */
int tfg_engine_pool_state(tfg_engine* engine, int slot, int* state_out, uint32_t* owner_out);

/* ---- host-side reference API --------------------------------------------
 * The reference's own C++ calls on host spans, served by the B200 objects and
 * sm_100a kernels (host arrays staged through HBM: H2D, one kernel, D2H).
 * include/tierflow_compat/ builds the reference's header API on these, so the
 * reference's scheduler / optimizer suites compile against this library with
 * only the include path changed (tests/dropin/). */
int tfg_now_ns(int64_t* out);                                                                /* common.hpp:21-26 */
int tfg_upscale16_host(const uint16_t* src, float* dst, uint64_t n, int dtype, int* all_finite); /* precision.hpp:17 */
int tfg_downscale16_host(const float* src, uint16_t* dst, uint64_t n, int dtype, uint64_t* overflows); /* precision.hpp:29 */
/* One-value f16_to_f32 / f32_to_f16 (fp16.hpp:21-88), bf16 alike: the
   kernels' codec run on the host (a scalar is not worth a device trip). */
int tfg_f16_to_f32(uint16_t h, int dtype, float* out);
int tfg_f32_to_f16(float x, int dtype, uint16_t* out);
/* GradBufferF16::accumulate (precision.hpp:66-75) on host arrays: acc[i] =
   narrow(widen(acc[i]) + widen(grads[i])) in fp32, staged through HBM (the
   reduce kernel with two sources). */
int tfg_accumulate16_host(uint16_t* acc, const uint16_t* grads, uint64_t n, int dtype);
/* adam_step(StateView, span<const float> g, hyper, t), optimizer.hpp:116-157: TFG_ERROR for t < 1,
 * TFG_CONFIG_ERROR for bad hyperparameters, TFG_GRADIENT_OVERFLOW (arrays untouched) on a
 * non-finite gradient. */
int tfg_adam_step_host(float* p, float* m, float* v, const float* g, uint64_t n, const tfg_adam_hyper* hyper,
                       uint64_t t);

/* HostBufferPool, pool.hpp:35-161: slots of 3*max_params fp32 state plus a max_params fp32 gradient
 * annex; the slot state machine of the engine (free -> prefetching -> cached -> updating -> cached
 * -> flushing -> free); illegal transitions fail with TFG_ERROR. */
typedef struct tfg_pool tfg_pool;
enum {
    TFG_POOL_PREFETCH_DONE = 0,
    TFG_POOL_BEGIN_UPDATE = 1,
    TFG_POOL_END_UPDATE = 2,
    TFG_POOL_BEGIN_FLUSH = 3,
    TFG_POOL_FLUSH_DONE = 4,
    TFG_POOL_EVICT = 5
};
int tfg_pool_create(int slots, uint64_t max_params, tfg_pool** out);                        /* pool.hpp:37-45 */
int tfg_pool_destroy(tfg_pool* pool);
int tfg_pool_slot_count(tfg_pool* pool, int* out);
int tfg_pool_try_reserve(tfg_pool* pool, uint32_t owner, int* slot_out);                    /* pool.hpp:52-62 */
int tfg_pool_find_cached(tfg_pool* pool, uint32_t owner, int* slot_out);
int tfg_pool_transition(tfg_pool* pool, int slot, int op);                                   /* pool.hpp:72-85 */
int tfg_pool_query(tfg_pool* pool, int slot, int* state_out, uint32_t* owner_out);         /* state: tfg SlotState order */
/* which 0: the slot's P||m||v (3*params floats), 1: its fp32 gradient annex (params floats);
 * TFG_ERROR when params exceeds the slot capacity (pool.hpp:123-131). */
int tfg_pool_span(tfg_pool* pool, int slot, uint64_t params, int which, float** ptr_out, uint64_t* len_out);

/* Subgroup residency transitions, optimizer.hpp:47-72 (TFG_ERROR on an illegal one). */
enum { TFG_SG_BEGIN_FLUSH = 0, TFG_SG_FINISH_FLUSH = 1, TFG_SG_BEGIN_PREFETCH = 2, TFG_SG_FINISH_PREFETCH = 3 };
int tfg_subgroup_step(tfg_subgroup_meta* sg, int op, int arg);

#ifdef __cplusplus
}
#endif

#endif /* TIERFLOW_B200_H */
