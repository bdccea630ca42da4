"""ctypes binding of the C ABI (include/tierflow_b200.h).

Loads paper_2509_02480_b200/lib/libtierflow_b200.so — the in-tree sm_100a
build — and fails loudly if it is missing: there is no CPU fallback for the
update path. Status codes become the reference's exception classes
(reference proj/include/tierflow/common.hpp:36-78).
"""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libtierflow_b200.so"
TUNING_PATH = Path(__file__).resolve().parent / "lib" / "libtierflow_b200_tuning.so"
MAX_TIERS = 8

TFG_F16, TFG_BF16 = 0, 1
LOCAL_DIR, REMOTE_DIR, MEM_THROTTLED, HOST_DRAM = 0, 1, 2, 3


class Error(RuntimeError):
    """tierflow::Error"""


class IoError(Error):
    """tierflow::IoError — storage backend failure."""


class FormatError(Error):
    """tierflow::FormatError — malformed subgroup file."""


class ConfigError(Error):
    """tierflow::ConfigError — bad configuration."""


class PlacementInconsistencyError(Error):
    """tierflow::PlacementInconsistencyError — read of an absent subgroup."""


class SchedulingBugError(Error):
    """tierflow::SchedulingBugError — the pipeline watchdog fired."""


class GradientOverflowError(Error):
    """tierflow::GradientOverflowError — non-finite gradients."""


class CudaError(Error):
    """CUDA runtime failure."""


_ERRORS = {1: Error, 2: IoError, 3: FormatError, 4: ConfigError, 5: PlacementInconsistencyError,
           6: SchedulingBugError, 7: GradientOverflowError, 8: CudaError}


class AdamHyperC(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("weight_decay", C.c_double)]


class TierSpecC(C.Structure):
    _fields_ = [("tier_id", C.c_int32), ("kind", C.c_int32), ("root", C.c_char_p), ("read_bw", C.c_double),
                ("write_bw", C.c_double), ("io_parallelism", C.c_int32), ("persistent", C.c_int32),
                ("lock_width", C.c_int32), ("direct_io", C.c_int32), ("lock_device", C.c_int32),
                ("capacity_bytes", C.c_uint64)]


class ScheduleOptionsC(C.Structure):
    _fields_ = [("pool_slots", C.c_int32), ("cache_slots", C.c_int32), ("enable_caching", C.c_int32),
                ("skip_gradients", C.c_int32), ("atomic_rw", C.c_int32), ("multi_path", C.c_int32),
                ("lock_dir", C.c_char_p), ("update_threads", C.c_int32), ("deadlock_timeout_s", C.c_double),
                ("update_pad_ns", C.c_uint64)]


class DeviceOptionsC(C.Structure):
    _fields_ = [("device", C.c_int32), ("grad_dtype", C.c_int32), ("param_dtype", C.c_int32),
                ("device_buffers", C.c_int32), ("zero_copy", C.c_int32), ("d2h_split", C.c_int32),
                ("hbm_retain", C.c_int32), ("h2d_split", C.c_int32), ("hbm_cache_slots", C.c_int32),
                ("host_grads", C.c_int32)]


class TierObservationC(C.Structure):
    _fields_ = [("read_transfers", C.c_uint64), ("read_bytes", C.c_double), ("read_seconds", C.c_double),
                ("write_transfers", C.c_uint64), ("write_bytes", C.c_double), ("write_seconds", C.c_double)]


class SubgroupIoC(C.Structure):
    _fields_ = [("id", C.c_uint32), ("fetched", C.c_uint32), ("flushed", C.c_uint32), ("pad", C.c_uint32),
                ("state_bytes", C.c_uint64), ("read_seconds", C.c_double), ("write_seconds", C.c_double)]


class PhaseStatsC(C.Structure):
    _fields_ = [("wall_seconds", C.c_double), ("params_updated", C.c_uint64), ("cache_hits", C.c_uint64),
                ("downscale_overflows", C.c_uint64), ("retained", C.c_int32), ("n_tiers", C.c_int32),
                ("flush_allocation", C.c_int32 * MAX_TIERS), ("tier_obs", TierObservationC * MAX_TIERS),
                ("n_subgroup_io", C.c_uint64), ("device_seconds", C.c_double), ("kernel_seconds", C.c_double),
                ("h2d_seconds", C.c_double), ("d2h_seconds", C.c_double), ("h2d_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64)]


class EventC(C.Structure):
    _fields_ = [("timestamp_ns", C.c_int64), ("worker_id", C.c_int32), ("kind", C.c_int32),
                ("subgroup_id", C.c_int64), ("tier_id", C.c_int32), ("pad", C.c_int32), ("bytes", C.c_uint64)]


class DeviceSpanC(C.Structure):
    _fields_ = [("id", C.c_uint32), ("h2d_start", C.c_float), ("h2d_end", C.c_float), ("k_start", C.c_float),
                ("k_end", C.c_float), ("d2h_end", C.c_float), ("host_resident", C.c_float),
                ("host_retired", C.c_float), ("d2h_start", C.c_float)]


class SubgroupMetaC(C.Structure):
    _fields_ = [("id", C.c_uint32), ("residency", C.c_int32), ("tier", C.c_int32), ("slot", C.c_int32),
                ("param_count", C.c_uint64), ("step_count", C.c_uint64)]


_vp = C.c_void_p
_u64 = C.c_uint64
_i = C.c_int
_d = C.c_double
_SIGS = {
    "tfg_last_error": (C.c_char_p, []),
    "tfg_abi_version": (_i, []),
    "tfg_device_count": (_i, [C.POINTER(_i)]),
    "tfg_device_alloc": (_i, [_i, _u64, C.POINTER(_vp)]),
    "tfg_device_free": (_i, [_i, _vp]),
    "tfg_ipc_get_handle": (_i, [_i, _vp, C.c_char_p]),
    "tfg_ipc_open_handle": (_i, [_i, C.c_char_p, C.POINTER(_vp)]),
    "tfg_ipc_close_handle": (_i, [_i, _vp]),
    "tfg_adam_fused": (_i, [_vp, _vp, _vp, _vp, _i, _vp, _i, _u64, C.POINTER(AdamHyperC), _u64, _vp, _vp]),
    "tfg_adam_fused_contiguous": (_i, [_vp, _u64, _vp, _i, _vp, _i, C.POINTER(AdamHyperC), _u64, _vp, _vp]),
    "tfg_adam_fused_gated": (_i, [_vp, _vp, _vp, _vp, _i, _vp, _i, _u64, C.POINTER(AdamHyperC), _u64, _vp, _vp, _vp]),
    "tfg_adam_fused_multi": (_i, [_vp, _vp, _vp, C.POINTER(_vp), _i, _i, _vp, _i, _u64, C.POINTER(AdamHyperC), _u64,
                                  _vp, _vp]),
    "tfg_adam_step": (_i, [_vp, _vp, _vp, _vp, _i, _vp, _i, _u64, C.POINTER(AdamHyperC), _u64,
                           C.POINTER(_u64), _vp]),
    "tfg_selftest_div_const": (_i, [_d, _u64, _u64, _i, _i, C.POINTER(_u64), C.POINTER(_d)]),
    "tfg_upscale16": (_i, [_vp, _vp, _u64, _i, _vp, _vp]),
    "tfg_downscale16": (_i, [_vp, _vp, _u64, _i, _vp, _vp]),
    "tfg_count_nonfinite16": (_i, [_vp, _u64, _i, _vp, _vp]),
    "tfg_synthetic_grads": (_i, [_vp, _u64, _i, _u64, C.c_uint32, _i, _i, _i, _vp]),
    "tfg_synthetic_state": (_i, [_vp, _vp, _vp, _u64, _u64, C.c_uint32, _vp]),
    "tfg_assign_subgroups": (_i, [_i, C.POINTER(_d), _i, C.POINTER(_i)]),
    "tfg_host_blocks_live": (_i, [C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "tfg_assign_subgroups_capped": (_i, [_i, C.POINTER(_d), C.POINTER(_i), _i, C.POINTER(_i)]),
    "tfg_destination_plan": (_i, [C.POINTER(C.c_uint32), _i, _i, C.POINTER(_d), _i, C.POINTER(_i), C.POINTER(_i),
                                  C.POINTER(_i)]),
    "tfg_update_order": (_i, [_i, C.POINTER(C.c_uint32), _i, _i, C.POINTER(C.c_uint32)]),
    "tfg_retention_capacity": (_i, [_i, _i, _i, _i, C.POINTER(_i)]),
    "tfg_update_bandwidth_estimates": (_i, [C.POINTER(_d), C.POINTER(_d), C.POINTER(_u64), _i, _d,
                                            C.POINTER(TierObservationC), _i]),
    "tfg_trace_create": (_i, [C.POINTER(_vp)]),
    "tfg_trace_destroy": (_i, [_vp]),
    "tfg_trace_size": (_i, [_vp, C.POINTER(_u64)]),
    "tfg_trace_copy": (_i, [_vp, _u64, C.POINTER(EventC), _u64, C.POINTER(_u64)]),
    "tfg_trace_record": (_i, [_vp, _i, _i, C.c_int64, _i, _u64]),
    "tfg_trace_record_at": (_i, [_vp, C.c_int64, _i, _i, C.c_int64, _i, _u64]),
    "tfg_trace_write": (_i, [_vp, C.c_char_p]),
    "tfg_trace_clear": (_i, [_vp]),
    "tfg_tier_create": (_i, [C.POINTER(TierSpecC), C.POINTER(_vp)]),
    "tfg_tier_destroy": (_i, [_vp]),
    "tfg_tier_bandwidths": (_i, [_vp, C.POINTER(_d), C.POINTER(_d)]),
    "tfg_tier_set_throttle_rates": (_i, [_vp, _d, _d]),
    "tfg_tier_write_subgroup": (_i, [_vp, C.c_uint32, _u64, _vp, C.POINTER(_u64), C.POINTER(_d)]),
    "tfg_tier_read_subgroup": (_i, [_vp, C.c_uint32, _u64, _vp, C.POINTER(_u64), C.POINTER(_d)]),
    "tfg_tier_write_grads": (_i, [_vp, C.c_uint32, _u64, _vp]),
    "tfg_tier_read_grads": (_i, [_vp, C.c_uint32, _u64, _vp]),
    "tfg_tier_has_subgroup": (_i, [_vp, C.c_uint32, C.POINTER(_i)]),
    "tfg_tier_remove_subgroup": (_i, [_vp, C.c_uint32]),
    "tfg_tier_probe": (_i, [_vp, _u64, _i, C.POINTER(_d), C.POINTER(_d), C.POINTER(_i)]),
    "tfg_tier_available_bytes": (_i, [_vp, C.POINTER(_u64)]),
    "tfg_pacer_create": (_i, [C.c_double, C.POINTER(_vp)]),
    "tfg_pacer_destroy": (_i, [_vp]),
    "tfg_pacer_set_rate": (_i, [_vp, C.c_double]),
    "tfg_pacer_rate": (_i, [_vp, C.POINTER(C.c_double)]),
    "tfg_pacer_acquire": (_i, [_vp, C.c_double]),
    "tfg_file_header_encode": (_i, [_vp, _vp]),
    "tfg_file_header_decode": (_i, [_vp, _vp]),
    "tfg_file_header_validate": (_i, [_vp, C.c_uint32, _u64]),
    "tfg_subgroup_file_name": (_i, [C.c_uint32, C.c_char_p, _u64]),
    "tfg_tier_lock_acquire": (_i, [C.c_char_p, _i, _i, _vp, _i, C.POINTER(_vp)]),
    "tfg_tier_lock_release": (_i, [_vp]),
    "tfg_engine_create": (_i, [_i, C.POINTER(_vp), _i, C.POINTER(ScheduleOptionsC), C.POINTER(AdamHyperC), _vp,
                               C.POINTER(DeviceOptionsC), C.POINTER(_vp)]),
    "tfg_engine_destroy": (_i, [_vp]),
    "tfg_engine_set_alpha": (_i, [_vp, _d]),
    "tfg_engine_set_fixed_ratio": (_i, [_vp, C.POINTER(_d), _i]),
    "tfg_engine_set_cache_slots": (_i, [_vp, _i]),
    "tfg_engine_add_subgroup": (_i, [_vp, C.c_uint32, _u64]),
    "tfg_engine_init_and_flush_all": (_i, [_vp, _u64]),
    "tfg_engine_run_backward_sim": (_i, [_vp, _i, _u64, _i]),
    "tfg_engine_gradients_finite": (_i, [_vp, C.POINTER(_i)]),
    "tfg_engine_grad_buffer": (_i, [_vp, C.c_uint32, C.POINTER(_vp)]),
    "tfg_engine_bind_grad_buffer": (_i, [_vp, C.c_uint32, _vp]),
    "tfg_engine_set_producer_stream": (_i, [_vp, _vp]),
    "tfg_engine_bind_grad_sources": (_i, [_vp, C.c_uint32, C.POINTER(_vp), C.c_int]),
    "tfg_engine_params16_buffer": (_i, [_vp, C.c_uint32, C.POINTER(_vp)]),
    "tfg_engine_run_update": (_i, [_vp, _i, C.POINTER(PhaseStatsC)]),
    "tfg_engine_last_subgroup_io": (_i, [_vp, C.POINTER(SubgroupIoC), _u64, C.POINTER(_u64)]),
    "tfg_engine_last_timeline": (_i, [_vp, C.POINTER(DeviceSpanC), _u64, C.POINTER(_u64)]),
    "tfg_engine_wait_host_resident": (_i, [_vp, C.c_uint32, C.POINTER(_i)]),
    "tfg_engine_enqueue_prefetch": (_i, [_vp, C.c_uint32, C.POINTER(_u64)]),
    "tfg_engine_enqueue_flush": (_i, [_vp, C.c_uint32, _i, C.POINTER(_u64)]),
    "tfg_engine_wait_ticket": (_i, [_vp, _u64, C.POINTER(_u64), C.POINTER(_d)]),
    "tfg_engine_read_state": (_i, [_vp, C.c_uint32, _vp]),
    "tfg_engine_read_params16": (_i, [_vp, C.c_uint32, _vp]),
    "tfg_engine_read_grads16": (_i, [_vp, C.c_uint32, _vp]),
    "tfg_engine_write_grads16": (_i, [_vp, C.c_uint32, _vp]),
    "tfg_now_ns": (_i, [C.POINTER(C.c_int64)]),
    "tfg_upscale16_host": (_i, [_vp, _vp, _u64, _i, C.POINTER(_i)]),
    "tfg_downscale16_host": (_i, [_vp, _vp, _u64, _i, C.POINTER(_u64)]),
    "tfg_accumulate16_host": (_i, [_vp, _vp, _u64, _i]),
    "tfg_f16_to_f32": (_i, [C.c_uint16, _i, C.POINTER(C.c_float)]),
    "tfg_f32_to_f16": (_i, [C.c_float, _i, C.POINTER(C.c_uint16)]),
    "tfg_adam_step_host": (_i, [_vp, _vp, _vp, _vp, _u64, C.POINTER(AdamHyperC), _u64]),
    "tfg_pool_create": (_i, [_i, _u64, C.POINTER(_vp)]),
    "tfg_pool_destroy": (_i, [_vp]),
    "tfg_pool_slot_count": (_i, [_vp, C.POINTER(_i)]),
    "tfg_pool_try_reserve": (_i, [_vp, C.c_uint32, C.POINTER(_i)]),
    "tfg_pool_find_cached": (_i, [_vp, C.c_uint32, C.POINTER(_i)]),
    "tfg_pool_transition": (_i, [_vp, _i, _i]),
    "tfg_pool_query": (_i, [_vp, _i, C.POINTER(_i), C.POINTER(C.c_uint32)]),
    "tfg_pool_span": (_i, [_vp, _i, _u64, _i, C.POINTER(_vp), C.POINTER(_u64)]),
    "tfg_subgroup_step": (_i, [C.POINTER(SubgroupMetaC), _i, _i]),
    "tfg_engine_meta": (_i, [_vp, C.c_uint32, C.POINTER(SubgroupMetaC)]),
    "tfg_engine_residency_census": (_i, [_vp, C.POINTER(_u64), C.POINTER(_u64), _i]),
    "tfg_engine_current_order": (_i, [_vp, C.POINTER(C.c_uint32), _i, C.POINTER(_i)]),
    "tfg_engine_estimates": (_i, [_vp, C.POINTER(_d), C.POINTER(_d), _i]),
    "tfg_engine_pool_state": (_i, [_vp, _i, C.POINTER(_i), C.POINTER(C.c_uint32)]),
}

# include/tierflow_b200_tuning.h (the kernel variants; a separate library)
_TUNING_SIGS = {
    "tfg_adam_variant_count": (_i, [C.POINTER(_i)]),
    "tfg_adam_fused_variant": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _u64, C.POINTER(AdamHyperC), _u64, _vp, _vp]),
    "tfg_adam_fused_multi_variant": (_i, [_i, _vp, _vp, _vp, C.POINTER(_vp), _i, _vp, _u64, C.POINTER(AdamHyperC),
                                          _u64, _vp, _vp]),
    "tfg_selftest_fast_step": (_i, [_u64, _u64, C.POINTER(_d), C.POINTER(_u64)]),
    "tfg_selftest_fast_rn": (_i, [_u64, _u64, C.POINTER(_u64)]),
}

_lock = threading.Lock()
_LIB: C.CDLL | None = None
_TUNING: C.CDLL | None = None


def load() -> C.CDLL:
    """The loaded library. Raises if the in-tree build is missing."""
    global _LIB
    with _lock:
        if _LIB is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} is not built; run `python -m paper_2509_02480_b200.build` "
                    "(the update path has no CPU fallback)")
            lib = C.CDLL(str(LIB_PATH))
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _LIB = lib
        return _LIB


def load_tuning() -> C.CDLL:
    """The tuning library (kernel variants), loaded only by sweeps and tests."""
    global _TUNING
    lib = load()
    with _lock:
        if _TUNING is None:
            if not TUNING_PATH.exists():
                raise ImportError(f"{TUNING_PATH} is not built; run `python -m paper_2509_02480_b200.build`")
            t = C.CDLL(str(TUNING_PATH))
            for name, (res, args) in _TUNING_SIGS.items():
                fn = getattr(t, name)
                fn.restype = res
                fn.argtypes = args
            _TUNING = t
        del lib
        return _TUNING


def call_tuning(name: str, *args) -> None:
    check(getattr(load_tuning(), name)(*args))


def check(rc: int) -> None:
    if rc != 0:
        msg = load().tfg_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, Error)(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def exported_symbols() -> list[str]:
    return list(_SIGS)
