"""Python mirror of the reference engine API over the C ABI.

Names, argument meaning and error behaviour follow the reference C++ API
(reference proj/include/tierflow/*.hpp) so tests read like the reference's
own: Tier / TierSpec (tier.hpp:43-241), EventTrace (trace.hpp:77-171),
ScheduleOptions / OffloadWorker / PhaseStats (scheduler.hpp:32-864),
assign_subgroups / DestinationPlan / update_bandwidth_estimates
(placement.hpp:30-225), adam_step (optimizer.hpp:116), upscale/downscale
(precision.hpp:17-37). Device arrays are torch CUDA tensors (plumbing only —
the arithmetic runs in the sm_100a kernels of libtierflow_b200.so).
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (ConfigError, CudaError, Error, FormatError, GradientOverflowError, IoError,  # noqa: F401
                   PlacementInconsistencyError, SchedulingBugError, TFG_BF16, TFG_F16)

F16, BF16 = TFG_F16, TFG_BF16


class TierKind(enum.IntEnum):
    local_dir = 0
    remote_dir = 1
    mem_throttled = 2
    host_dram = 3


class EventKind(enum.IntEnum):
    prefetch_start = 0
    prefetch_end = 1
    update_start = 2
    update_end = 3
    flush_start = 4
    flush_end = 5
    lock_acquire = 6
    lock_release = 7
    h2d_start = 8
    h2d_end = 9
    grad_upscale_start = 10
    grad_upscale_end = 11
    cache_hit = 12


class Residency(enum.IntEnum):
    host_cached = 0
    in_flight = 1
    on_tier = 2


class SlotState(enum.IntEnum):
    free_slot = 0
    prefetching = 1
    updating = 2
    flushing = 3
    cached = 4


@dataclass
class IoStats:
    bytes: int = 0
    seconds: float = 0.0

    def bytes_per_second(self) -> float:
        return self.bytes / self.seconds if self.seconds > 0 else 0.0


@dataclass
class AdamHyper:
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0

    def c(self) -> _lib.AdamHyperC:
        return _lib.AdamHyperC(self.lr, self.beta1, self.beta2, self.eps, self.weight_decay)


@dataclass
class TierSpec:
    tier_id: int = 0
    kind: TierKind = TierKind.local_dir
    root: str = ""
    read_bw: float = 0.0
    write_bw: float = 0.0
    io_parallelism: int = 1
    persistent: bool = False
    lock_width: int = 1
    direct_io: bool = True
    # 0: own semaphore (reference); k > 0: shared by all tiers with the same k
    # (one physical device)
    lock_device: int = 0
    # 0: unlimited (reference); else the state bytes the tier may hold
    capacity_bytes: int = 0


@dataclass
class ProbeResult:
    read_bw: float
    write_bw: float
    low_confidence: bool


@dataclass
class ScheduleOptions:
    pool_slots: int = 4
    cache_slots: int = -1
    enable_caching: bool = True
    skip_gradients: bool = True
    atomic_rw: bool = True
    multi_path: bool = True
    lock_dir: str = ""
    update_threads: int = 1
    deadlock_timeout_s: float = 30.0
    update_pad_ns: int = 0

    def retention_capacity(self, subgroup_count: int) -> int:
        return retention_capacity(self.enable_caching, self.pool_slots, self.cache_slots, subgroup_count)

    def c(self) -> _lib.ScheduleOptionsC:
        return _lib.ScheduleOptionsC(self.pool_slots, self.cache_slots, int(self.enable_caching),
                                     int(self.skip_gradients), int(self.atomic_rw), int(self.multi_path),
                                     self.lock_dir.encode() if self.lock_dir else None, self.update_threads,
                                     self.deadlock_timeout_s, self.update_pad_ns)


@dataclass
class DeviceOptions:
    device: int = 0
    grad_dtype: int = F16
    param_dtype: int = F16
    device_buffers: int = 3
    # 0: copy engines both ways through the device ring; 1: the kernel streams
    # the pinned slot over PCIe both ways; 2: DMA in, kernel epilogue writes back.
    zero_copy: int = 0
    d2h_split: int = 1
    # Retained subgroups keep their updated state in HBM between phases.
    # 1: their host slot stays reserved (C = min(cache_slots, pool_slots - 3));
    # 2: HBM cache, the slot streams again and C = cache_slots.
    hbm_retain: int = 1
    # concurrent H2D copy streams per subgroup (1 or 2)
    h2d_split: int = 1
    # hbm_retain 2: HBM buffers for retained subgroups (0: all of C); fewer
    # gives a two-level cache, the rest retained in host slots
    hbm_cache_slots: int = 0
    # 16-bit gradients / working params in pinned host memory, streamed with the state
    host_grads: bool = False


@dataclass
class Event:
    timestamp_ns: int
    worker_id: int
    kind: EventKind
    subgroup_id: int
    tier_id: int
    bytes: int


@dataclass
class TierObservation:
    read_transfers: int = 0
    read_bytes: float = 0.0
    read_seconds: float = 0.0
    write_transfers: int = 0
    write_bytes: float = 0.0
    write_seconds: float = 0.0


@dataclass
class SubgroupIoTimes:
    id: int
    state_bytes: int
    read_seconds: float
    write_seconds: float
    fetched: bool
    flushed: bool


@dataclass
class PhaseStats:
    wall_seconds: float = 0.0
    params_updated: int = 0
    cache_hits: int = 0
    downscale_overflows: int = 0
    retained: int = 0
    flush_allocation: list = field(default_factory=list)
    tier_obs: list = field(default_factory=list)
    subgroup_io: list = field(default_factory=list)
    device_seconds: float = 0.0
    kernel_seconds: float = 0.0
    h2d_seconds: float = 0.0
    d2h_seconds: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0


@dataclass
class SubgroupMeta:
    id: int
    residency: Residency
    tier: int
    slot: int
    param_count: int
    step_count: int


@dataclass
class SyntheticGradSource:
    """Seeded gradient generator (scheduler.hpp:85-102); the engine realises it on the GPU."""
    seed: int = 42


def _as_f32(a: np.ndarray) -> np.ndarray:
    if not (isinstance(a, np.ndarray) and a.dtype == np.float32 and a.flags.c_contiguous):
        raise ConfigError("expected a C-contiguous float32 numpy array")
    return a


# ---------------------------------------------------------------------------
# Placement (host, pure)


@dataclass
class AllocationVector:
    counts: list
    total: int


def assign_subgroups(M: int, bandwidths: Sequence[float]) -> AllocationVector:
    n = len(bandwidths)
    bw = (C.c_double * max(n, 1))(*bandwidths)
    out = (C.c_int * max(n, 1))()
    _lib.call("tfg_assign_subgroups", M, bw, n, out)
    return AllocationVector(list(out)[:n], M)


def host_blocks_live() -> tuple:
    """(blocks, bytes) of host blocks alive in the process (leak accounting)."""
    b, n, f = C.c_int64(), C.c_int64(), C.c_int64()
    _lib.call("tfg_host_blocks_live", C.byref(b), C.byref(n), C.byref(f))
    return b.value, n.value


def host_block_free_failures() -> int:
    """cudaFreeHost calls that failed (pinned memory the process could not return)."""
    b, n, f = C.c_int64(), C.c_int64(), C.c_int64()
    _lib.call("tfg_host_blocks_live", C.byref(b), C.byref(n), C.byref(f))
    return f.value


def assign_subgroups_capped(M: int, bandwidths: Sequence[float], caps: Sequence[int]) -> AllocationVector:
    """Capacity-aware Eq. 1 (caps[i] < 0: unlimited); the reference allocation
    whenever it fits every cap."""
    n = len(bandwidths)
    if len(caps) != n:
        raise ConfigError("one cap per tier")
    bw = (C.c_double * max(n, 1))(*bandwidths)
    cp = (C.c_int * max(n, 1))(*caps)
    out = (C.c_int * max(n, 1))()
    _lib.call("tfg_assign_subgroups_capped", M, bw, cp, n, out)
    return AllocationVector(list(out)[:n], M)


@dataclass
class TierAssignment:
    host_retain: bool
    tier: int


class DestinationPlan:
    def __init__(self, order: Sequence[int], capacity: int, bandwidths: Sequence[float]):
        M, n = len(order), len(bandwidths)
        o = (C.c_uint32 * max(M, 1))(*order)
        bw = (C.c_double * max(n, 1))(*bandwidths)
        retain = (C.c_int * max(M, 1))()
        tier = (C.c_int * max(M, 1))()
        alloc = (C.c_int * max(n, 1))()
        _lib.call("tfg_destination_plan", o, M, capacity, bw, n, retain, tier, alloc)
        self._map = {int(order[k]): TierAssignment(bool(retain[k]), int(tier[k])) for k in range(M)}
        self._alloc = AllocationVector(list(alloc)[:n], M - sum(retain[k] for k in range(M)))
        self._retained = sum(retain[k] for k in range(M))

    def assign_storage_tier(self, sg: int) -> TierAssignment:
        if sg not in self._map:
            raise Error(f"destination plan: unknown subgroup {sg}")
        return self._map[sg]

    def flush_allocation(self) -> AllocationVector:
        return self._alloc

    def retained_count(self) -> int:
        return self._retained


@dataclass
class UpdatePlan:
    iteration: int
    ascending: bool
    order: list

    @staticmethod
    def make(iteration: int, sorted_ids: Sequence[int], alternate: bool) -> "UpdatePlan":
        M = len(sorted_ids)
        ids = (C.c_uint32 * max(M, 1))(*sorted_ids)
        out = (C.c_uint32 * max(M, 1))()
        _lib.call("tfg_update_order", iteration, ids, M, int(alternate), out)
        return UpdatePlan(iteration, (not alternate) or iteration % 2 == 0, list(out)[:M])

    def next_after(self, sg: int) -> Optional[int]:
        for k in range(len(self.order) - 1):
            if self.order[k] == sg:
                return self.order[k + 1]
        return None


def retention_capacity(enable_caching: bool, pool_slots: int, cache_slots: int, subgroup_count: int) -> int:
    out = C.c_int()
    _lib.call("tfg_retention_capacity", int(enable_caching), pool_slots, cache_slots, subgroup_count, C.byref(out))
    return out.value


class BandwidthEstimate:
    """min(read, write) per tier with an EMA (placement.hpp:104-162)."""

    def __init__(self, read_bw: Sequence[float], write_bw: Sequence[float], alpha: float = 0.5):
        if not (alpha > 0.0) or alpha > 1.0:
            raise ConfigError("bandwidth EMA alpha must be in (0, 1]")
        self.read_bw = list(map(float, read_bw))
        self.write_bw = list(map(float, write_bw))
        self.sample_count = [0] * len(self.read_bw)
        self.alpha = alpha

    def effective(self, i: int) -> float:
        return min(self.read_bw[i], self.write_bw[i])

    def effective_all(self) -> list:
        return [self.effective(i) for i in range(len(self.read_bw))]


def update_bandwidth_estimates(est: BandwidthEstimate, observed: Sequence[TierObservation]) -> None:
    n = len(est.read_bw)
    r = (C.c_double * max(n, 1))(*est.read_bw)
    w = (C.c_double * max(n, 1))(*est.write_bw)
    s = (C.c_uint64 * max(n, 1))(*est.sample_count)
    obs = (_lib.TierObservationC * max(len(observed), 1))(
        *[_lib.TierObservationC(o.read_transfers, o.read_bytes, o.read_seconds, o.write_transfers, o.write_bytes,
                                o.write_seconds) for o in observed])
    _lib.call("tfg_update_bandwidth_estimates", r, w, s, n, est.alpha, obs, len(observed))
    est.read_bw, est.write_bw, est.sample_count = list(r)[:n], list(w)[:n], list(s)[:n]


# ---------------------------------------------------------------------------
# Trace


class EventTrace:
    def __init__(self):
        h = C.c_void_p()
        _lib.call("tfg_trace_create", C.byref(h))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:  # not during interpreter teardown
            _lib.load().tfg_trace_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def record(self, kind: int, worker: int, subgroup: int, tier: int, bytes_: int) -> None:
        _lib.call("tfg_trace_record", self._h, int(kind), worker, subgroup, tier, bytes_)

    def size(self) -> int:
        n = C.c_uint64()
        _lib.call("tfg_trace_size", self._h, C.byref(n))
        return n.value

    def snapshot(self, begin: int = 0) -> list:
        total = self.size()
        if total <= begin:
            return []
        buf = (_lib.EventC * (total - begin))()
        got = C.c_uint64()
        _lib.call("tfg_trace_copy", self._h, begin, buf, total - begin, C.byref(got))
        return [Event(e.timestamp_ns, e.worker_id, EventKind(e.kind), e.subgroup_id, e.tier_id, e.bytes)
                for e in buf[:got.value]]

    snapshot_from = snapshot

    def write(self, path: str) -> None:
        _lib.call("tfg_trace_write", self._h, os.fspath(path).encode())

    def clear(self) -> None:
        _lib.call("tfg_trace_clear", self._h)


# ---------------------------------------------------------------------------
# Tiers


class Tier:
    def __init__(self, spec: TierSpec):
        self._root = (spec.root or "").encode()
        cs = _lib.TierSpecC(spec.tier_id, int(spec.kind), self._root, spec.read_bw, spec.write_bw,
                            spec.io_parallelism, int(spec.persistent), spec.lock_width, int(spec.direct_io),
                            spec.lock_device, spec.capacity_bytes)
        h = C.c_void_p()
        _lib.call("tfg_tier_create", C.byref(cs), C.byref(h))
        self._h = h
        self._spec = spec

    def close(self) -> None:
        """Drops this handle's reference to the native tier (an engine built on
        it keeps its own); the tier's blobs are freed with the last one."""
        if getattr(self, "_h", None) and _lib is not None:  # not during interpreter teardown
            _lib.load().tfg_tier_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    @property
    def handle(self):
        return self._h

    def id(self) -> int:
        return self._spec.tier_id

    def spec(self) -> TierSpec:
        r, w = C.c_double(), C.c_double()
        _lib.call("tfg_tier_bandwidths", self._h, C.byref(r), C.byref(w))
        self._spec.read_bw, self._spec.write_bw = r.value, w.value
        return self._spec

    def set_throttle_rates(self, read_bps: float, write_bps: float) -> None:
        _lib.call("tfg_tier_set_throttle_rates", self._h, read_bps, write_bps)

    def write_subgroup(self, sg: int, params: int, state: np.ndarray) -> IoStats:
        state = _as_f32(state)
        if state.size != 3 * params:
            raise Error("write_subgroup: state length mismatch")
        b, s = C.c_uint64(), C.c_double()
        _lib.call("tfg_tier_write_subgroup", self._h, sg, params, state.ctypes.data, C.byref(b), C.byref(s))
        return IoStats(b.value, s.value)

    def read_subgroup(self, sg: int, params: int, state: np.ndarray) -> IoStats:
        state = _as_f32(state)
        if state.size != 3 * params:
            raise Error("read_subgroup: state length mismatch")
        b, s = C.c_uint64(), C.c_double()
        _lib.call("tfg_tier_read_subgroup", self._h, sg, params, state.ctypes.data, C.byref(b), C.byref(s))
        return IoStats(b.value, s.value)

    def write_grads(self, sg: int, params: int, grads: np.ndarray) -> None:
        grads = _as_f32(grads)
        if grads.size != params:
            raise Error("write_grads: length mismatch")
        _lib.call("tfg_tier_write_grads", self._h, sg, params, grads.ctypes.data)

    def read_grads(self, sg: int, params: int, grads: np.ndarray) -> None:
        grads = _as_f32(grads)
        if grads.size != params:
            raise Error("read_grads: length mismatch")
        _lib.call("tfg_tier_read_grads", self._h, sg, params, grads.ctypes.data)

    def has_subgroup(self, sg: int) -> bool:
        out = C.c_int()
        _lib.call("tfg_tier_has_subgroup", self._h, sg, C.byref(out))
        return bool(out.value)

    def remove_subgroup(self, sg: int) -> None:
        _lib.call("tfg_tier_remove_subgroup", self._h, sg)

    def probe_bandwidth(self, probe_bytes: int, repetitions: int) -> ProbeResult:
        r, w, lc = C.c_double(), C.c_double(), C.c_int()
        _lib.call("tfg_tier_probe", self._h, probe_bytes, repetitions, C.byref(r), C.byref(w), C.byref(lc))
        self._spec.read_bw, self._spec.write_bw = r.value, w.value
        return ProbeResult(r.value, w.value, bool(lc.value))

    def available_bytes(self) -> int:
        out = C.c_uint64()
        _lib.call("tfg_tier_available_bytes", self._h, C.byref(out))
        return out.value


class TierLockGuard:
    """Node-level tier semaphore (tier_lock.hpp:36-101); width 1 = exclusive flock."""

    def __init__(self, lock_dir: str, tier: int, worker: int, trace: Optional[EventTrace] = None, width: int = 1):
        tok = C.c_void_p()
        _lib.call("tfg_tier_lock_acquire", os.fspath(lock_dir).encode(), tier, worker,
                  trace.handle if trace else None, width, C.byref(tok))
        self._tok = tok

    def release(self) -> None:
        if self._tok:
            _lib.call("tfg_tier_lock_release", self._tok)
            self._tok = None

    def held(self) -> bool:
        return bool(self._tok)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.release()

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


def acquire_tier_lock(lock_dir: str, tier: int, worker: int, trace: Optional[EventTrace] = None) -> TierLockGuard:
    return TierLockGuard(lock_dir, tier, worker, trace)


def tier_lock_path(lock_dir: str, tier: int) -> str:
    return os.path.join(lock_dir, f"tier_{tier}.lock")


# ---------------------------------------------------------------------------
# Engine


class Ticket:
    """A queued transfer (the reference's shared_future<IoStats>)."""

    def __init__(self, engine: "OffloadWorker", ticket: int):
        self._e, self._t, self._result = engine, ticket, None

    def get(self) -> IoStats:
        if self._result is None:
            b, s = C.c_uint64(), C.c_double()
            _lib.call("tfg_engine_wait_ticket", self._e.handle, self._t, C.byref(b), C.byref(s))
            self._result = IoStats(b.value, s.value)
        return self._result


class OffloadWorker:
    """One update-phase engine per GPU rank (scheduler.hpp:286-864)."""

    def __init__(self, worker_id: int, tiers: Sequence[Tier], opt: ScheduleOptions, hyper: AdamHyper,
                 trace: EventTrace, device: Optional[DeviceOptions] = None):
        device = device or DeviceOptions()
        self._tiers = list(tiers)  # keep the tier handles alive
        self._trace = trace
        arr = (C.c_void_p * len(self._tiers))(*[t.handle.value for t in self._tiers])
        h = C.c_void_p()
        o, hy = opt.c(), hyper.c()
        d = _lib.DeviceOptionsC(device.device, device.grad_dtype, device.param_dtype, device.device_buffers,
                                int(device.zero_copy), device.d2h_split, int(device.hbm_retain),
                                device.h2d_split, device.hbm_cache_slots, int(device.host_grads))
        _lib.call("tfg_engine_create", worker_id, arr, len(self._tiers), C.byref(o), C.byref(hy),
                  trace.handle if trace else None, C.byref(d), C.byref(h))
        self._h = h
        self._id = worker_id
        self._opt = opt
        self._device = device
        self._params: dict[int, int] = {}

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.call("tfg_engine_destroy", self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def id(self) -> int:
        return self._id

    def options(self) -> ScheduleOptions:
        return self._opt

    def set_alpha(self, alpha: float) -> None:
        _lib.call("tfg_engine_set_alpha", self._h, alpha)

    def set_fixed_ratio(self, ratio: Sequence[float]) -> None:
        arr = (C.c_double * max(len(ratio), 1))(*ratio)
        _lib.call("tfg_engine_set_fixed_ratio", self._h, arr, len(ratio))

    def set_cache_slots(self, cache_slots: int) -> None:
        """Retention capacity C for the following phases (between phases)."""
        _lib.call("tfg_engine_set_cache_slots", self._h, cache_slots)

    def add_subgroup(self, sg: int, param_count: int) -> None:
        _lib.call("tfg_engine_add_subgroup", self._h, sg, param_count)
        self._params[sg] = param_count

    def subgroup_ids(self) -> list:
        return sorted(self._params)

    def total_params(self) -> int:
        return sum(self._params.values())

    def init_and_flush_all(self, seed: int) -> None:
        _lib.call("tfg_engine_init_and_flush_all", self._h, seed)

    def run_backward_sim(self, iteration: int, source, accum_steps: int = 1) -> None:
        seed = source.seed if hasattr(source, "seed") else int(source)
        _lib.call("tfg_engine_run_backward_sim", self._h, iteration, seed, accum_steps)

    def gradients_finite(self) -> bool:
        out = C.c_int()
        _lib.call("tfg_engine_gradients_finite", self._h, C.byref(out))
        return bool(out.value)

    def grad_buffer(self, sg: int) -> int:
        p = C.c_void_p()
        _lib.call("tfg_engine_grad_buffer", self._h, sg, C.byref(p))
        return p.value

    def bind_grad_buffer(self, sg: int, device_ptr: int) -> None:
        _lib.call("tfg_engine_bind_grad_buffer", self._h, sg, C.c_void_p(device_ptr))

    def set_producer_stream(self, stream=None) -> None:
        """The CUDA stream (torch.cuda.Stream, raw handle, or None for the
        legacy default stream) that produces the gradients: every run_update
        is ordered after the work queued on it, no host sync needed."""
        handle = getattr(stream, "cuda_stream", stream) or 0
        _lib.call("tfg_engine_set_producer_stream", self._h, C.c_void_p(handle))

    def bind_grad_sources(self, sg: int, device_ptrs) -> None:
        """Feed subgroup `sg` from the fp32 sum of several 16-bit device
        buffers (in order, rounded once): the fused reduce + update."""
        arr = (C.c_void_p * len(device_ptrs))(*device_ptrs)
        _lib.call("tfg_engine_bind_grad_sources", self._h, sg, arr, len(device_ptrs))

    def params16_buffer(self, sg: int) -> int:
        p = C.c_void_p()
        _lib.call("tfg_engine_params16_buffer", self._h, sg, C.byref(p))
        return p.value

    def run_update(self, iteration: int) -> PhaseStats:
        st = _lib.PhaseStatsC()
        _lib.call("tfg_engine_run_update", self._h, iteration, C.byref(st))
        n = st.n_tiers
        io = (_lib.SubgroupIoC * max(st.n_subgroup_io, 1))()
        got = C.c_uint64()
        _lib.call("tfg_engine_last_subgroup_io", self._h, io, st.n_subgroup_io, C.byref(got))
        return PhaseStats(
            wall_seconds=st.wall_seconds, params_updated=st.params_updated, cache_hits=st.cache_hits,
            downscale_overflows=st.downscale_overflows, retained=st.retained,
            flush_allocation=list(st.flush_allocation)[:n],
            tier_obs=[TierObservation(o.read_transfers, o.read_bytes, o.read_seconds, o.write_transfers,
                                      o.write_bytes, o.write_seconds) for o in st.tier_obs[:n]],
            subgroup_io=[SubgroupIoTimes(e.id, e.state_bytes, e.read_seconds, e.write_seconds, bool(e.fetched),
                                         bool(e.flushed)) for e in io[:got.value]],
            device_seconds=st.device_seconds, kernel_seconds=st.kernel_seconds, h2d_seconds=st.h2d_seconds,
            d2h_seconds=st.d2h_seconds, h2d_bytes=st.h2d_bytes, d2h_bytes=st.d2h_bytes)

    def last_timeline(self) -> list:
        """Per-subgroup pipeline timeline of the last run_update, plan order:
        dicts of h2d_start/h2d_end/k_start/k_end/d2h_end (device ms) and
        host_resident/host_retired (host ms)."""
        n = len(self._params)
        buf = (_lib.DeviceSpanC * max(n, 1))()
        got = C.c_uint64()
        _lib.call("tfg_engine_last_timeline", self._h, buf, n, C.byref(got))
        return [{f: getattr(s, f) for f, _ in _lib.DeviceSpanC._fields_} for s in buf[:got.value]]

    def wait_host_resident(self, sg: int) -> int:
        slot = C.c_int()
        _lib.call("tfg_engine_wait_host_resident", self._h, sg, C.byref(slot))
        return slot.value

    def enqueue_prefetch(self, sg: int) -> Optional[Ticket]:
        t = C.c_uint64()
        _lib.call("tfg_engine_enqueue_prefetch", self._h, sg, C.byref(t))
        return Ticket(self, t.value) if t.value else None

    def enqueue_flush(self, sg: int, dest: int) -> Ticket:
        t = C.c_uint64()
        _lib.call("tfg_engine_enqueue_flush", self._h, sg, dest, C.byref(t))
        return Ticket(self, t.value)

    def read_current_state(self, sg: int) -> np.ndarray:
        out = np.empty(3 * self._params[sg], np.float32)
        _lib.call("tfg_engine_read_state", self._h, sg, out.ctypes.data)
        return out

    def read_params16(self, sg: int) -> np.ndarray:
        out = np.empty(self._params[sg], np.uint16)
        _lib.call("tfg_engine_read_params16", self._h, sg, out.ctypes.data)
        return out

    def meta(self, sg: int) -> SubgroupMeta:
        m = _lib.SubgroupMetaC()
        _lib.call("tfg_engine_meta", self._h, sg, C.byref(m))
        return SubgroupMeta(m.id, Residency(m.residency), m.tier, m.slot, m.param_count, m.step_count)

    def residency_census(self):
        n = len(self._tiers)
        host = C.c_uint64()
        per = (C.c_uint64 * n)()
        _lib.call("tfg_engine_residency_census", self._h, C.byref(host), per, n)
        return host.value, list(per)

    def current_order(self) -> list:
        M = len(self._params)
        out = (C.c_uint32 * max(M, 1))()
        n = C.c_int()
        _lib.call("tfg_engine_current_order", self._h, out, M, C.byref(n))
        return list(out)[:n.value]

    def estimates(self):
        n = len(self._tiers)
        r, w = (C.c_double * n)(), (C.c_double * n)()
        _lib.call("tfg_engine_estimates", self._h, r, w, n)
        return list(r), list(w)

    def pool_state(self, slot: int):
        s, o = C.c_int(), C.c_uint32()
        _lib.call("tfg_engine_pool_state", self._h, slot, C.byref(s), C.byref(o))
        return SlotState(s.value), o.value


# ---------------------------------------------------------------------------
# Kernel-level operators on torch CUDA tensors


def _ptr(t) -> int:
    return t.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def adam_fused(p, m, v, grad16, param16, t: int, hyper: AdamHyper = AdamHyper(), grad_dtype: int = F16,
               param_dtype: int = F16, counters=None, stream=None, gate=None) -> None:
    """Fused widen -> Adam -> narrow on device tensors, async on `stream`.
    gate: optional device int64 tensor; the launch writes nothing when it is
    nonzero at kernel start (a whole-phase non-finite count on the stream)."""
    n = p.numel()
    for x in (m, v, grad16, param16):
        if x.numel() != n:
            raise Error("adam_fused: length mismatch")
    hy = hyper.c()
    cnt = _ptr(counters) if counters is not None else None
    if gate is None:
        _lib.call("tfg_adam_fused", _ptr(p), _ptr(m), _ptr(v), _ptr(grad16), grad_dtype, _ptr(param16), param_dtype,
                  n, C.byref(hy), t, cnt, _stream(stream))
    else:
        _lib.call("tfg_adam_fused_gated", _ptr(p), _ptr(m), _ptr(v), _ptr(grad16), grad_dtype, _ptr(param16),
                  param_dtype, n, C.byref(hy), t, cnt, _ptr(gate), _stream(stream))


def adam_fused_multi(p, m, v, grads: Sequence, param16, t: int, hyper: AdamHyper = AdamHyper(),
                     grad_dtype: int = F16, param_dtype: int = F16, counters=None, stream=None) -> None:
    """Reduce + update in one pass: the gradient is the fp32 sum (in order) of
    the 16-bit `grads` buffers — tensors, or raw device pointers such as mapped
    NVLink peer buffers — rounded once to grad_dtype."""
    n = p.numel()
    ptrs = [g if isinstance(g, int) else _ptr(g) for g in grads]
    arr = (C.c_void_p * len(ptrs))(*ptrs)
    hy = hyper.c()
    _lib.call("tfg_adam_fused_multi", _ptr(p), _ptr(m), _ptr(v), arr, len(ptrs), grad_dtype, _ptr(param16),
              param_dtype, n, C.byref(hy), t, _ptr(counters) if counters is not None else None, _stream(stream))


F32 = 2  # gradient kind of the ZeRO-3 baseline flow (fp32 gradients from storage)


def adam_step(p, m, v, grad16, param16, t: int, hyper: AdamHyper = AdamHyper(), grad_dtype: int = F16,
              param_dtype: int = F16, stream=None) -> int:
    """Reference-semantics step (optimizer.hpp:116-157): raises
    GradientOverflowError before mutating on non-finite gradients; returns the
    narrowing overflow count."""
    n = p.numel()
    for x in (m, v, grad16, param16):
        if x.numel() != n:
            raise Error("adam_step: length mismatch")
    hy = hyper.c()
    over = C.c_uint64()
    _lib.call("tfg_adam_step", _ptr(p), _ptr(m), _ptr(v), _ptr(grad16), grad_dtype, _ptr(param16), param_dtype, n,
              C.byref(hy), t, C.byref(over), _stream(stream))
    return over.value


def adam_variant_count() -> int:
    n = C.c_int()
    _lib.call_tuning("tfg_adam_variant_count", C.byref(n))
    return n.value


def adam_fused_variant(variant: int, p, m, v, grad16, param16, t: int, hyper: AdamHyper = AdamHyper(), counters=None,
                       stream=None) -> None:
    """Tuning hook: the fused kernel in launch configuration `variant` (F16/F16)."""
    hy = hyper.c()
    _lib.call_tuning("tfg_adam_fused_variant", variant, _ptr(p), _ptr(m), _ptr(v), _ptr(grad16), _ptr(param16), p.numel(),
              C.byref(hy), t, _ptr(counters) if counters is not None else None, _stream(stream))


def adam_fused_multi_variant(variant: int, p, m, v, grads: Sequence, param16, t: int, hyper: AdamHyper = AdamHyper(),
                             counters=None, stream=None) -> None:
    """Tuning hook: the n-source reduce + update in form `variant` (0 = staged kernel for 2/4/8 sources,
    1 = register kernel; F16/F16). grads: tensors or raw device pointers."""
    ptrs = [g if isinstance(g, int) else _ptr(g) for g in grads]
    arr = (C.c_void_p * len(ptrs))(*ptrs)
    hy = hyper.c()
    _lib.call_tuning("tfg_adam_fused_multi_variant", variant, _ptr(p), _ptr(m), _ptr(v), arr, len(ptrs), _ptr(param16),
                     p.numel(), C.byref(hy), t, _ptr(counters) if counters is not None else None, _stream(stream))


def selftest_div_const(divisor: float, n: int, seed: int = 1, exp_lo: int = -160, exp_span: int = 170):
    """(mismatches, first_bad_numerator) of the constant-divisor quotient vs div.rn.f64."""
    mm, fb = C.c_uint64(), C.c_double()
    _lib.call("tfg_selftest_div_const", divisor, n, seed, exp_lo, exp_span, C.byref(mm), C.byref(fb))
    return mm.value, fb.value


def upscale16(src, dst, dtype: int = F16, nonfinite=None, stream=None) -> None:
    _lib.call("tfg_upscale16", _ptr(src), _ptr(dst), src.numel(), dtype,
              _ptr(nonfinite) if nonfinite is not None else None, _stream(stream))


def downscale16(src, dst, dtype: int = F16, overflows=None, stream=None) -> None:
    _lib.call("tfg_downscale16", _ptr(src), _ptr(dst), src.numel(), dtype,
              _ptr(overflows) if overflows is not None else None, _stream(stream))


def count_nonfinite16(src, count, dtype: int = F16, stream=None) -> None:
    _lib.call("tfg_count_nonfinite16", _ptr(src), src.numel(), dtype, _ptr(count), _stream(stream))


def synthetic_grads(out, seed: int, subgroup: int, iteration: int, step: int = 0, accumulate: bool = False,
                    dtype: int = F16, stream=None) -> None:
    _lib.call("tfg_synthetic_grads", _ptr(out), out.numel(), dtype, seed, subgroup, iteration, step,
              int(accumulate), _stream(stream))


def synthetic_state(p, m, v, seed: int, subgroup: int, stream=None) -> None:
    _lib.call("tfg_synthetic_state", _ptr(p), _ptr(m), _ptr(v), p.numel(), seed, subgroup, _stream(stream))


IPC_HANDLE_BYTES = 64


def device_alloc(device: int, nbytes: int) -> int:
    p = C.c_void_p()
    _lib.call("tfg_device_alloc", device, nbytes, C.byref(p))
    return p.value


def device_free(device: int, ptr: int) -> None:
    _lib.call("tfg_device_free", device, C.c_void_p(ptr))


def ipc_get_handle(device: int, ptr: int) -> bytes:
    buf = C.create_string_buffer(IPC_HANDLE_BYTES)
    _lib.call("tfg_ipc_get_handle", device, C.c_void_p(ptr), buf)
    return buf.raw


def ipc_open_handle(device: int, handle: bytes) -> int:
    if len(handle) != IPC_HANDLE_BYTES:
        raise ValueError("IPC handle must be 64 bytes")
    p = C.c_void_p()
    _lib.call("tfg_ipc_open_handle", device, handle, C.byref(p))
    return p.value


def ipc_close_handle(device: int, ptr: int) -> None:
    _lib.call("tfg_ipc_close_handle", device, C.c_void_p(ptr))


def device_count() -> int:
    n = C.c_int()
    _lib.call("tfg_device_count", C.byref(n))
    return n.value
