"""CPU oracle for the update phase — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package, and only as the checker (or as the timed
reference CPU implementation). The product package paper_2509_02480_b200 never
imports it.

Two libraries:
  * liboracle.so  — tierflow_oracle.c, an independent C restatement of the
    reference arithmetic (16-bit codecs, Adam, generators, Eq. 1 placement,
    destination plan, schedule model).
  * _ref/libtierflow_ref.so — the unmodified reference headers compiled in
    place (oracle/ref_driver.cpp), present wherever `make -C oracle` ran with
    /root/reference available; it travels to the GPU box prebuilt.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"
REF_PATH = HERE / "_ref" / "libtierflow_ref.so"

_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

_lib = None
_ref = None


def build() -> None:
    """(Re)build liboracle.so and, where the reference is present, _ref."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        L.orc_f32_to_f16.restype = C.c_uint16
        L.orc_f32_to_f16.argtypes = [C.c_float]
        L.orc_f16_to_f32.restype = C.c_float
        L.orc_f16_to_f32.argtypes = [C.c_uint16]
        L.orc_f32_to_bf16.restype = C.c_uint16
        L.orc_f32_to_bf16.argtypes = [C.c_float]
        L.orc_bf16_to_f32.restype = C.c_float
        L.orc_bf16_to_f32.argtypes = [C.c_uint16]
        L.orc_f16_to_double.restype = C.c_double
        L.orc_f16_to_double.argtypes = [C.c_uint16]
        L.orc_narrow16_array.argtypes = [_f32p, _u16p, C.c_uint64, C.c_int, C.POINTER(C.c_uint64)]
        L.orc_count_nonfinite16.restype = C.c_uint64
        L.orc_count_nonfinite16.argtypes = [_u16p, C.c_uint64, C.c_int]
        L.orc_adam_step.argtypes = [_f32p, _f32p, _f32p, _f32p, C.c_uint64] + [C.c_double] * 5 + [C.c_uint64]
        L.orc_adam_fused.argtypes = ([_f32p, _f32p, _f32p, _u16p, C.c_int, _u16p, C.c_int, C.c_uint64]
                                     + [C.c_double] * 5 + [C.c_uint64, C.POINTER(C.c_uint64)])
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_synthetic_grads.argtypes = [_u16p, C.c_uint64, C.c_int, C.c_uint64, C.c_uint32, C.c_int, C.c_int,
                                          C.c_int]
        L.orc_synthetic_params.argtypes = [_f32p, C.c_uint64, C.c_uint64, C.c_uint32]
        L.orc_assign_subgroups.argtypes = [C.c_int, _f64p, C.c_int, _i32p]
        L.orc_destination_plan.argtypes = [C.c_int, C.c_int, _f64p, C.c_int, _i32p, _i32p, _i32p]
        L.orc_retention_capacity.argtypes = [C.c_int] * 4
        L.orc_update_order.argtypes = [C.c_int, _u32p, C.c_int, C.c_int, _u32p]
        L.orc_schedule_model.argtypes = ([_u32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _f64p, C.c_int]
                                         + [_u32p, _i32p, _i32p, _i32p])
        _lib = L
    return _lib


def ref_available() -> bool:
    return REF_PATH.exists()


class RefTierCfg(C.Structure):
    _fields_ = [("kind", C.c_int), ("root", C.c_char_p), ("read_bps", C.c_double), ("write_bps", C.c_double),
                ("io_parallelism", C.c_int)]


class RefRunCfg(C.Structure):
    _fields_ = [("n_subgroups", C.c_int), ("params", C.POINTER(C.c_uint64)), ("n_tiers", C.c_int),
                ("tiers", C.POINTER(RefTierCfg)), ("fixed_ratio", C.POINTER(C.c_double)), ("pool_slots", C.c_int),
                ("cache_slots", C.c_int), ("enable_caching", C.c_int), ("multi_path", C.c_int),
                ("atomic_rw", C.c_int), ("update_threads", C.c_int), ("lock_dir", C.c_char_p),
                ("seed", C.c_uint64), ("iterations", C.c_int), ("accum_steps", C.c_int), ("lr", C.c_double),
                ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double), ("weight_decay", C.c_double),
                ("skip_mask", C.c_uint32), ("skip_gradients", C.c_int), ("backward_once", C.c_int)]


class RefIterOut(C.Structure):
    _fields_ = [("update_seconds", C.c_double), ("backward_seconds", C.c_double), ("params_updated", C.c_uint64),
                ("cache_hits", C.c_uint64), ("overflows", C.c_uint64), ("retained", C.c_int),
                ("flush_allocation", C.c_int * 8), ("trace_begin", C.c_uint64), ("trace_end", C.c_uint64)]


class RefEvent(C.Structure):
    _fields_ = [("ts", C.c_int64), ("worker", C.c_int32), ("kind", C.c_int32), ("sg", C.c_int64),
                ("tier", C.c_int32), ("pad", C.c_int32), ("bytes", C.c_uint64)]


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_PATH.exists():
            build()
        if not REF_PATH.exists():
            raise FileNotFoundError(f"{REF_PATH} not built (reference sources absent here)")
        R = C.CDLL(str(REF_PATH))
        R.ref_last_error.restype = C.c_char_p
        R.ref_adam_step.argtypes = [_f32p, _f32p, _f32p, _f32p, C.c_uint64] + [C.c_double] * 5 + [C.c_uint64, C.c_int]
        R.ref_f32_to_f16.restype = C.c_uint16
        R.ref_f32_to_f16.argtypes = [C.c_float]
        R.ref_f16_to_f32.restype = C.c_float
        R.ref_f16_to_f32.argtypes = [C.c_uint16]
        R.ref_upscale.argtypes = [_u16p, _f32p, C.c_uint64, C.POINTER(C.c_int)]
        R.ref_downscale.argtypes = [_f32p, _u16p, C.c_uint64, C.POINTER(C.c_uint64)]
        R.ref_assign_subgroups.argtypes = [C.c_int, _f64p, C.c_int, _i32p]
        R.ref_destination_plan.argtypes = [_u32p, C.c_int, C.c_int, _f64p, C.c_int, _i32p, _i32p, _i32p]
        R.ref_synthetic_grads.argtypes = [_u16p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_int, C.c_int]
        R.ref_accumulated_grads.argtypes = [_u16p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_int, C.c_int]
        R.ref_synthetic_params.argtypes = [_f32p, C.c_uint64, C.c_uint64, C.c_uint32]
        R.ref_update_order.argtypes = [C.c_int, _u32p, C.c_int, C.c_int, _u32p]
        R.ref_retention_capacity.argtypes = [C.c_int] * 4
        R.ref_run_engine.argtypes = [C.POINTER(RefRunCfg), C.POINTER(RefIterOut), C.c_void_p, C.POINTER(RefEvent),
                                     C.c_uint64, C.POINTER(C.c_uint64)]
        _ref = R
    return _ref


# ---------------------------------------------------------------------------
# numpy conveniences over liboracle


def f32_to_f16(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32).ravel()
    out = np.empty(x.size, np.uint16)
    lib().orc_narrow16_array(x, out, x.size, 0, None)
    return out


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32).ravel()
    out = np.empty(x.size, np.uint16)
    lib().orc_narrow16_array(x, out, x.size, 1, None)
    return out


def widen16(h: np.ndarray, kind: int) -> np.ndarray:
    h = np.ascontiguousarray(h, dtype=np.uint16).ravel()
    L = lib()
    f = L.orc_f16_to_f32 if kind == 0 else L.orc_bf16_to_f32
    if kind == 1:
        return (h.astype(np.uint32) << 16).view(np.float32)
    # f16: exact via the oracle decode, vectorised with a 65536-entry table
    table = np.array([f(i) for i in range(65536)], dtype=np.float32) if _F16_TABLE[0] is None else _F16_TABLE[0]
    _F16_TABLE[0] = table
    return table[h]


_F16_TABLE = [None]


def narrow16(x: np.ndarray, kind: int) -> tuple[np.ndarray, int]:
    x = np.ascontiguousarray(x, dtype=np.float32).ravel()
    out = np.empty(x.size, np.uint16)
    over = C.c_uint64(0)
    lib().orc_narrow16_array(x, out, x.size, kind, C.byref(over))
    return out, int(over.value)


def adam_fused(p, m, v, g16, grad_kind, out_kind, t, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0):
    """Oracle of the fused kernel on copies; returns (p, m, v, p16, overflows)."""
    p = np.array(p, dtype=np.float32, copy=True)
    m = np.array(m, dtype=np.float32, copy=True)
    v = np.array(v, dtype=np.float32, copy=True)
    g16 = np.ascontiguousarray(g16, dtype=np.uint16)
    p16 = np.empty(p.size, np.uint16)
    over = C.c_uint64(0)
    rc = lib().orc_adam_fused(p, m, v, g16, grad_kind, p16, out_kind, p.size, lr, beta1, beta2, eps, weight_decay,
                              t, C.byref(over))
    if rc != 0:
        raise ValueError(f"oracle adam_fused rc={rc}")
    return p, m, v, p16, int(over.value)


def synthetic_grads(n: int, seed: int, sg: int, iteration: int, steps: int = 1, kind: int = 0) -> np.ndarray:
    out = np.zeros(n, np.uint16)
    for s in range(steps):
        lib().orc_synthetic_grads(out, n, kind, seed, sg, iteration, s, 1 if s > 0 else 0)
    return out


def synthetic_params(n: int, seed: int, sg: int) -> np.ndarray:
    out = np.empty(n, np.float32)
    lib().orc_synthetic_params(out, n, seed, sg)
    return out


def assign_subgroups(M: int, bw) -> list[int]:
    bw = np.ascontiguousarray(bw, dtype=np.float64)
    out = np.zeros(bw.size, np.int32)
    if lib().orc_assign_subgroups(M, bw, bw.size, out) != 0:
        raise ValueError("assign_subgroups: invalid input")
    return out.tolist()


def destination_plan(M: int, capacity: int, bw):
    bw = np.ascontiguousarray(bw, dtype=np.float64)
    retain = np.zeros(M, np.int32)
    tier = np.zeros(M, np.int32)
    alloc = np.zeros(bw.size, np.int32)
    if lib().orc_destination_plan(M, capacity, bw, bw.size, retain, tier, alloc) != 0:
        raise ValueError("destination_plan: invalid input")
    return retain.tolist(), tier.tolist(), alloc.tolist()


def schedule_model(ids, iters, pool_slots, cache_slots, caching, multi_path, bw):
    ids = np.ascontiguousarray(sorted(ids), dtype=np.uint32)
    M = ids.size
    bw = np.ascontiguousarray(bw, dtype=np.float64)
    order = np.zeros(iters * M, np.uint32)
    hit = np.zeros(iters * M, np.int32)
    dest = np.zeros(iters * M, np.int32)
    origin = np.zeros(iters * M, np.int32)
    rc = lib().orc_schedule_model(ids, M, iters, pool_slots, cache_slots, int(caching), int(multi_path), bw, bw.size,
                                  order, hit, dest, origin)
    if rc != 0:
        raise ValueError("schedule_model: invalid input")
    sh = (iters, M)
    return order.reshape(sh), hit.reshape(sh), dest.reshape(sh), origin.reshape(sh)


def run_engine_oracle(param_counts, seed, iters, pool_slots, cache_slots, caching, multi_path, bw, accum_steps=1,
                      grad_kind=0, out_kind=0, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0):
    """End state of the update phase computed by the oracle: per subgroup
    (P, m, v, p16) after `iters` update phases, plus the schedule model."""
    M = len(param_counts)
    states = []
    for sg, n in enumerate(param_counts):
        states.append([synthetic_params(n, seed, sg), np.zeros(n, np.float32), np.zeros(n, np.float32),
                       np.zeros(n, np.uint16)])
    for it in range(iters):
        for sg, n in enumerate(param_counts):
            g = synthetic_grads(n, seed, sg, it, accum_steps, grad_kind)
            p, m, v, p16, _ = adam_fused(states[sg][0], states[sg][1], states[sg][2], g, grad_kind, out_kind, it + 1,
                                         lr, beta1, beta2, eps, weight_decay)
            states[sg] = [p, m, v, p16]
    sched = schedule_model(list(range(M)), iters, pool_slots, cache_slots, caching, multi_path, bw)
    return states, sched


def run_ref_engine(param_counts, tiers, *, fixed_ratio=None, pool_slots=4, cache_slots=-1, enable_caching=True,
                   multi_path=True, atomic_rw=True, update_threads=1, lock_dir=None, seed=42, iterations=3,
                   accum_steps=1, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, skip_mask=0,
                   want_states=True, events_cap=1 << 16, skip_gradients=True, backward_once=False):
    """Runs the UNMODIFIED reference OffloadWorker (via oracle/_ref).

    tiers: list of dicts {kind: 0|1|2, root, read_bps, write_bps, io_parallelism}.
    Returns {"iters": [...], "states": [per-subgroup P||m||v] | None, "events": [(kind, sg, tier, bytes)]}.
    """
    R = ref()
    M = len(param_counts)
    params = (C.c_uint64 * M)(*param_counts)
    keep = [t.get("root", "").encode() if t.get("root") else None for t in tiers]
    tc = (RefTierCfg * len(tiers))(*[RefTierCfg(t["kind"], keep[i], t.get("read_bps", 0.0), t.get("write_bps", 0.0),
                                                t.get("io_parallelism", 1)) for i, t in enumerate(tiers)])
    ratio = (C.c_double * len(tiers))(*fixed_ratio) if fixed_ratio is not None else None
    lock = lock_dir.encode() if lock_dir else None
    cfg = RefRunCfg(M, params, len(tiers), tc, ratio, pool_slots, cache_slots, int(enable_caching), int(multi_path),
                    int(atomic_rw), update_threads, lock, seed, iterations, accum_steps, lr, beta1, beta2, eps,
                    weight_decay, skip_mask, int(skip_gradients), int(backward_once))
    iters = (RefIterOut * iterations)()
    total = sum(3 * n for n in param_counts)
    states = np.empty(total, np.float32) if want_states else None
    ev = (RefEvent * events_cap)()
    nev = C.c_uint64()
    rc = R.ref_run_engine(C.byref(cfg), iters, states.ctypes.data if want_states else None, ev, events_cap,
                          C.byref(nev))
    if rc != 0:
        raise RuntimeError(f"reference engine failed rc={rc}: {R.ref_last_error().decode()}")
    out_states = None
    if want_states:
        out_states, off = [], 0
        for n in param_counts:
            out_states.append(states[off:off + 3 * n].copy())
            off += 3 * n
    events = [(e.kind, e.sg, e.tier, e.bytes) for e in ev[:min(nev.value, events_cap)]]
    it_out = []
    for r in iters:
        it_out.append(dict(update_seconds=r.update_seconds, backward_seconds=r.backward_seconds,
                           params_updated=r.params_updated, cache_hits=r.cache_hits, overflows=r.overflows,
                           retained=r.retained, flush_allocation=list(r.flush_allocation)[:len(tiers)],
                           trace_begin=r.trace_begin, trace_end=r.trace_end))
    return {"iters": it_out, "states": out_states, "events": events}


# EventKind indices (reference trace.hpp:19-33).
EV_PREFETCH_END, EV_FLUSH_END, EV_CACHE_HIT = 1, 5, 12


def phase_sequences(events, begin, end, n_tiers):
    """Timing-independent sequences of one phase: cache-hit ids in order,
    per-tier prefetch order and per-tier flushed ids (as sorted lists)."""
    hits, pf, fl = [], [[] for _ in range(n_tiers)], [[] for _ in range(n_tiers)]
    for kind, sg, tier, _b in events[begin:end]:
        if kind == EV_CACHE_HIT:
            hits.append(int(sg))
        elif kind == EV_PREFETCH_END and tier >= 0:
            pf[tier].append(int(sg))
        elif kind == EV_FLUSH_END and tier >= 0:
            fl[tier].append(int(sg))
    return {"hits": hits, "prefetch": pf, "flush": [sorted(x) for x in fl]}
