"""Benchmark driver, run config and reports for the B200 update engine — the
reference's L5/L6 layer (config.hpp, harness.hpp, report.hpp, tools/bench.cpp)
rebuilt over the C ABI so reference configs and reports carry over.

    python -m paper_2509_02480_b200.harness run --config cfg.json [--mode engine|baseline]
        [--trace-out t.csv] [--report-out dir] [--iterations N] [--workers N] [--seed S]
        [--enable-caching|--no-enable-caching] [--skip-gradients|--no-skip-gradients]
        [--atomic-rw|--no-atomic-rw] [--multi-path|--no-multi-path] [--multiprocess]
    python -m paper_2509_02480_b200.harness probe --tier <root> [--bytes-mib N] [--reps N]
    python -m paper_2509_02480_b200.harness compare <report_a> <report_b> [--out file]

Config schema = the reference's (config.hpp:150-215: model, tiers[], placement,
optim, schedule, run, ablation) plus an optional "device" section
({device, grad_dtype, param_dtype, device_buffers, zero_copy, d2h_split,
hbm_retain, h2d_split, hbm_cache_slots}), the tier kind "host_dram" and the
per-tier keys lock_device and capacity_gb. Semantics follow the reference: ragged last
subgroup (config.hpp:77-87), mode-derived ablation flags (config.hpp:91-105),
lock-dir precedence TIERFLOW_LOCK_DIR > config > tmp (config.hpp:108-112),
contiguous worker sharding (harness.hpp:118-126), non-finite gradients skip
the step (harness.hpp:218-228), means over measured iterations
(report.hpp:81-106), effective I/O = mean 2*size/(t_r+t_w) (report.hpp:25-37).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import math
import os
import subprocess
import sys
import tempfile
import threading
import time
from dataclasses import asdict, dataclass, field
from pathlib import Path
from typing import Callable, List, Optional, Sequence

from . import tierflow as tf
from .parallel import shard

KINDS = {"local_dir": tf.TierKind.local_dir, "remote_dir": tf.TierKind.remote_dir,
         "mem_throttled": tf.TierKind.mem_throttled, "host_dram": tf.TierKind.host_dram}


# ---------------------------------------------------------------------------
# config


@dataclass
class TierConfig:
    kind: str = "local_dir"
    root: str = ""
    read_mb_s: float = 0.0
    write_mb_s: float = 0.0
    io_parallelism: int = 1
    persistent: bool = False
    probe: bool = False
    probe_mib: float = 8.0
    probe_reps: int = 3
    # B200 extensions (absent from the reference schema; 0 = reference behaviour)
    lock_device: int = 0
    capacity_gb: float = 0.0


@dataclass
class RunConfig:
    total_params: int = 24 * 2_796_202
    subgroup_param_count: int = 2_796_202
    tiers: List[TierConfig] = field(default_factory=list)
    alpha: float = 0.5
    ratio: List[float] = field(default_factory=list)
    optim: tf.AdamHyper = field(default_factory=tf.AdamHyper)
    pool_slots: int = 6
    cache_slots: int = -1
    workers_per_node: int = 1
    lock_dir: str = ""
    update_threads: int = 0
    deadlock_timeout_s: float = 30.0
    iterations: int = 10
    warmup_iterations: int = 2
    grad_accum_steps: int = 1
    mode: str = "engine"
    seed: int = 42
    forward_stub_ms: float = 1.0
    update_pad_us: float = 0.0
    enable_caching: Optional[bool] = None
    skip_gradients: Optional[bool] = None
    atomic_rw: Optional[bool] = None
    multi_path: Optional[bool] = None
    device: tf.DeviceOptions = field(default_factory=tf.DeviceOptions)

    def subgroup_count(self) -> int:
        return (self.total_params + self.subgroup_param_count - 1) // self.subgroup_param_count

    def subgroup_params(self, index: int) -> int:
        return min(self.subgroup_param_count, self.total_params - index * self.subgroup_param_count)

    def engine_mode(self) -> bool:
        return self.mode == "engine"

    def resolve_lock_dir(self) -> str:
        env = os.environ.get("TIERFLOW_LOCK_DIR")
        if env:
            return env
        if self.lock_dir:
            return self.lock_dir
        return os.path.join(tempfile.gettempdir(), "tierflow-locks")

    def schedule_options(self) -> tf.ScheduleOptions:
        base = self.engine_mode()
        pick = lambda v: base if v is None else v  # noqa: E731
        return tf.ScheduleOptions(pool_slots=self.pool_slots, cache_slots=self.cache_slots,
                                  enable_caching=pick(self.enable_caching), skip_gradients=pick(self.skip_gradients),
                                  atomic_rw=pick(self.atomic_rw), multi_path=pick(self.multi_path),
                                  lock_dir=self.resolve_lock_dir(), update_threads=self.update_threads,
                                  deadlock_timeout_s=self.deadlock_timeout_s,
                                  update_pad_ns=int(self.update_pad_us * 1000.0))

    def validate(self) -> None:
        E = tf.ConfigError
        if self.total_params <= 0:
            raise E("model.total_params must be > 0")
        if self.subgroup_param_count <= 0:
            raise E("model.subgroup_param_count must be > 0")
        if not self.tiers:
            raise E("at least one tier is required")
        for t in self.tiers:
            if t.kind not in KINDS:
                raise E(f"unknown tier kind: {t.kind}")
            if t.kind == "mem_throttled" and (t.read_mb_s <= 0 or t.write_mb_s <= 0):
                raise E("mem_throttled tiers need read/write rates")
            if t.kind in ("local_dir", "remote_dir") and not t.root:
                raise E("directory tiers need a root path")
            if t.io_parallelism < 1:
                raise E("tier io_parallelism must be >= 1")
        if self.ratio and len(self.ratio) != len(self.tiers):
            raise E("placement.ratio length must match the tier count")
        if not (self.alpha > 0.0) or self.alpha > 1.0:
            raise E("placement.alpha must be in (0, 1]")
        h = self.optim
        if not h.lr > 0 or not 0 <= h.beta1 < 1 or not 0 <= h.beta2 < 1 or not h.eps > 0 or h.weight_decay < 0:
            raise E("invalid optim hyperparameters")
        if self.pool_slots < 3:
            raise E("schedule.pool_slots must be >= 3")
        if self.workers_per_node < 1:
            raise E("workers_per_node must be >= 1")
        if self.iterations < 1:
            raise E("run.iterations must be >= 1")
        if self.warmup_iterations < 0 or self.warmup_iterations >= self.iterations:
            raise E("warmup_iterations must be < iterations")
        if self.grad_accum_steps < 1:
            raise E("grad_accum_steps must be >= 1")
        if self.mode not in ("engine", "baseline"):
            raise E("run.mode must be engine or baseline")
        if self.subgroup_count() < self.workers_per_node:
            raise E("need at least one subgroup per worker")

    @staticmethod
    def from_json(j: dict) -> "RunConfig":
        c = RunConfig()
        m = j.get("model", {})
        c.total_params = int(m.get("total_params", c.total_params))
        c.subgroup_param_count = int(m.get("subgroup_param_count", c.subgroup_param_count))
        if "tiers" in j:
            c.tiers = []
            for t in j["tiers"]:
                kind = t.get("kind", "local_dir")
                if kind not in KINDS:
                    raise tf.ConfigError(f"unknown tier kind: {kind}")
                c.tiers.append(TierConfig(kind=kind, root=t.get("root", ""), read_mb_s=float(t.get("read_mb_s", 0.0)),
                                          write_mb_s=float(t.get("write_mb_s", 0.0)),
                                          io_parallelism=int(t.get("io_parallelism", 1)),
                                          persistent=bool(t.get("persistent", kind == "remote_dir")),
                                          probe=bool(t.get("probe", False)), probe_mib=float(t.get("probe_mib", 8.0)),
                                          probe_reps=int(t.get("probe_reps", 3)),
                                          lock_device=int(t.get("lock_device", 0)),
                                          capacity_gb=float(t.get("capacity_gb", 0.0))))
        p = j.get("placement", {})
        c.alpha = float(p.get("alpha", 0.5))
        c.ratio = [float(x) for x in p.get("ratio", [])]
        o = j.get("optim", {})
        c.optim = tf.AdamHyper(lr=float(o.get("lr", 1e-3)), beta1=float(o.get("beta1", 0.9)),
                               beta2=float(o.get("beta2", 0.999)), eps=float(o.get("eps", 1e-8)),
                               weight_decay=float(o.get("weight_decay", 0.0)))
        s = j.get("schedule", {})
        c.pool_slots = int(s.get("pool_slots", c.pool_slots))
        c.cache_slots = int(s.get("cache_slots", c.cache_slots))
        c.workers_per_node = int(s.get("workers_per_node", c.workers_per_node))
        c.lock_dir = s.get("lock_dir", c.lock_dir)
        c.update_threads = int(s.get("update_threads", c.update_threads))
        c.deadlock_timeout_s = float(s.get("deadlock_timeout_s", c.deadlock_timeout_s))
        r = j.get("run", {})
        c.iterations = int(r.get("iterations", c.iterations))
        c.warmup_iterations = int(r.get("warmup_iterations", c.warmup_iterations))
        c.grad_accum_steps = int(r.get("grad_accum_steps", c.grad_accum_steps))
        c.mode = r.get("mode", c.mode)
        c.seed = int(r.get("seed", c.seed))
        c.forward_stub_ms = float(r.get("forward_stub_ms", c.forward_stub_ms))
        c.update_pad_us = float(r.get("update_pad_us", c.update_pad_us))
        a = j.get("ablation", {})
        for k in ("enable_caching", "skip_gradients", "atomic_rw", "multi_path"):
            if k in a:
                setattr(c, k, bool(a[k]))
        d = j.get("device", {})
        c.device = tf.DeviceOptions(device=int(d.get("device", 0)), grad_dtype=int(d.get("grad_dtype", tf.F16)),
                                    param_dtype=int(d.get("param_dtype", tf.F16)),
                                    device_buffers=int(d.get("device_buffers", 3)),
                                    zero_copy=bool(d.get("zero_copy", False)), d2h_split=int(d.get("d2h_split", 1)),
                                    hbm_retain=int(d.get("hbm_retain", 1)), h2d_split=int(d.get("h2d_split", 1)),
                                    hbm_cache_slots=int(d.get("hbm_cache_slots", 0)))
        return c

    @staticmethod
    def from_file(path) -> "RunConfig":
        try:
            text = Path(path).read_text()
        except OSError:
            raise tf.ConfigError(f"cannot open config file {path}")
        try:
            j = json.loads(text)
        except json.JSONDecodeError as e:
            raise tf.ConfigError(f"config parse error in {path}: {e}")
        return RunConfig.from_json(j)


# ---------------------------------------------------------------------------
# reports


def effective_io_throughput(io_times: Sequence[tf.SubgroupIoTimes]) -> Optional[float]:
    """Mean over moved subgroups of 2*state_bytes/(t_read+t_write); None when
    nothing moved (report.hpp:25-37)."""
    vals = [2.0 * e.state_bytes / (e.read_seconds + e.write_seconds) for e in io_times
            if e.fetched and e.flushed and e.read_seconds + e.write_seconds > 0]
    return sum(vals) / len(vals) if vals else None


@dataclass
class IterationReport:
    iteration: int = 0
    warmup: bool = False
    skipped: bool = False
    forward_s: float = 0.0
    backward_s: float = 0.0
    update_s: float = 0.0
    update_throughput_mparams: float = 0.0
    effective_io_bps: Optional[float] = None
    update_read_bytes: list = field(default_factory=list)
    update_write_bytes: list = field(default_factory=list)
    backward_write_bytes: list = field(default_factory=list)
    host_pct: float = 0.0
    tier_pct: list = field(default_factory=list)
    cache_hits: int = 0
    overflow_count: int = 0
    flush_allocation: list = field(default_factory=list)
    retained: int = 0
    # B200 extras (device timeline of the phase, summed over workers)
    kernel_s: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0

    def iter_s(self) -> float:
        return self.forward_s + self.backward_s + self.update_s


@dataclass
class RunSummary:
    mode: str = ""
    iterations: int = 0
    warmup_iterations: int = 0
    subgroups: int = 0
    workers: int = 1
    total_params: int = 0
    subgroup_param_count: int = 0
    seed: int = 0
    iters: list = field(default_factory=list)
    mean_iter_s: float = 0.0
    mean_forward_s: float = 0.0
    mean_backward_s: float = 0.0
    mean_update_s: float = 0.0
    mean_update_throughput_mparams: float = 0.0
    mean_effective_io_bps: Optional[float] = None

    def compute_aggregates(self) -> None:
        meas = [r for r in self.iters if not r.warmup and not r.skipped]
        if meas:
            n = len(meas)
            self.mean_iter_s = sum(r.iter_s() for r in meas) / n
            self.mean_forward_s = sum(r.forward_s for r in meas) / n
            self.mean_backward_s = sum(r.backward_s for r in meas) / n
            self.mean_update_s = sum(r.update_s for r in meas) / n
            self.mean_update_throughput_mparams = sum(r.update_throughput_mparams for r in meas) / n
        eio = [r.effective_io_bps for r in meas if r.effective_io_bps is not None]
        self.mean_effective_io_bps = sum(eio) / len(eio) if eio else None


def _iteration_json(r: IterationReport) -> dict:
    d = asdict(r)
    d["iter_s"] = r.iter_s()
    order = ["iteration", "warmup", "skipped", "forward_s", "backward_s", "update_s", "iter_s",
             "update_throughput_mparams", "effective_io_bps", "update_read_bytes", "update_write_bytes",
             "backward_write_bytes", "host_pct", "tier_pct", "cache_hits", "overflow_count", "flush_allocation",
             "retained", "kernel_s", "h2d_bytes", "d2h_bytes"]
    return {k: d[k] for k in order}


def summary_to_json(s: RunSummary) -> dict:
    keys = ["mode", "iterations", "warmup_iterations", "subgroups", "workers", "total_params",
            "subgroup_param_count", "seed", "mean_iter_s", "mean_forward_s", "mean_backward_s", "mean_update_s",
            "mean_update_throughput_mparams", "mean_effective_io_bps"]
    j = {k: getattr(s, k) for k in keys}
    j["iterations_detail"] = [_iteration_json(r) for r in s.iters]
    return j


def summary_from_json(j: dict) -> RunSummary:
    s = RunSummary(**{k: j[k] for k in ("mode", "iterations", "warmup_iterations", "subgroups", "workers",
                                        "total_params", "subgroup_param_count", "seed", "mean_iter_s",
                                        "mean_forward_s", "mean_backward_s", "mean_update_s",
                                        "mean_update_throughput_mparams", "mean_effective_io_bps")})
    for rj in j["iterations_detail"]:
        rj = dict(rj)
        rj.pop("iter_s", None)
        s.iters.append(IterationReport(**rj))
    return s


def load_summary(path) -> RunSummary:
    try:
        return summary_from_json(json.loads(Path(path).read_text()))
    except OSError:
        raise tf.IoError(f"cannot open report {path}")


def _g(v: float) -> str:
    return "%.17g" % v


def emit_report(s: RunSummary, out_dir) -> None:
    """summary.json + iterations.csv, bytewise deterministic (report.hpp:224-261)."""
    d = Path(out_dir)
    try:
        d.mkdir(parents=True, exist_ok=True)
    except OSError:
        raise tf.IoError(f"cannot create report directory {d}")
    (d / "summary.json").write_text(json.dumps(summary_to_json(s), indent=2) + "\n")
    tiers = len(s.iters[0].tier_pct) if s.iters else 0
    buf = io.StringIO()
    head = ("iteration,warmup,skipped,forward_s,backward_s,update_s,iter_s,update_throughput_mparams,"
            "effective_io_bps,cache_hits,overflow_count,retained,host_pct")
    for t in range(tiers):
        head += f",tier{t}_pct,tier{t}_read_bytes,tier{t}_write_bytes,tier{t}_backward_write_bytes,tier{t}_alloc"
    buf.write(head + "\n")
    for r in s.iters:
        row = [str(r.iteration), str(int(r.warmup)), str(int(r.skipped)), _g(r.forward_s), _g(r.backward_s),
               _g(r.update_s), _g(r.iter_s()), _g(r.update_throughput_mparams),
               _g(r.effective_io_bps) if r.effective_io_bps is not None else "na", str(r.cache_hits),
               str(r.overflow_count), str(r.retained), _g(r.host_pct)]
        for t in range(tiers):
            pick = lambda a: a[t] if t < len(a) else 0  # noqa: E731
            row += [_g(pick(r.tier_pct)), str(pick(r.update_read_bytes)), str(pick(r.update_write_bytes)),
                    str(pick(r.backward_write_bytes)), str(pick(r.flush_allocation))]
        buf.write(",".join(row) + "\n")
    (d / "iterations.csv").write_text(buf.getvalue())


def compare_reports(a: RunSummary, b: RunSummary) -> dict:
    """Candidate a against baseline b (report.hpp:264-279)."""
    return {
        "candidate_mode": a.mode, "baseline_mode": b.mode,
        "mean_iter_s": a.mean_iter_s, "mean_update_s": a.mean_update_s, "mean_backward_s": a.mean_backward_s,
        "baseline_mean_iter_s": b.mean_iter_s, "baseline_mean_update_s": b.mean_update_s,
        "baseline_mean_backward_s": b.mean_backward_s,
        "speedup_vs_baseline": b.mean_iter_s / a.mean_iter_s if a.mean_iter_s > 0 else 0.0,
        "update_speedup_vs_baseline": b.mean_update_s / a.mean_update_s if a.mean_update_s > 0 else 0.0,
        "backward_speedup_vs_baseline": b.mean_backward_s / a.mean_backward_s if a.mean_backward_s > 0 else 0.0,
    }


# ---------------------------------------------------------------------------
# runner


class BenchRunner:
    """Builds tiers and GPU engines from a RunConfig and runs the iteration
    loop: forward stub -> backward sim -> finite check / skip -> update phase
    (harness.hpp:32-279). Workers are threads (one engine each, all on
    cfg.device.device) unless worker_rank selects one shard for this process."""

    def __init__(self, cfg: RunConfig, worker_rank: int = -1):
        cfg.validate()
        self.cfg = cfg
        self.rank = worker_rank
        self.trace = tf.EventTrace()
        self.before_iteration: Optional[Callable[[int, "BenchRunner"], None]] = None
        self.after_backward: Optional[Callable[[int, "BenchRunner"], None]] = None
        self.tiers: List[tf.Tier] = []
        self.workers: List[tf.OffloadWorker] = []
        self._build_tiers()
        self._build_workers()

    def _build_tiers(self):
        for i, tc in enumerate(self.cfg.tiers):
            spec = tf.TierSpec(i, KINDS[tc.kind], tc.root or f"{tc.kind}{i}", tc.read_mb_s * 1e6, tc.write_mb_s * 1e6,
                               tc.io_parallelism, tc.persistent, lock_device=tc.lock_device,
                               capacity_bytes=int(tc.capacity_gb * 1e9))
            if tc.kind == "host_dram" and spec.read_bw <= 0:
                spec.read_bw = spec.write_bw = 50e9  # block exchange; the PCIe leg is the transfer cost
            tier = tf.Tier(spec)
            if tc.kind in ("local_dir", "remote_dir") and (tc.probe or tc.read_mb_s <= 0):
                tier.probe_bandwidth(int(tc.probe_mib * 1024 * 1024), tc.probe_reps)
            self.tiers.append(tier)

    def _make_worker(self, w: int) -> tf.OffloadWorker:
        c = self.cfg
        e = tf.OffloadWorker(w, self.tiers, c.schedule_options(), c.optim, self.trace, c.device)
        e.set_alpha(c.alpha)
        if c.ratio:
            e.set_fixed_ratio(c.ratio)
        begin, count = shard(c.subgroup_count(), c.workers_per_node, w)
        for k in range(count):
            e.add_subgroup(begin + k, c.subgroup_params(begin + k))
        return e

    def _build_workers(self):
        world = self.cfg.workers_per_node
        if self.rank >= 0:
            if self.rank >= world:
                raise tf.ConfigError("worker rank out of range")
            self.workers.append(self._make_worker(self.rank))
        else:
            self.workers = [self._make_worker(w) for w in range(world)]

    def worker(self, i: int) -> tf.OffloadWorker:
        return self.workers[i]

    def worker_count(self) -> int:
        return len(self.workers)

    def _preflight(self):
        skip = self.cfg.schedule_options().skip_gradients
        need = sum((12 + (0 if skip else 4)) * w._params[i] for w in self.workers for i in w.subgroup_ids())
        for t in self.tiers:
            if t.available_bytes() < need + need // 16:
                raise tf.ConfigError(f"tier {t.id()}: insufficient capacity for {need} bytes of offloaded state")

    def _parallel(self, fn):
        if len(self.workers) == 1:
            fn(0)
            return
        errs = []

        def run(i):
            try:
                fn(i)
            except BaseException as e:  # noqa: BLE001
                errs.append(e)
        ths = [threading.Thread(target=run, args=(i,)) for i in range(len(self.workers))]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        if errs:
            raise errs[0]

    def _bytes_in_window(self, begin: int):
        n = len(self.tiers)
        rd, wr = [0] * n, [0] * n
        for e in self.trace.snapshot(begin):
            if 0 <= e.tier_id < n:
                if e.kind == tf.EventKind.prefetch_end:
                    rd[e.tier_id] += e.bytes
                elif e.kind == tf.EventKind.flush_end:
                    wr[e.tier_id] += e.bytes
        return rd, wr

    def _fill_distribution(self, r: IterationReport):
        host, total, per = 0, 0, [0] * len(self.tiers)
        for w in self.workers:
            h, t = w.residency_census()
            host += h
            per = [a + b for a, b in zip(per, t)]
            total += w.total_params()
        r.host_pct = 100.0 * host / total if total else 0.0
        r.tier_pct = [100.0 * p / total if total else 0.0 for p in per]

    def run_iteration(self, it: int) -> IterationReport:
        c = self.cfg
        r = IterationReport(iteration=it, warmup=it < c.warmup_iterations)
        f0 = time.perf_counter()
        if c.forward_stub_ms > 0:
            time.sleep(c.forward_stub_ms / 1e3)
        r.forward_s = time.perf_counter() - f0
        mark = self.trace.size()
        b0 = time.perf_counter()
        src = tf.SyntheticGradSource(c.seed)
        self._parallel(lambda w: self.workers[w].run_backward_sim(it, src, c.grad_accum_steps))
        r.backward_s = time.perf_counter() - b0
        _, r.backward_write_bytes = self._bytes_in_window(mark)
        if self.after_backward:
            self.after_backward(it, self)
        if not all(w.gradients_finite() for w in self.workers):
            r.skipped = True
            r.overflow_count = 1
            self._fill_distribution(r)
            r.update_read_bytes = [0] * len(self.tiers)
            r.update_write_bytes = [0] * len(self.tiers)
            return r
        mark = self.trace.size()
        stats = [None] * len(self.workers)
        u0 = time.perf_counter()
        self._parallel(lambda w: stats.__setitem__(w, self.workers[w].run_update(it)))
        r.update_s = time.perf_counter() - u0
        r.update_read_bytes, r.update_write_bytes = self._bytes_in_window(mark)
        params = sum(s.params_updated for s in stats)
        r.cache_hits = sum(s.cache_hits for s in stats)
        r.overflow_count = sum(s.downscale_overflows for s in stats)
        r.retained = sum(s.retained for s in stats)
        r.flush_allocation = [sum(s.flush_allocation[t] for s in stats) for t in range(len(self.tiers))]
        r.update_throughput_mparams = params / r.update_s / 1e6
        r.effective_io_bps = effective_io_throughput([e for s in stats for e in s.subgroup_io])
        r.kernel_s = sum(s.kernel_seconds for s in stats)
        r.h2d_bytes = sum(s.h2d_bytes for s in stats)
        r.d2h_bytes = sum(s.d2h_bytes for s in stats)
        self._fill_distribution(r)
        return r

    def run(self) -> RunSummary:
        self._preflight()
        self._parallel(lambda w: self.workers[w].init_and_flush_all(self.cfg.seed))
        c = self.cfg
        s = RunSummary(mode=c.mode, iterations=c.iterations, warmup_iterations=c.warmup_iterations,
                       subgroups=c.subgroup_count(), workers=1 if self.rank >= 0 else c.workers_per_node,
                       total_params=c.total_params, subgroup_param_count=c.subgroup_param_count, seed=c.seed)
        for it in range(c.iterations):
            if self.before_iteration:
                self.before_iteration(it, self)
            s.iters.append(self.run_iteration(it))
        s.compute_aggregates()
        return s

    def write_trace(self, path) -> None:
        Path(path).parent.mkdir(parents=True, exist_ok=True)
        self.trace.write(str(path))

    def close(self):
        for w in self.workers:
            w.close()


# ---------------------------------------------------------------------------
# CLI (tools/bench.cpp)


def _apply_overrides(cfg: RunConfig, a) -> None:
    if a.mode:
        cfg.mode = a.mode
    if a.iterations and a.iterations > 0:
        cfg.iterations = a.iterations
    if a.workers and a.workers > 0:
        cfg.workers_per_node = a.workers
    if a.seed is not None and a.seed >= 0:
        cfg.seed = a.seed
    for k in ("enable_caching", "skip_gradients", "atomic_rw", "multi_path"):
        v = getattr(a, k)
        if v is not None:
            setattr(cfg, k, v)


def _print_summary(s: RunSummary) -> None:
    print(f"mode={s.mode} subgroups={s.subgroups} workers={s.workers} params={s.total_params}")
    for r in s.iters:
        tag = " (warmup)" if r.warmup else (" (skipped)" if r.skipped else "")
        print(f"iter {r.iteration:2d}{tag} forward={r.forward_s:.4f}s backward={r.backward_s:.4f}s "
              f"update={r.update_s:.4f}s thru={r.update_throughput_mparams:.1f} Mparams/s hits={r.cache_hits}")
    print(f"mean: iter={s.mean_iter_s:.4f}s forward={s.mean_forward_s:.4f}s backward={s.mean_backward_s:.4f}s "
          f"update={s.mean_update_s:.4f}s thru={s.mean_update_throughput_mparams:.1f} Mparams/s")
    if s.mean_effective_io_bps is not None:
        print(f"mean effective I/O: {s.mean_effective_io_bps / 1e6:.1f} MB/s")


def _rank_path(path: str, rank: int) -> str:
    p = Path(path)
    return str(p.parent / f"{p.stem}.rank{rank}{p.suffix}")


def _cmd_run(a) -> int:
    cfg = RunConfig.from_file(a.config)
    _apply_overrides(cfg, a)
    if a.multiprocess and a.worker_rank < 0:
        procs = []
        for rank in range(cfg.workers_per_node):
            argv = [sys.executable, "-m", "paper_2509_02480_b200.harness", "run", "--config", a.config,
                    "--worker-rank", str(rank)] + _passthrough(a)
            if a.trace_out:
                argv += ["--trace-out", _rank_path(a.trace_out, rank)]
            if a.report_out:
                argv += ["--report-out", os.path.join(a.report_out, f"rank{rank}")]
            procs.append(subprocess.Popen(argv))
        rc = max(p.wait() for p in procs)
        if rc == 0 and a.trace_out:  # merge per-rank traces by timestamp
            rows, header = [], None
            for rank in range(cfg.workers_per_node):
                with open(_rank_path(a.trace_out, rank)) as f:
                    rd = list(csv.reader(f))
                header = rd[0]
                rows += rd[1:]
            rows.sort(key=lambda r: int(r[0]))
            with open(a.trace_out, "w", newline="") as f:
                wtr = csv.writer(f)
                wtr.writerow(header)
                wtr.writerows(rows)
        return rc
    runner = BenchRunner(cfg, a.worker_rank)
    s = runner.run()
    if a.trace_out:
        runner.write_trace(a.trace_out)
    if a.report_out:
        emit_report(s, a.report_out)
    _print_summary(s)
    runner.close()
    return 0


def _passthrough(a) -> list:
    out = []
    if a.mode:
        out += ["--mode", a.mode]
    if a.iterations:
        out += ["--iterations", str(a.iterations)]
    if a.workers:
        out += ["--workers", str(a.workers)]
    if a.seed is not None and a.seed >= 0:
        out += ["--seed", str(a.seed)]
    for k in ("enable_caching", "skip_gradients", "atomic_rw", "multi_path"):
        v = getattr(a, k)
        if v is not None:
            out.append(("--" if v else "--no-") + k.replace("_", "-"))
    return out


def _cmd_probe(a) -> int:
    t = tf.Tier(tf.TierSpec(0, tf.TierKind.local_dir, a.tier))
    r = t.probe_bandwidth(int(a.bytes_mib * 1024 * 1024), a.reps)
    print(json.dumps({"root": a.tier, "read_bw": r.read_bw, "write_bw": r.write_bw,
                      "low_confidence": r.low_confidence}))
    return 0


def _cmd_compare(a) -> int:
    j = compare_reports(load_summary(Path(a.a) / "summary.json" if Path(a.a).is_dir() else a.a),
                        load_summary(Path(a.b) / "summary.json" if Path(a.b).is_dir() else a.b))
    text = json.dumps(j, indent=2)
    if a.out:
        Path(a.out).write_text(text + "\n")
    print(text)
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="harness")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("--config", required=True)
    r.add_argument("--mode", choices=["engine", "baseline"])
    r.add_argument("--trace-out")
    r.add_argument("--report-out")
    r.add_argument("--iterations", type=int)
    r.add_argument("--workers", type=int)
    r.add_argument("--seed", type=int)
    r.add_argument("--multiprocess", action="store_true")
    r.add_argument("--worker-rank", type=int, default=-1)
    for k in ("enable-caching", "skip-gradients", "atomic-rw", "multi-path"):
        dest = k.replace("-", "_")
        r.add_argument(f"--{k}", dest=dest, action="store_true", default=None)
        r.add_argument(f"--no-{k}", dest=dest, action="store_false")
    p = sub.add_parser("probe")
    p.add_argument("--tier", required=True)
    p.add_argument("--bytes-mib", type=float, default=8.0)
    p.add_argument("--reps", type=int, default=3)
    c = sub.add_parser("compare")
    c.add_argument("a")
    c.add_argument("b")
    c.add_argument("--out")
    a = ap.parse_args(argv)
    try:
        return {"run": _cmd_run, "probe": _cmd_probe, "compare": _cmd_compare}[a.cmd](a)
    except tf.Error as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
