#!/usr/bin/env python
"""Update-phase benchmark (BASELINE.json metric: update-phase params/s,
device-timed, vs the HBM and PCIe/tier rooflines).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself
under torch.distributed.run with N ranks (one per GPU, NCCL, 127.0.0.1); under
torchrun WORLD_SIZE must equal --gpus.

A step is one update phase over the rank's optimizer state, seeded synthetic
state and 16-bit gradients from the reference generators.

N = 1 (BASELINE configs[1]): Llama-2-7B-shaped state,
6,738,415,616 params in 68 subgroups of 100M (the last 38,415,616).
  value   device-resident update phase: the 68 subgroups' P/m/v, gradients and
          working params resident in HBM (108 GB); the whole-phase non-finite
          check, then one fused sm_100a kernel per subgroup; CUDA events on the
          launching stream. Roofline: HBM, 28 algorithmic bytes/param.
  e2e     the same metric through the engine's C ABI with the state on HOST
          tiers: pinned host DRAM + a local O_DIRECT directory ("NVMe") tier,
          Eq. 1 placing subgroups over both (the DRAM tier's rate is the
          measured PCIe rate; the NVMe tier's rate is learned by the EMA):
          prefetch, H2D, kernel, D2H, flush/retain inside the timed region.
          `streaming_c0` is the same pipeline with no retention (C = 0).
  spill   SURVEY C4: a Llama-2-70B rank's situation, host DRAM capped so the
          state spills to two directory tiers ("NVMe" + "remote"); bounded
          sample of 12 subgroups. Roofline: the directory tiers' probed rates.
N > 1 (BASELINE configs[2]): 20B params, 200 subgroups of 100M,
ZeRO-3 contiguous shards, the gradient reduce-scatter inside the timed phase.
  value   every rank's 16-bit contribution to every subgroup is mapped over
          CUDA IPC (NVLink peer loads); each owner's fused kernel sums the N
          contributions while it streams P/m/v (reduce + update in one pass).
          `exchange_nccl` times NCCL reduce_scatter (pipelined per subgroup on
          a side stream) followed by the single-source kernel.
  e2e     the same through the engine with per-rank tiers (DRAM + NVMe +
          remote) and the owned subgroups bound to the peers' contributions.
cpu_baseline / --impl reference: the reference CPU engine (oracle/_ref: the
unmodified reference headers compiled in place) on the same config: the same
subgroup size, tier kinds and retained fraction, a bounded number of
subgroups, all host threads, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BASE = json.loads((ROOT / "BASELINE.json").read_text())
METRIC = BASE["metric"]
ALG_BYTES_PER_PARAM = 28  # P,m,v fp32 read+write (24) + 16-bit grad read (2) + 16-bit params write (2)
DT = 0  # 16-bit gradient / working-param kind: 0 f16 (the reference's), 1 bf16 (--dtype)

WORKLOADS = {
    "llama2-7b": dict(total=6_738_415_616, sub=100_000_000, survey="C2",
                      desc="Llama-2-7B-shaped optimizer state: 68 subgroups x 100M params (last 38,415,616)"),
    "20b": dict(total=20_000_000_000, sub=100_000_000, survey="C3",
                desc="20B-param optimizer state: 200 subgroups x 100M, ZeRO-3-sharded over the ranks"),
    "llama2-70b": dict(total=68_976_648_192, sub=100_000_000, survey="C4",
                       desc="Llama-2-70B-shaped optimizer state: 690 subgroups x 100M params (last 76,648,192)"),
    "ref-1b": dict(total=1_000_000_000, sub=125_000_000, survey="C1",
                   desc="reference CPU config: 1B params, 8 x 125M"),
    "tiny": dict(total=8 * 10_000_000, sub=10_000_000, survey="-", desc="smoke-sized: 8 subgroups x 10M params"),
}
# e2e defaults (N = 1): HBM cache (hbm_retain 2) holding C = 29 of 68 subgroups
# (35 GB) + 12 ring buffers (14 GB) beside the 27 GB of 16-bit gradients and
# working params: 76 GB of the 180 GB.
RETAINED_FRACTION = 29 / 68


def subgroup_sizes(total: int, sub: int) -> list[int]:
    n = (total + sub - 1) // sub
    return [min(sub, total - k * sub) for k in range(n)]


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# clocks sampled during a timed region


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        if shutil.which("nvidia-smi"):
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(2)

    def summary(self) -> dict:
        sm, mx, power, reasons = [], 0.0, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
                power.append(float(parts[2]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[3:7]):
                if flag.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(power) if power else None}


# ---------------------------------------------------------------------------
# distributed plumbing


def spawn_ranks(argv: list[str], n: int) -> int:
    """--gpus N without a torchrun environment: run this script under
    torch.distributed.run with N ranks on this node (rendezvous on 127.0.0.1)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + list(argv)
    log(f"bench: spawning {n} ranks: {' '.join(cmd)}")
    return subprocess.call(cmd)


def dist_init():
    """One process per GPU over NCCL. TFB_BENCH_BACKEND=gloo folds the local
    ranks onto the visible devices: exercises the multi-rank plumbing on a
    1-GPU box (not a measurement)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    backend = os.environ.get("TFB_BENCH_BACKEND", "nccl")
    ndev = torch.cuda.device_count()
    if world > 1 and backend == "nccl" and ndev < world:
        raise SystemExit(f"bench.py: {world} ranks need {world} visible GPUs, found {ndev}")
    local = local % max(1, ndev)
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _allreduce(world, x: float, op) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=getattr(dist.ReduceOp, op))
    return float(t.item())


def allsum(world, x: float) -> float:
    return _allreduce(world, x, "SUM")


def allmax(world, x: float) -> float:
    return _allreduce(world, x, "MAX")


def allmin(world, x: float) -> float:
    return _allreduce(world, x, "MIN")


def setup_all_ranks(world, fn):
    """Runs one rank's setup; every rank learns whether all succeeded before
    anyone enters the leg's per-phase barriers, so a failure on one rank ends
    the leg everywhere instead of leaving the others waiting."""
    err = None
    try:
        out = fn()
    except Exception as exc:  # reported below on every rank
        out, err = None, exc
    if allmin(world, 0.0 if err else 1.0) < 1.0:
        raise RuntimeError(f"setup failed on a rank: {err}" if err else "setup failed on another rank")
    return out


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def ncu_traffic(params_per_launch: float) -> float | None:
    """DRAM bytes (read + write) per launch of the fused kernel, from the
    committed ncu --set full summary, scaled from its capture size to this
    run's mean launch size (the kernel's traffic is linear in params)."""
    f = ROOT / "profiles" / "ncu_adam_fused.json"
    if f.exists():
        try:
            d = json.loads(f.read_text())
            return round(d["dram_bytes_per_launch"] / d["params_per_launch"] * params_per_launch)
        except Exception:
            return None
    return None


# ---------------------------------------------------------------------------
# value (N = 1): device-resident update phase


def device_leg(tf, sizes, base_id, steps, warmup, seed, rank, world):
    """As the engine's run_update: the whole-phase non-finite check (every
    gradient read once, counted into one device word), then one fused update
    per subgroup that runs only if that word is zero (device-side gate: no host
    round trip between the check and the updates)."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.Stream(dev)
    # 16 B/param resident (P, m, v, gradient, working params); a shard larger
    # than HBM (the 70B shape on one GPU) is timed on the subgroups that fit.
    free, _ = torch.cuda.mem_get_info(dev)
    fit = int((free - 8e9) // (16 * max(sizes) + 8192))
    owned = len(sizes)
    sizes = sizes[:int(allmin(world, max(1, min(len(sizes), fit))))]
    states, grads, p16s = [], [], []
    with torch.cuda.stream(stream):
        for k, n in enumerate(sizes):
            st = torch.empty(3 * n, dtype=torch.float32, device=dev)
            g = torch.empty(n, dtype=torch.int16, device=dev)
            tf.synthetic_state(st[:n], st[n:2 * n], st[2 * n:], seed, base_id + k, stream=stream)
            tf.synthetic_grads(g, seed, base_id + k, 0, dtype=DT, stream=stream)
            states.append(st)
            grads.append(g)
            p16s.append(torch.empty(n, dtype=torch.int16, device=dev))
    counters = torch.zeros(2, dtype=torch.int64, device=dev)
    gate = torch.zeros(1, dtype=torch.int64, device=dev)
    hyper = tf.AdamHyper()
    stream.synchronize()

    def step(t, events=None):
        with torch.cuda.stream(stream):
            gate.zero_()
        for k in range(len(sizes)):
            tf.count_nonfinite16(grads[k], gate, DT, stream=stream)
        for k, n in enumerate(sizes):
            st = states[k]
            if events is not None:
                events[k][0].record(stream)
            tf.adam_fused(st[:n], st[n:2 * n], st[2 * n:], grads[k], p16s[k], t, hyper, DT, DT, counters=counters,
                          stream=stream, gate=gate)
            if events is not None:
                events[k][1].record(stream)

    for w in range(warmup):
        step(w + 1)
    stream.synchronize()
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in sizes]
          for _ in range(steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        start.record(stream)
        for s in range(steps):
            step(warmup + s + 1, ev[s])
        end.record(stream)
        stream.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    total_ms = start.elapsed_time(end)
    kernel_ms = sum(a.elapsed_time(b) for row in ev for a, b in row)
    if int(gate.item()) != 0 or counters[0].item() != 0:
        raise RuntimeError("non-finite gradients in the device leg")
    del states, grads, p16s
    torch.cuda.empty_cache()
    return dict(total_ms=total_ms, kernel_ms=kernel_ms, launches=steps * len(sizes),
                all_launches=2 * steps * len(sizes), clocks=clk.summary(), params=sum(sizes),
                timed_subgroups=len(sizes), owned=owned, copy_sustained_gbs=sustained_copy_gbs(stream, total_ms))


def sustained_copy_gbs(stream, busy_ms):
    """Context for the roofline denominator: a device-to-device copy (read +
    write bytes) run back to back for as long as the timed region, i.e. under
    the same power cap the update phase sees. Not the reported peak."""
    import torch
    n = 1 << 30  # 2 GiB of bf16 each way
    a = torch.empty(n, dtype=torch.bfloat16, device=stream.device)
    b = torch.empty_like(a)
    with torch.cuda.stream(stream):
        b.copy_(a)
        reps = max(4, int(busy_ms / 0.7))  # ~0.7 ms per 4 GiB copy
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            b.copy_(a)
        e1.record(stream)
    stream.synchronize()
    gbs = reps * 4 * n / (e0.elapsed_time(e1) / 1e3) / 1e9
    del a, b
    torch.cuda.empty_cache()
    return round(gbs, 1)


# ---------------------------------------------------------------------------
# value (N > 1): the gradient exchange inside the update phase
#
# Each rank owns the contiguous block parallel.shard() gives it. Every rank's
# 16-bit contribution to a subgroup is the backward's output, emitted bucket
# by bucket: contributions live in a rolling window of buckets
# (PeerGradients(window=W)), so subgroup k of owner o's shard is in bucket
# slot (k % W) * N + o on every rank. Per step either
#   fused  each owner's kernel reads the N contributions of its subgroup
#          (its own from local HBM, N-1 over NVLink peer loads) and sums them
#          while it streams P/m/v: 2(N-1) B/param over NVLink, no collective;
#   nccl   for each k, reduce_scatter of bucket slot block k (N chunks, one
#          per owner) on a side stream into a double-buffered output, the
#          single-source kernel on the compute stream (collective for k+1
#          overlapping kernel k): the collective-then-kernel baseline.
# Contributions are checked finite once by their producer rank (before the
# barrier that publishes them); the owners' kernels count the rounded sums.


EXCHANGE_WINDOW = 4


def exchange_leg(tf, sizes, steps, warmup, seed, rank, world, mode):
    import torch
    import torch.distributed as dist

    from paper_2509_02480_b200 import parallel
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.Stream(dev)
    comm = torch.cuda.Stream(dev)
    M = len(sizes)
    W = EXCHANGE_WINDOW
    slot = (max(sizes) + 7) // 8 * 8
    begin, count = parallel.shard(M, world, rank)
    # HBM: 14 B/param for an owned subgroup (P, m, v + working params) beside
    # the contribution window; a shard that does not fit is timed on the first
    # S subgroups (the same S on every rank).
    free, _ = torch.cuda.mem_get_info(dev)
    window_bytes = 2 * W * world * slot + (4 * slot if mode == "nccl" else 0)
    fit = int((free - window_bytes - 8e9) // (14 * slot + 4096))
    S = int(allmin(world, min(count, max(1, fit))))
    owned = list(range(begin, begin + S))
    states, p16s = [], []
    counters = torch.zeros(2, dtype=torch.int64, device=dev)
    hyper = tf.AdamHyper()
    with torch.cuda.stream(stream):
        for sg in owned:
            n = sizes[sg]
            st = torch.empty(3 * n, dtype=torch.float32, device=dev)
            tf.synthetic_state(st[:n], st[n:2 * n], st[2 * n:], seed, sg, stream=stream)
            states.append(st)
            p16s.append(torch.empty(n, dtype=torch.int16, device=dev))
    pg = parallel.PeerGradients(sizes, world, rank, device=dev.index, dtype="bf16" if DT else "f16", window=W)
    bad = torch.zeros(1, dtype=torch.int64, device=dev)
    with torch.cuda.stream(stream):
        for s_ in range(W * world):  # this rank's contribution in every bucket slot
            buf = pg.slot_view(s_)
            tf.synthetic_grads(buf.view(torch.int16), seed + 100 * rank, s_, 0, dtype=DT, stream=stream)
            tf.count_nonfinite16(buf.view(torch.int16), bad, DT, stream=stream)  # the producer's check
    stream.synchronize()
    if allsum(world, float(bad.item())) != 0:
        raise RuntimeError("non-finite gradient contributions")
    flat = out = None
    if mode == "nccl":
        flat = pg.slot_view(0, W * world)  # the whole window: slot-major, N chunks per bucket
        out = [torch.empty(slot, dtype=flat.dtype, device=dev) for _ in range(2)]
    barrier(world)  # every contribution written before any owner reads it
    kernel_done = [torch.cuda.Event() for _ in range(2)]

    def step(t, events=None):
        for k, sg in enumerate(owned):
            n = sizes[sg]
            st = states[k]
            if mode == "nccl":
                b = k % 2
                blk = flat[(k % W) * world * slot:((k % W) + 1) * world * slot]
                comm.wait_event(kernel_done[b])  # out[b] free: kernel k-2 has read it
                with torch.cuda.stream(comm):
                    work = dist.reduce_scatter_tensor(out[b], blk, op=dist.ReduceOp.SUM, async_op=True)
                with torch.cuda.stream(stream):
                    work.wait()
            if events is not None:
                events[k][0].record(stream)
            if mode == "fused":
                tf.adam_fused_multi(st[:n], st[n:2 * n], st[2 * n:], pg.sources(sg), p16s[k], t, hyper, DT, DT,
                                    counters=counters, stream=stream)
            else:
                tf.adam_fused(st[:n], st[n:2 * n], st[2 * n:], out[k % 2][:n].view(torch.int16), p16s[k], t, hyper,
                              DT, DT, counters=counters, stream=stream)
                kernel_done[k % 2].record(stream)
            if events is not None:
                events[k][1].record(stream)

    for w in range(warmup):
        step(w + 1)
    stream.synchronize()
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in owned]
          for _ in range(steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        start.record(stream)
        for s in range(steps):
            step(warmup + s + 1, ev[s])
        end.record(stream)
        stream.synchronize()
    torch.cuda.synchronize()
    barrier(world)  # no rank frees its contribution while a peer still reads it
    total_ms = start.elapsed_time(end)
    kernel_ms = sum(a.elapsed_time(b) for row in ev for a, b in row)
    if counters[0].item() != 0:
        raise RuntimeError("non-finite gradient sums in the exchange leg")
    pg.close()
    del states, p16s, flat, out
    torch.cuda.empty_cache()
    return dict(total_ms=total_ms, kernel_ms=kernel_ms, launches=steps * len(owned), all_launches=steps * len(owned),
                clocks=clk.summary(), params=sum(sizes[sg] for sg in owned), timed_subgroups=len(owned),
                owned=count)


# ---------------------------------------------------------------------------
# e2e: end to end through the engine C ABI with host tiers


def pcie_probe(trials: int = 3):
    """PCIe ceilings for the pipeline bound: H2D alone, D2H alone, and both at
    once on two streams (the duplex ceiling), 1 GiB page-aligned pinned
    buffers, best of `trials` (a short probe otherwise reads below what a
    long phase sustains)."""
    import torch
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    h2, d2 = torch.empty(n, dtype=torch.uint8, pin_memory=True), torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {"h2d": 0.0, "d2h": 0.0, "bidir": 0.0}
    for _ in range(trials):
        for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                         ("d2h", lambda: h.copy_(d, non_blocking=True))):
            fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(3):
                fn()
            b.record()
            torch.cuda.synchronize()
            out[name] = max(out[name], 3 * n / (a.elapsed_time(b) / 1e3))
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s1.wait_event(a)
        s2.wait_event(a)
        for _ in range(4):
            with torch.cuda.stream(s1):
                d.copy_(h, non_blocking=True)
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        b.record()
        torch.cuda.synchronize()
        out["bidir"] = max(out["bidir"], 8 * n / (a.elapsed_time(b) / 1e3))
    del h, d, h2, d2
    return out


WRITEBACK_BLOCKS = 4  # engine.hpp kWritebackBlocks (HBM cache mode)


def e2e_shard(sizes, world, pool_slots, cache_slots, hbm_retain=2):
    """(subgroups, pool_slots, cache_slots) each rank streams in the e2e leg.
    Host blocks of 12 B/param are pinned by the pool slots, by every subgroup
    on the host-DRAM tier and (HBM cache mode) by the write-back lane; a
    subgroup retained in HBM pins none in mode 2 but keeps its slot in mode 1.
    N ranks on one host share 70% of MemAvailable. When the request does not
    fit, the pool shrinks first (to a third of the rank's blocks, at least 4
    slots) and then the shard."""
    try:
        avail = next(int(l.split()[1]) * 1024 for l in open("/proc/meminfo") if l.startswith("MemAvailable:"))
    except (OSError, StopIteration):
        return sizes, pool_slots, cache_slots
    blocks = int(0.7 * avail / world // (12 * max(sizes) + 4096))
    hbm_cache = hbm_retain == 2 and cache_slots >= 0
    extra = WRITEBACK_BLOCKS if hbm_cache else 0

    def cache_for(n):  # a shrunk shard keeps the requested retained fraction, at most 3/7 of it
        return min(cache_slots, n * cache_slots // len(sizes), 3 * n // 7) if hbm_cache else 0

    def need(pool, n):  # retained in HBM: no host block
        return pool + extra + n - cache_for(n)

    pool = pool_slots
    if need(pool, len(sizes)) > blocks:
        pool = max(4, min(pool_slots, blocks // 3))
    n = len(sizes)
    while n > 1 and need(pool, n) > blocks:
        n -= 1
    if hbm_cache:
        cache = cache_for(n)
    else:
        cache = cache_slots if cache_slots < 0 else min(cache_slots, max(0, pool - 3))
    return sizes[:n], pool, cache


def run_phases(w, world, rank, warmup, steps, backward, tag):
    """Backward (untimed), then run_update timed with CUDA events on the
    legacy stream around the C-ABI call (which returns after the phase's last
    D2H and flush); max over ranks is taken by the caller."""
    import torch
    phases = []
    for it in range(warmup + steps):
        if backward is not None:
            backward(it)
        barrier(world)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        census = w.residency_census() if os.environ.get("TFB_TIMELINE_DIR") else None
        st = w.run_update(it)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        barrier(world)
        if it >= warmup:
            phases.append((ms, st))
        if census is not None:  # diagnostics: every phase's per-subgroup timeline
            d = Path(os.environ["TFB_TIMELINE_DIR"])
            d.mkdir(parents=True, exist_ok=True)
            (d / f"{tag.replace(' ', '_').replace('=', '')}_r{rank}_p{it}.json").write_text(json.dumps(dict(
                ms=ms, hits=st.cache_hits, alloc=st.flush_allocation, census_before=census,
                timeline=w.last_timeline(),
                io=[dict(id=e.id, read_s=e.read_seconds, write_s=e.write_seconds, fetched=e.fetched,
                         flushed=e.flushed) for e in st.subgroup_io])))
        log(f"[rank {rank}] {tag} phase {it}: {ms:.0f} ms, hits {st.cache_hits}, alloc {st.flush_allocation}, "
            f"kernel {st.kernel_seconds*1e3:.0f} ms, h2d {st.h2d_seconds*1e3:.0f} ms, d2h {st.d2h_seconds*1e3:.0f} ms")
    return phases


def pipeline_roofline(phases, pcie, dir_probes):
    """Per-phase bound: PCIe (each direction's bytes over its measured rate,
    and both over the duplex ceiling) against the directory tiers (bytes
    actually moved over the probed rates; tiers sharing one physical device
    add up). The host_dram tier moves subgroups by block exchange: its cost is
    the PCIe leg."""
    h2d_b = statistics.mean(p[1].h2d_bytes for p in phases)
    d2h_b = statistics.mean(p[1].d2h_bytes for p in phases)
    pcie_s = max(h2d_b / pcie["h2d"], d2h_b / pcie["d2h"], (h2d_b + d2h_b) / pcie["bidir"])
    tier_s, per_tier = 0.0, []
    for i, pr in dir_probes.items():
        rb = statistics.mean(p[1].tier_obs[i].read_bytes for p in phases)
        wb = statistics.mean(p[1].tier_obs[i].write_bytes for p in phases)
        sec = rb / pr.read_bw + wb / pr.write_bw
        tier_s += sec  # one device holds every directory tier here
        per_tier.append(dict(tier=i, read_bytes=rb, write_bytes=wb, read_gbs=round(pr.read_bw / 1e9, 2),
                             write_gbs=round(pr.write_bw / 1e9, 2), seconds=round(sec, 4)))
    return dict(h2d=h2d_b, d2h=d2h_b, pcie_s=pcie_s, tier_s=tier_s, bound_s=max(pcie_s, tier_s), per_tier=per_tier)


def e2e_leg(tf, sizes, base_id, steps, warmup, seed, rank, world, tier_root, pool_slots, cache_slots, ring,
            hbm_retain=2, peer=None, remote=False, c0_steps=0, host_grads=False):
    """peer: a parallel.PeerGradients holding every rank's contribution to
    every subgroup: the engine's owned subgroups are bound to the world's
    contributions, so each update reduces them over CUDA IPC / NVLink inside
    the kernel. remote: a third ("remote_dir") tier beside DRAM and NVMe
    (SURVEY C3). c0_steps > 0: afterwards, the same engine with no retention
    (C = 0) for c0_steps timed phases."""
    # The bandwidth EMA settles the NVMe tier's rate over the first phases
    # (paper §3.3); time the converged pipeline.
    warmup = max(warmup, 5)
    import torch
    dev = torch.cuda.current_device()
    pcie = pcie_probe()
    root = Path(tier_root) / f"rank{rank}"
    if root.exists():
        shutil.rmtree(root)
    root.mkdir(parents=True)
    dirs = [tf.Tier(tf.TierSpec(1, tf.TierKind.local_dir, str(root / "nvme"), 0.0, 0.0, io_parallelism=4,
                                lock_device=1))]
    if remote:
        dirs.append(tf.Tier(tf.TierSpec(2, tf.TierKind.remote_dir, str(root / "remote"), 0.0, 0.0, io_parallelism=4,
                                        lock_device=1)))
    probes = {t.id(): t.probe_bandwidth(1 << 30, 3) for t in dirs}
    # Host DRAM tier: blocks move by exchange; Eq. 1 sees it at the measured
    # PCIe rate (the engine keeps a host_dram tier's configured rate).
    dram_bw = min(pcie["h2d"], pcie["d2h"])
    dram = tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", dram_bw, dram_bw))
    trace = tf.EventTrace()
    # One lock directory for the node: the ranks' directory tiers on one
    # physical disk (lock_device 1) share one semaphore, the paper's
    # node-level contention control, although their paths are per rank.
    opt = tf.ScheduleOptions(pool_slots=pool_slots, cache_slots=cache_slots,
                             lock_dir=str(Path(tier_root) / "e2e_locks"))
    t0 = time.time()

    def setup():
        w = tf.OffloadWorker(rank, [dram] + dirs, opt, tf.AdamHyper(), trace,
                             tf.DeviceOptions(dev, DT, DT, ring, 0, 1, hbm_retain, host_grads=host_grads))
        for k, n in enumerate(sizes):
            w.add_subgroup(base_id + k, n)
        w.init_and_flush_all(seed)
        if peer is not None:
            peer.bind(w, [base_id + k for k in range(len(sizes))])
        return w
    w = setup_all_ranks(world, setup)
    init_s = time.time() - t0
    log(f"[rank {rank}] e2e init {init_s:.1f}s, probes " +
        ", ".join(f"tier {i}: r={p.read_bw/1e9:.2f} w={p.write_bw/1e9:.2f} GB/s" for i, p in probes.items()) +
        f", pcie h2d={pcie['h2d']/1e9:.1f} d2h={pcie['d2h']/1e9:.1f} bidir={pcie['bidir']/1e9:.1f} GB/s")
    src = tf.SyntheticGradSource(seed)
    backward = None if peer is not None else (lambda it: w.run_backward_sim(it, src, 1))
    phases = run_phases(w, world, rank, warmup, steps, backward, "e2e")
    if os.environ.get("TFB_TIMELINE"):  # diagnostics: the last phase's per-subgroup timeline
        st = phases[-1][1]
        Path(os.environ["TFB_TIMELINE"]).write_text(json.dumps(dict(
            ms=phases[-1][0], alloc=st.flush_allocation, timeline=w.last_timeline(),
            io=[dict(id=e.id, read_s=e.read_seconds, write_s=e.write_seconds, fetched=e.fetched, flushed=e.flushed)
                for e in st.subgroup_io])))
    rl = pipeline_roofline(phases, pcie, probes)
    last = phases[-1][1]
    M = len(sizes)
    res = dict(ms=statistics.mean(p[0] for p in phases), params=sum(sizes), h2d=int(rl["h2d"]), d2h=int(rl["d2h"]),
               init_s=init_s, hits=statistics.mean(p[1].cache_hits for p in phases), alloc=last.flush_allocation,
               retained=last.retained, pcie=pcie, probes={i: (p.read_bw, p.write_bw) for i, p in probes.items()},
               bound_ms=rl["bound_s"] * 1e3, pcie_bound_ms=rl["pcie_s"] * 1e3, tier_bound_ms=rl["tier_s"] * 1e3,
               per_tier=rl["per_tier"], kernel_ms=statistics.mean(p[1].kernel_seconds for p in phases) * 1e3,
               launches=len(phases) * M, tier_read_bytes=sum(o.read_bytes for o in last.tier_obs),
               tier_write_bytes=sum(o.write_bytes for o in last.tier_obs), subgroups=M)
    if c0_steps > 0:
        w.set_cache_slots(0)
        ph0 = run_phases(w, world, rank, 2, c0_steps, backward, "e2e C=0")
        if os.environ.get("TFB_TIMELINE_C0"):  # diagnostics: the last C = 0 phase's timeline
            st = ph0[-1][1]
            Path(os.environ["TFB_TIMELINE_C0"]).write_text(json.dumps(dict(
                ms=ph0[-1][0], alloc=st.flush_allocation, timeline=w.last_timeline(),
                io=[dict(id=e.id, read_s=e.read_seconds, write_s=e.write_seconds, fetched=e.fetched,
                         flushed=e.flushed) for e in st.subgroup_io])))
        rl0 = pipeline_roofline(ph0, pcie, probes)
        res["c0"] = dict(ms=statistics.mean(p[0] for p in ph0), h2d=int(rl0["h2d"]), d2h=int(rl0["d2h"]),
                         bound_ms=rl0["bound_s"] * 1e3, pcie_bound_ms=rl0["pcie_s"] * 1e3,
                         tier_bound_ms=rl0["tier_s"] * 1e3, alloc=ph0[-1][1].flush_allocation,
                         hits=statistics.mean(p[1].cache_hits for p in ph0))
        res["launches"] += len(ph0) * M
    w.close()
    del w
    shutil.rmtree(root, ignore_errors=True)
    return res


def e2e_line(r, world, extra):
    e_ms = allmax(world, r["ms"])
    line = {"value": allsum(world, r["params"]) / (e_ms / 1e3), "unit": "params/s",
            "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"], "ms_per_step": round(e_ms, 2),
            "pipeline_bound_ms": round(r["bound_ms"], 1), "pipeline_frac": round(r["bound_ms"] / e_ms, 4),
            "pcie_bound_ms": round(r["pcie_bound_ms"], 1), "tier_bound_ms": round(r["tier_bound_ms"], 1),
            "per_tier": r["per_tier"],
            "tier_bytes_per_step": {"read": r["tier_read_bytes"], "write": r["tier_write_bytes"]},
            "cache_hits_per_phase": r["hits"], "flush_allocation": r["alloc"], "retained": r["retained"],
            "pcie_gbs": {k: round(v / 1e9, 1) for k, v in r["pcie"].items()},
            "kernel_ms_per_phase": round(r["kernel_ms"], 2), "init_s": round(r["init_s"], 1),
            "gpu_launches": r["launches"], "subgroups_per_rank": r["subgroups"]}
    if "c0" in r:
        c0 = r["c0"]
        c_ms = allmax(world, c0["ms"])
        line["streaming_c0"] = {"value": allsum(world, r["params"]) / (c_ms / 1e3), "unit": "params/s",
                                "ms_per_step": round(c_ms, 2), "h2d_bytes_per_step": c0["h2d"],
                                "d2h_bytes_per_step": c0["d2h"], "pipeline_bound_ms": round(c0["bound_ms"], 1),
                                "pipeline_frac": round(c0["bound_ms"] / c_ms, 4),
                                "tier_bound_ms": round(c0["tier_bound_ms"], 1), "flush_allocation": c0["alloc"],
                                "cache_hits_per_phase": c0["hits"],
                                "note": "same engine, retention capacity C = 0: every subgroup streams both ways"}
    line.update(extra)
    return line


# ---------------------------------------------------------------------------
# spill: a capacity-capped host-DRAM tier and a few pinned staging
# slots, so Eq. 1 spills the state to two directory tiers (local "NVMe" +
# "remote"); the retention capacity held in HBM (hbm_retain=2). Tier-bound;
# bounded sample of a Llama-2-70B rank at N=4 (173 subgroups: ~80 fit the HBM
# beside the 16-bit gradient/param arenas, i.e. ~46% retained; host DRAM
# capped to a third of the rest).


def spill_leg(tf, sizes, base_id, rank, world, tier_root, seed, warmup=4, steps=4, pool=8, ring=4, M=12,
              lock_width=1):
    """SURVEY C4 sample. warmup 4: the first phases write subgroup files to
    tiers they have not been on yet (a fresh file is allocated on first
    write: 4.1 vs 5.5 GB/s for an in-place overwrite); the
    timed phases see the steady state, where every file is overwritten in
    place."""
    import torch
    dev = torch.cuda.current_device()
    root = Path(tier_root) / f"spill_rank{rank}"
    shutil.rmtree(root, ignore_errors=True)
    root.mkdir(parents=True)
    # Bounded by the disk the ranks share (at most half its free space): when
    # N ranks' full-size subgroups do not fit, the subgroups shrink rather
    # than the sample (params/s stays comparable).
    free = shutil.disk_usage(root).free
    sub = min(max(sizes), int(0.5 * free / world / M // 12) // 4096 * 4096)
    sub = int(allmin(world, sub))  # the same sample on every rank
    if sub < 1_000_000:
        raise RuntimeError(f"not enough free disk for the spill sample ({free / 1e9:.1f} GB)")
    sizes = [sub] * M
    cache = M // 2  # HBM retention: ~46% of a 70B rank at N=4
    dram_cap = max(1, (M - cache) // 3)  # host DRAM holds a third of the rest
    block = 4096 * ((32 + 12 * max(sizes) + 4095) // 4096)
    for d in ("nvme", "remote"):
        (root / d).mkdir()
    # Tiers on one physical device share one semaphore (contention control
    # per device, TierSpec.lock_device): their transfers take turns instead of
    # seeking against each other.
    same_device = os.stat(root / "nvme").st_dev == os.stat(root / "remote").st_dev
    lock_dev = 1 if same_device else 0
    dirs = [tf.Tier(tf.TierSpec(1, tf.TierKind.local_dir, str(root / "nvme"), 0.0, 0.0, io_parallelism=4,
                                lock_width=lock_width, lock_device=lock_dev)),
            tf.Tier(tf.TierSpec(2, tf.TierKind.remote_dir, str(root / "remote"), 0.0, 0.0, io_parallelism=4,
                                lock_width=lock_width, lock_device=lock_dev))]
    probes = [t.probe_bandwidth(1 << 30, 3) for t in dirs]
    dram = tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 50e9, 50e9, capacity_bytes=dram_cap * block))
    tiers = [dram] + dirs
    trace = tf.EventTrace()
    # One lock directory for every rank of the node: with lock_device, the
    # ranks' tiers on one physical disk share one semaphore (the paper's
    # node-level contention control) even though their paths are partitioned.
    opt = tf.ScheduleOptions(pool_slots=pool, cache_slots=cache, lock_dir=str(Path(tier_root) / "spill_locks"))

    def setup():
        w = tf.OffloadWorker(rank, tiers, opt, tf.AdamHyper(), trace, tf.DeviceOptions(dev, DT, DT, ring, 0, 1, 2))
        for k, n in enumerate(sizes):
            w.add_subgroup(base_id + k, n)
        w.init_and_flush_all(seed)
        return w
    w = setup_all_ranks(world, setup)
    src = tf.SyntheticGradSource(seed)
    phases = run_phases(w, world, rank, warmup, steps, lambda it: w.run_backward_sim(it, src, 1), "spill")
    timeline = [dict(ms=round(ms, 1), io=[dict(id=e.id, read_s=round(e.read_seconds, 4),
                                                 write_s=round(e.write_seconds, 4)) for e in st.subgroup_io])
                for ms, st in phases[-1:]]
    w.close()
    del w
    shutil.rmtree(root, ignore_errors=True)
    ms = statistics.mean(p[0] for p in phases)
    per_tier = []
    for i, pr in enumerate(probes, start=1):  # tier 0 (host DRAM) moves blocks by exchange: no tier time
        rb = statistics.mean(p[1].tier_obs[i].read_bytes for p in phases)
        wb = statistics.mean(p[1].tier_obs[i].write_bytes for p in phases)
        per_tier.append(dict(read_bytes=rb, write_bytes=wb, read_gbs=round(pr.read_bw / 1e9, 2),
                             write_gbs=round(pr.write_bw / 1e9, 2), seconds=rb / pr.read_bw + wb / pr.write_bw))
    parallel_s = max(t["seconds"] for t in per_tier)
    # One physical device: its ceiling is the best rate any probe of it saw,
    # and every rank's tier roots sit under the one tier_root (the node's
    # bytes share it).
    dev_r = max(pr.read_bw for pr in probes)
    dev_w = max(pr.write_bw for pr in probes)
    rb_all = allsum(world, sum(t["read_bytes"] for t in per_tier))
    wb_all = allsum(world, sum(t["write_bytes"] for t in per_tier))
    serial_s = rb_all / dev_r + wb_all / dev_w
    bound_s = serial_s if same_device else parallel_s
    return dict(ms=ms, params=sum(sizes), subgroups=M, subgroup_params=sub, cache=cache, pool=pool,
                same_device=same_device, lock_device=lock_dev, dram_cap=dram_cap,
                bound_ms=bound_s * 1e3, independent_bound_ms=parallel_s * 1e3, per_tier=per_tier,
                hits=statistics.mean(p[1].cache_hits for p in phases), alloc=phases[-1][1].flush_allocation,
                launches=(warmup + steps) * M, phase_ms=[round(p[0], 1) for p in phases], last_phase_io=timeline)


# ---------------------------------------------------------------------------
# reference CPU engine (oracle/_ref), same config, bounded sample


def reference_sample(wl, world, steps, warmup, tier_root, seed=42, n_sub=7):
    """The reference OffloadWorker::run_update on the line's config: the same
    subgroup size, tier kinds (host DRAM as the reference's in-memory tier at
    the PCIe rate our DRAM tier is given, a local directory tier as NVMe, and
    a remote directory tier at N > 1) and retained fraction, on n_sub
    subgroups (7 = 3 retained + 4 streamed, i.e. the 29/68 of the C2 line),
    all host threads. Gradients come from one backward and are reused by the
    later phases (the update's cost does not depend on their values)."""
    import oracle
    threads = os.cpu_count() or 1
    root = Path(tier_root) / "ref"
    shutil.rmtree(root, ignore_errors=True)
    root.mkdir(parents=True)
    sub = wl["sub"]
    C = max(1, round(n_sub * RETAINED_FRACTION))
    tiers = [dict(kind=2, read_bps=50e9, write_bps=50e9), dict(kind=0, root=str(root / "nvme"), io_parallelism=4)]
    if world > 1:
        tiers.append(dict(kind=1, root=str(root / "remote"), io_parallelism=4))
    t0 = time.time()
    res = oracle.run_ref_engine([sub] * n_sub, tiers, pool_slots=C + 3, cache_slots=C, update_threads=threads,
                                lock_dir=str(root / "locks"), seed=seed, iterations=warmup + steps,
                                want_states=False, events_cap=1, backward_once=True)
    wall = time.time() - t0
    shutil.rmtree(root, ignore_errors=True)
    its = res["iters"][warmup:]
    per = [it["params_updated"] / it["update_seconds"] for it in its]
    return dict(value=statistics.mean(per), update_s=[it["update_seconds"] for it in its], cores=threads,
                params=n_sub * sub, wall=wall, alloc=its[-1]["flush_allocation"],
                sample=(f"reference OffloadWorker::run_update (oracle/_ref), {n_sub} subgroups x {sub:,} params, "
                        f"C={C} retained (pool {C + 3}), tiers [mem_throttled 50 GB/s as host DRAM, local_dir"
                        f"{', remote_dir' if world > 1 else ''}], update_threads={threads}, "
                        f"{steps} timed of {warmup + steps} phases"))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def line_config(wl_name, world, dtype):
    """The workload both arms report (identical dicts)."""
    wl = WORKLOADS[wl_name]
    sizes = subgroup_sizes(wl["total"], wl["sub"])
    from paper_2509_02480_b200.parallel import shard
    per_rank = len(sizes) if world == 1 else shard(len(sizes), world, 0)[1]
    return {"workload": wl["desc"], "survey_config": wl["survey"], "params_total": sum(sizes),
            "subgroup_params": wl["sub"], "subgroups_per_rank": per_rank, "grad_dtype": dtype, "param_dtype": dtype,
            "tiers": "host DRAM + local NVMe" + (" + remote" if world > 1 else ""),
            "retained_fraction": round(RETAINED_FRACTION, 4) if world == 1 else None,
            "l2": "inputs larger than L2 (>= 1.2 GB of state per subgroup launch vs 126 MB L2; no flush needed)",
            "parallelism": (f"zero3-shard x{world}" + (", gradient reduce-scatter in the update" if world > 1 else ""))}


# ---------------------------------------------------------------------------


def reference_main(a, wl_name):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    world = a.gpus
    r = reference_sample(WORKLOADS[wl_name], world, a.steps, a.warmup, a.tier_root)
    line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": "params/s",
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": statistics.mean(r["update_s"]) * 1e3, "higher_is_better": True,
            "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generators)", "config": line_config(wl_name, world, a.dtype),
            "cpu_baseline": {"value": r["value"], "unit": "params/s", "cores": r["cores"], "kind": "reference",
                             "sample": r["sample"], "cpu": cpu_model()},
            "e2e": {"value": r["value"], "unit": "params/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=None,
                    help="default: llama2-7b (C2) at N=1, 20b (C3) at N>1")
    ap.add_argument("--tier-root", default=os.environ.get("TFB_TIER_ROOT", str(ROOT / "gpurun_out" / "bench_tiers")))
    ap.add_argument("--pool-slots", type=int, default=16)
    ap.add_argument("--cache-slots", type=int, default=29,
                    help="retention capacity C (HBM cache); -1: pool_slots - 3 (reference default)")
    ap.add_argument("--ring", type=int, default=12)
    ap.add_argument("--hbm-retain", type=int, default=2,
                    help="0 host retention, 1 HBM retention with a reserved host slot, 2 HBM cache")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--dtype", choices=["f16", "bf16"], default="f16",
                    help="16-bit gradient and working-param kind (f16 = the reference's fp16)")
    ap.add_argument("--exchange", choices=["none", "fused", "nccl"], default=None,
                    help="gradient reduce-scatter in the update (default: none at N=1, fused at N>1; "
                         "at N>1 the nccl form is also timed unless --skip-nccl)")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-spill", action="store_true", help="skip the directory-tier spill sample (SURVEY C4)")
    ap.add_argument("--spill-lock-width", type=int, default=1,
                    help="concurrent transfers the spill sample's device semaphore admits")
    ap.add_argument("--skip-nccl", action="store_true")
    ap.add_argument("--c0-steps", type=int, default=5, help="timed phases of the C=0 streaming e2e (0: skip)")
    ap.add_argument("--host-grads", action="store_true",
                    help="e2e: 16-bit gradients and working params in pinned host memory, streamed with the state")
    a = ap.parse_args(argv)

    global DT
    DT = 1 if a.dtype == "bf16" else 0
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and a.gpus > 1 and a.impl == "ours":
        return spawn_ranks(argv, a.gpus)
    world_env = int(env_world or 1)
    if a.impl == "ours" and world_env != a.gpus:
        log(f"bench.py: WORLD_SIZE={world_env} but --gpus {a.gpus}")
        return 2
    wl_name = a.workload or ("llama2-7b" if a.gpus == 1 else "20b")
    if a.impl == "reference":
        return reference_main(a, wl_name)

    wl = WORKLOADS[wl_name]
    sizes = subgroup_sizes(wl["total"], wl["sub"])
    world, rank, local = dist_init()
    import torch
    from paper_2509_02480_b200 import build as _build
    if rank == 0 and not _build.up_to_date():
        _build.build()
    barrier(world)
    from paper_2509_02480_b200 import parallel
    from paper_2509_02480_b200 import tierflow as tf
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device")
    torch.cuda.set_device(local)
    exchange = a.exchange or ("none" if world == 1 else "fused")

    pk = peaks()
    alg_bytes = ALG_BYTES_PER_PARAM
    nccl_line = None
    if exchange == "none":
        # weak scaling: every rank its own copy of the workload's shape
        base_id = rank * len(sizes)
        dl = device_leg(tf, sizes, base_id, a.steps, a.warmup, a.seed, rank, world)
        scaling = "weak"
    else:
        dl = exchange_leg(tf, sizes, a.steps, a.warmup, a.seed, rank, world, exchange)
        if exchange == "fused":  # own contribution local, N-1 over NVLink, P/m/v 24, params 2
            alg_bytes = 26 + 2 * world
        scaling = "strong"
        if world > 1 and exchange == "fused" and not a.skip_nccl:
            try:
                nl = exchange_leg(tf, sizes, a.steps, a.warmup, a.seed, rank, world, "nccl")
                n_ms = allmax(world, nl["total_ms"] / a.steps)
                nccl_line = {"value": allsum(world, nl["params"]) / (n_ms / 1e3), "unit": "params/s",
                             "ms_per_step": n_ms, "kernel_ms_per_step": nl["kernel_ms"] / a.steps,
                             "path": "NCCL reduce_scatter per subgroup bucket (side stream, double-buffered), "
                                     "then the single-source fused kernel"}
            except Exception as exc:
                nccl_line = {"error": f"{type(exc).__name__}: {exc}"}
                log(f"nccl exchange leg failed: {exc}")
    step_ms = allmax(world, dl["total_ms"] / a.steps)
    value = allsum(world, dl["params"]) / (step_ms / 1e3)
    kernel_s_per_launch = dl["kernel_ms"] / 1e3 / max(1, dl["launches"])
    params_per_launch = dl["params"] / max(1, dl["timed_subgroups"])
    achieved = alg_bytes * params_per_launch / kernel_s_per_launch / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": ncu_traffic(params_per_launch),
                "peak_source": pk["source"], "alg_bytes_per_param": alg_bytes,
                "kernel": (f"adam_fused_kernel (float4 quads, 4 CTAs x 256 threads per SM; binary64 element math, "
                           f"constant-divisor quotients; {world} gradient sources summed in-kernel, {world - 1} "
                           f"read from the peers' NVLink-mapped memory)" if exchange == "fused" else
                           "adam_staged_kernel (P, m, v, g tiles of 2048 params staged in shared memory by "
                           "cp.async.bulk, 2 stages per CTA, 2 CTAs x 512 threads per SM; binary64 element math, "
                           "constant-divisor quotients)"),
                "traffic_source": "profiles/ncu_adam_fused.json (ncu --set full, dram bytes per 100M-param launch)",
                "copy_sustained_gbs": dl.get("copy_sustained_gbs"),
                "frac_of_copy_sustained": (round(achieved / dl["copy_sustained_gbs"], 4)
                                           if dl.get("copy_sustained_gbs") else None)}

    # The spill leg runs before the e2e leg: its disk-bound phases are then
    # not measured behind the e2e leg's directory-tier writes still draining
    # on the box's (virtualised) disk.
    spill = None
    if exchange == "none" and not a.skip_spill:
        try:
            r = spill_leg(tf, sizes, rank * len(sizes), rank, world, a.tier_root, a.seed,
                          lock_width=a.spill_lock_width)
            s_ms = allmax(world, r["ms"])
            spill = {"value": allsum(world, r["params"]) / (s_ms / 1e3), "unit": "params/s",
                     "ms_per_step": round(s_ms, 1), "phase_ms": r["phase_ms"],
                     "tier_bound_ms": round(r["bound_ms"], 1), "tier_frac": round(r["bound_ms"] / s_ms, 4),
                     "independent_tier_bound_ms": round(r["independent_bound_ms"], 1),
                     "tiers_share_one_device": r["same_device"], "device_semaphore": bool(r["lock_device"]),
                     "per_tier": r["per_tier"], "subgroups_per_rank": r["subgroups"],
                     "subgroup_params": r["subgroup_params"], "cache_slots": r["cache"], "pool_slots": r["pool"],
                     "dram_tier_capacity_subgroups": r["dram_cap"], "cache_hits_per_phase": r["hits"],
                     "flush_allocation": r["alloc"], "gpu_launches": r["launches"],
                     "last_phase_io": r["last_phase_io"],
                     "workload": WORKLOADS["llama2-70b"]["desc"] + ": a rank at N=4 (173 subgroups, ~46% fit the "
                                 "HBM cache), bounded sample of 12 subgroups, 6 retained in HBM, host DRAM capped",
                     "path": "C ABI tfg_engine_run_update, tiers [host_dram capped, local_dir O_DIRECT, "
                             "remote_dir O_DIRECT], retention in HBM (hbm_retain=2)"}
        except Exception as exc:
            spill = {"error": f"{type(exc).__name__}: {exc}"}
            log(f"spill leg failed: {exc}")

    e2e = None
    if not a.skip_e2e:
        try:
            if exchange == "none":
                e_sizes, pool, cache = e2e_shard(sizes, world, a.pool_slots, a.cache_slots, a.hbm_retain)
                # every rank streams the same shard shape (MemAvailable is read at slightly different times)
                n_e = int(allmin(world, len(e_sizes)))
                pool = int(allmin(world, pool))
                cache = int(allmin(world, cache)) if cache >= 0 else cache
                e_sizes = e_sizes[:n_e]
                r = e2e_leg(tf, e_sizes, rank * len(sizes), a.steps, a.warmup, a.seed, rank, world, a.tier_root,
                            pool, cache, a.ring, a.hbm_retain, c0_steps=min(a.c0_steps, a.steps),
                            host_grads=a.host_grads)
                e2e = e2e_line(r, world, {"hbm_retain": a.hbm_retain, "pool_slots": pool, "cache_slots": cache,
                                          "ring": a.ring,
                                          "path": "C ABI tfg_engine_run_update, tiers [host_dram pinned, "
                                                  "local_dir O_DIRECT], Eq. 1 over both"})
            elif exchange == "fused":
                begin, count = parallel.shard(len(sizes), world, rank)
                owned = sizes[begin:begin + count]
                e_sizes, pool, cache = e2e_shard(owned, world, a.pool_slots, a.cache_slots, a.hbm_retain)
                n_e = int(allmin(world, len(e_sizes)))
                pool = int(allmin(world, pool))
                cache = int(allmin(world, cache)) if cache >= 0 else cache
                e_sizes = e_sizes[:n_e]
                with parallel.PeerGradients(sizes, world, rank, device=torch.cuda.current_device(),
                                            dtype="bf16" if DT else "f16", window=EXCHANGE_WINDOW) as pg:
                    for s_ in range(EXCHANGE_WINDOW * world):
                        tf.synthetic_grads(pg.slot_view(s_).view(torch.int16), a.seed + 100 * rank, s_, 0, dtype=DT)
                    torch.cuda.synchronize()
                    barrier(world)  # every contribution written before any owner reads it
                    r = e2e_leg(tf, e_sizes, begin, a.steps, a.warmup, a.seed, rank, world, a.tier_root, pool, cache,
                                a.ring, a.hbm_retain, peer=pg, remote=True)
                    barrier(world)  # no rank frees its contribution while a peer may still read it
                e2e = e2e_line(r, world, {"hbm_retain": a.hbm_retain, "pool_slots": pool, "cache_slots": cache,
                                          "ring": a.ring, "gradient_sources": world,
                                          "path": "C ABI tfg_engine_run_update with bind_grad_sources (fused "
                                                  "reduce-scatter over CUDA IPC), tiers [host_dram pinned, "
                                                  "local_dir O_DIRECT, remote_dir O_DIRECT]"})
            else:
                e2e = {"skipped": "--exchange nccl times the device-resident update only"}
        except Exception as exc:  # keep the device-timed line; report the failure
            e2e = {"error": f"{type(exc).__name__}: {exc}"}
            log(f"e2e leg failed: {exc}")

    e2e_launches = (e2e or {}).get("gpu_launches", 0) + (spill or {}).get("gpu_launches", 0)
    cpu = None
    if rank == 0 and not a.skip_cpu:
        try:
            r = reference_sample(wl, world, 2, 1, a.tier_root)  # 2 timed phases (~11 s of CPU work)
            cpu = {"value": r["value"], "unit": "params/s", "cores": r["cores"], "kind": "reference",
                   "sample": r["sample"], "cpu": cpu_model()}
        except Exception as exc:
            cpu = {"error": f"{type(exc).__name__}: {exc}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "params/s", "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded reference generators: synthetic_param_init, SyntheticGradSource)",
                "config": line_config(wl_name, world, a.dtype),
                "value_setup": {"state": "fp32 P/m/v resident in HBM", "exchange": exchange,
                                "subgroups_timed_per_rank": dl["timed_subgroups"],
                                "owned_per_rank": dl.get("owned", dl["timed_subgroups"]),
                                "params_timed_per_rank": dl["params"],
                                "nonfinite_check": ("whole-phase count kernel, device-side gate on the updates"
                                                    if exchange == "none" else
                                                    "each contribution checked by its producer rank; owners count "
                                                    "the rounded sums in-kernel")},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "spill": spill,
                "gpu_launches": dl.get("all_launches", dl["launches"]) + e2e_launches,
                "clocks": dl["clocks"]}
        if nccl_line is not None:
            line["exchange_nccl"] = nccl_line
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
