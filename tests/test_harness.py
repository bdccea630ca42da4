"""The benchmark driver / config / report layer (paper_2509_02480_b200.harness)
against the reference's test_harness.cpp. CPU tests cover config, metrics and
report emission; -m gpu tests run the engine through the harness."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture
def H(tf):
    from paper_2509_02480_b200 import harness
    return harness


def small_config(H, lock_dir, mode="engine"):
    # test_harness.cpp:31-51
    return H.RunConfig.from_json({
        "model": {"total_params": 12 * 50_000, "subgroup_param_count": 50_000},
        "tiers": [{"kind": "mem_throttled", "read_mb_s": 200, "write_mb_s": 200},
                  {"kind": "mem_throttled", "read_mb_s": 100, "write_mb_s": 100}],
        "schedule": {"pool_slots": 6, "update_threads": 1, "lock_dir": lock_dir},
        "run": {"iterations": 4, "warmup_iterations": 1, "mode": mode, "forward_stub_ms": 0.5, "seed": 77}})


def test_config_parsing_and_validation(H, tmp_path):
    # test_harness.cpp:62-116
    f = tmp_path / "cfg.json"
    f.write_text(json.dumps({
        "model": {"total_params": 1000000, "subgroup_param_count": 300000},
        "tiers": [{"kind": "mem_throttled", "read_mb_s": 200, "write_mb_s": 100},
                  {"kind": "local_dir", "root": "/tmp/tf-x", "io_parallelism": 2}],
        "placement": {"alpha": 0.25, "ratio": [2, 1]},
        "optim": {"lr": 0.01, "beta1": 0.8, "weight_decay": 0.02},
        "schedule": {"pool_slots": 5, "workers_per_node": 2, "update_threads": 3},
        "run": {"iterations": 6, "warmup_iterations": 2, "mode": "baseline", "seed": 9},
        "ablation": {"multi_path": True}}))
    cfg = H.RunConfig.from_file(f)
    assert cfg.total_params == 1_000_000 and cfg.subgroup_count() == 4
    assert cfg.subgroup_params(0) == 300_000 and cfg.subgroup_params(3) == 100_000
    assert cfg.tiers[0].kind == "mem_throttled" and cfg.tiers[1].io_parallelism == 2
    assert cfg.alpha == 0.25 and cfg.ratio == [2, 1] and cfg.optim.lr == 0.01 and cfg.optim.beta1 == 0.8
    assert cfg.workers_per_node == 2 and cfg.mode == "baseline"
    cfg.validate()
    o = cfg.schedule_options()
    assert not o.enable_caching and not o.skip_gradients and o.multi_path
    import copy
    for attr, val in [("warmup_iterations", 6), ("pool_slots", 2), ("mode", "turbo"), ("ratio", [1, 2, 3])]:
        bad = copy.deepcopy(cfg)
        setattr(bad, attr, val)
        with pytest.raises(H.tf.ConfigError):
            bad.validate()
    with pytest.raises(H.tf.ConfigError):
        H.RunConfig.from_file(tmp_path / "missing.json")
    # B200 extensions: device section and per-tier keys
    f.write_text(json.dumps({
        "model": {"total_params": 1000000, "subgroup_param_count": 300000},
        "tiers": [{"kind": "host_dram", "capacity_gb": 2.5},
                  {"kind": "local_dir", "root": "/tmp/tf-y", "lock_device": 1},
                  {"kind": "remote_dir", "root": "/tmp/tf-z", "lock_device": 1}],
        "device": {"hbm_retain": 2, "hbm_cache_slots": 3, "h2d_split": 2}}))
    cfg = H.RunConfig.from_file(f)
    assert cfg.tiers[0].capacity_gb == 2.5 and cfg.tiers[1].lock_device == cfg.tiers[2].lock_device == 1
    assert (cfg.device.hbm_retain, cfg.device.hbm_cache_slots, cfg.device.h2d_split) == (2, 3, 2)
    # the reference's own desk configs parse and validate
    for ref in ("desk.json", "local-dirs.json"):
        p = Path("/root/reference/proj/configs") / ref
        if p.exists():
            H.RunConfig.from_file(p).validate()


def test_lock_dir_precedence(H, monkeypatch):
    cfg = H.RunConfig(lock_dir="/tmp/from-config")
    monkeypatch.setenv("TIERFLOW_LOCK_DIR", "/tmp/from-env")
    assert cfg.resolve_lock_dir() == "/tmp/from-env"
    monkeypatch.delenv("TIERFLOW_LOCK_DIR")
    assert cfg.resolve_lock_dir() == "/tmp/from-config"
    cfg.lock_dir = ""
    assert cfg.resolve_lock_dir()


def test_effective_io_formula(H):
    S = H.tf.SubgroupIoTimes
    assert abs(H.effective_io_throughput([S(0, 1_000_000_000, 0.25, 0.25, True, True)]) - 4e9) < 1
    assert H.effective_io_throughput([S(i, 10, 0, 0, False, False) for i in range(3)]) is None
    assert abs(H.effective_io_throughput([S(0, 100_000_000, 1.0, 1.0, True, True)]) - 100e6) < 1e-3


def test_aggregates_exclude_warmups_and_skips(H):
    # test_harness.cpp:323-341
    R = H.IterationReport
    m1 = R(iteration=1, update_s=2.0, forward_s=1.0, backward_s=1.0, update_throughput_mparams=10)
    s = H.RunSummary(iters=[R(iteration=0, warmup=True, update_s=100.0), m1,
                            R(iteration=2, skipped=True, update_s=50.0),
                            R(iteration=3, update_s=4.0, forward_s=1.0, backward_s=1.0, update_throughput_mparams=20)])
    s.compute_aggregates()
    assert s.mean_update_s == 3.0 and s.mean_iter_s == 5.0 and s.mean_update_throughput_mparams == 15.0


def test_emit_report_deterministic_and_roundtrips(H, tmp_path):
    R = H.IterationReport
    s = H.RunSummary(mode="engine", iterations=4, warmup_iterations=1, subgroups=12, total_params=600000,
                     subgroup_param_count=50000, seed=77,
                     iters=[R(iteration=i, warmup=i == 0, update_s=0.1 * (i + 1), tier_pct=[60.0, 40.0],
                              update_read_bytes=[1, 2], update_write_bytes=[3, 4], backward_write_bytes=[0, 0],
                              flush_allocation=[8, 4], cache_hits=3 * (i > 0), effective_io_bps=1e8 if i else None)
                            for i in range(4)])
    s.compute_aggregates()
    H.emit_report(s, tmp_path / "a")
    H.emit_report(s, tmp_path / "b")
    for f in ("summary.json", "iterations.csv"):
        assert (tmp_path / "a" / f).read_bytes() == (tmp_path / "b" / f).read_bytes()
    lines = [l for l in (tmp_path / "a" / "iterations.csv").read_text().splitlines() if l]
    assert len(lines) == 1 + 4
    back = H.load_summary(tmp_path / "a" / "summary.json")
    assert back.mode == s.mode and back.mean_update_s == s.mean_update_s and back.iters[2].cache_hits == 3


def test_compare_reports(H):
    # test_harness.cpp:378-393
    e = H.RunSummary(mode="engine", mean_iter_s=2.0, mean_update_s=1.5, mean_backward_s=0.2)
    b = H.RunSummary(mode="baseline", mean_iter_s=5.0, mean_update_s=3.0, mean_backward_s=1.0)
    j = H.compare_reports(e, b)
    assert j["speedup_vs_baseline"] == 2.5 and j["update_speedup_vs_baseline"] == 2.0
    assert j["mean_iter_s"] == 2.0 and j["baseline_mean_iter_s"] == 5.0


def test_cli_probe(tmp_path):
    out = subprocess.run([sys.executable, "-m", "paper_2509_02480_b200.harness", "probe", "--tier",
                          str(tmp_path), "--bytes-mib", "4", "--reps", "2"], capture_output=True, text=True,
                         cwd=ROOT, timeout=120)
    assert out.returncode == 0, out.stderr
    j = json.loads(out.stdout)
    assert j["read_bw"] > 0 and j["write_bw"] > 0


# ---------------------------------------------------------------------------


@pytest.mark.gpu
def test_engine_run_distribution_and_hits(H, cuda, lock_dir):
    # test_harness.cpp:153-166
    r = H.BenchRunner(small_config(H, lock_dir))
    s = r.run()
    assert len(s.iters) == 4
    for it in s.iters:
        assert abs(it.host_pct + sum(it.tier_pct) - 100.0) < 0.1
        assert it.cache_hits == (0 if it.iteration == 0 else 3)
        assert it.backward_write_bytes == [0, 0]
    assert s.mean_update_throughput_mparams > 0
    r.close()


@pytest.mark.gpu
def test_baseline_run_byte_accounting(H, cuda, lock_dir):
    # test_harness.cpp:201-218
    r = H.BenchRunner(small_config(H, lock_dir, "baseline"))
    s = r.run()
    P, M = 50_000, 12
    for it in s.iters:
        assert it.host_pct == 0 and it.tier_pct == [100.0, 0.0] and it.cache_hits == 0
        assert it.backward_write_bytes[0] == 4 * P * M
        assert it.update_read_bytes[0] == 16 * P * M and it.update_write_bytes[0] == 12 * P * M
    r.close()


@pytest.mark.gpu
def test_determinism_bytes_and_state(H, cuda, lock_dir):
    # test_harness.cpp:229-248
    runs = []
    for _ in range(2):
        cfg = small_config(H, lock_dir)
        cfg.ratio = [2.0, 1.0]
        r = H.BenchRunner(cfg)
        s = r.run()
        runs.append((s, [r.worker(0).read_current_state(i) for i in r.worker(0).subgroup_ids()]))
        r.close()
    (a, sa), (b, sb) = runs
    for x, y in zip(a.iters, b.iters):
        assert (x.update_read_bytes, x.update_write_bytes, x.backward_write_bytes, x.cache_hits) == \
               (y.update_read_bytes, y.update_write_bytes, y.backward_write_bytes, y.cache_hits)
    for u, v in zip(sa, sb):
        assert np.array_equal(u.view(np.uint32), v.view(np.uint32))


@pytest.mark.gpu
def test_engine_beats_baseline(H, cuda, lock_dir):
    # test_harness.cpp:250-279: >= 1.3x update speedup on the throttled tiers
    def make(mode):
        return H.RunConfig.from_json({
            "model": {"total_params": 350_000 * 12, "subgroup_param_count": 350_000},
            "tiers": [{"kind": "mem_throttled", "read_mb_s": 200, "write_mb_s": 200},
                      {"kind": "mem_throttled", "read_mb_s": 100, "write_mb_s": 100}],
            "schedule": {"pool_slots": 4, "lock_dir": lock_dir},
            "run": {"iterations": 3, "warmup_iterations": 1, "mode": mode, "forward_stub_ms": 0.0}})
    res = {}
    for mode in ("engine", "baseline"):
        r = H.BenchRunner(make(mode))
        res[mode] = r.run().mean_update_s
        r.close()
    assert res["baseline"] / res["engine"] >= 1.3, res


@pytest.mark.gpu
def test_ragged_tail_and_trace_files(H, cuda, lock_dir, tmp_path):
    # test_harness.cpp:281-321
    cfg = small_config(H, lock_dir)
    cfg.total_params = 3 * 50_000 + 20_000
    cfg.iterations, cfg.warmup_iterations = 2, 0
    assert cfg.subgroup_count() == 4 and cfg.subgroup_params(3) == 20_000
    r = H.BenchRunner(cfg)
    r.run()
    assert r.worker(0).read_current_state(3).size == 3 * 20_000
    r.write_trace(tmp_path / "t.csv")
    r.write_trace(tmp_path / "t.jsonl")
    rows = (tmp_path / "t.csv").read_text().splitlines()
    assert rows[0] == "timestamp_ns,worker_id,kind,subgroup_id,tier_id,bytes" and len(rows) - 1 == r.trace.size()
    assert '"kind"' in (tmp_path / "t.jsonl").read_text().splitlines()[0]
    r.close()


@pytest.mark.gpu
def test_gradient_overflow_skips_the_step(H, cuda, lock_dir):
    # test_harness.cpp:343-366
    from cuda.bindings import runtime as rt
    cfg = small_config(H, lock_dir)
    cfg.iterations, cfg.warmup_iterations = 3, 0
    r = H.BenchRunner(cfg)

    def poke(it, runner):
        if it == 1:
            ptr = runner.worker(0).grad_buffer(3)
            val = np.array([0x7C00], np.uint16)
            err, = rt.cudaMemcpy(ptr + 2 * 17, val.ctypes.data, 2, rt.cudaMemcpyKind.cudaMemcpyHostToDevice)
            assert err == rt.cudaError_t.cudaSuccess
    r.after_backward = poke
    s = r.run()
    assert [i.skipped for i in s.iters] == [False, True, False] and s.iters[1].overflow_count >= 1
    for sg in r.worker(0).subgroup_ids():
        assert r.worker(0).meta(sg).step_count == 3  # iterations 0 and 2 applied (t = 1, 3)
    r.close()


@pytest.mark.gpu
def test_multiworker_threads_shard_and_stay_exclusive(H, cuda, lock_dir):
    # test_harness.cpp:424-452
    cfg = small_config(H, lock_dir)
    cfg.workers_per_node = 2
    cfg.iterations, cfg.warmup_iterations = 2, 0
    r = H.BenchRunner(cfg)
    s = r.run()
    assert r.worker_count() == 2 and r.worker(0).subgroup_ids() == list(range(6))
    assert r.worker(1).subgroup_ids()[0] == 6
    held, opened = {}, {}
    for e in r.trace.snapshot():
        if e.kind == H.tf.EventKind.lock_acquire:
            opened[(e.tier_id, e.worker_id)] = e.timestamp_ns
        elif e.kind == H.tf.EventKind.lock_release:
            held.setdefault(e.tier_id, []).append((opened[(e.tier_id, e.worker_id)], e.timestamp_ns))
    for iv in held.values():
        iv.sort()
        assert all(iv[i][1] <= iv[i + 1][0] for i in range(len(iv) - 1))
    assert s.iters[0].cache_hits == 0 and s.iters[1].cache_hits == 6
    r.close()


@pytest.mark.gpu
def test_preflight_rejects_impossible_tier(H, cuda, lock_dir):
    cfg = small_config(H, lock_dir)
    cfg.tiers.append(H.TierConfig(kind="local_dir", root="/proc/tierflow-no-space/x", read_mb_s=1, write_mb_s=1))
    with pytest.raises(H.tf.Error):
        H.BenchRunner(cfg).run()


@pytest.mark.gpu
def test_cli_multiprocess_lock_exclusivity(cuda, tmp_path):
    """acceptance criterion 7, process half: 4 worker processes x 2 tiers via the
    CLI, merged per-rank traces, no overlapping held-lock intervals per tier."""
    cfg = {"model": {"total_params": 24 * 20_000, "subgroup_param_count": 20_000},
           "tiers": [{"kind": "local_dir", "root": str(tmp_path / "t0"), "read_mb_s": 1000, "write_mb_s": 1000},
                     {"kind": "remote_dir", "root": str(tmp_path / "t1"), "read_mb_s": 600, "write_mb_s": 600}],
           "schedule": {"pool_slots": 3, "workers_per_node": 4, "lock_dir": str(tmp_path / "locks")},
           "run": {"iterations": 5, "warmup_iterations": 0, "forward_stub_ms": 0.0}}
    (tmp_path / "cfg.json").write_text(json.dumps(cfg))
    out = subprocess.run([sys.executable, "-m", "paper_2509_02480_b200.harness", "run", "--config",
                          str(tmp_path / "cfg.json"), "--multiprocess", "--trace-out", str(tmp_path / "trace.csv")],
                         capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    rows = [l.split(",") for l in (tmp_path / "trace.csv").read_text().splitlines()[1:]]
    held, opened, n = {}, {}, 0
    for ts, worker, kind, sg, tier, b in rows:
        if kind == "lock_acquire":
            opened[(tier, worker)] = int(ts)
            n += 1
        elif kind == "lock_release":
            held.setdefault(tier, []).append((opened.pop((tier, worker)), int(ts)))
    assert n >= 200 and len({r[1] for r in rows}) == 4
    for iv in held.values():
        iv.sort()
        assert all(iv[i][1] <= iv[i + 1][0] for i in range(len(iv) - 1))
