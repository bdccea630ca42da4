"""bench.py host-side logic (no GPU): workload shapes, the e2e host-memory
sizing rule, and the reference arm's line on a non-zero rank."""
import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def test_workload_shapes_match_survey():
    # C2 = 68 subgroups @100M, last 38,415,616; C3 = 200 @100M
    s = bench.subgroup_sizes(**{k: bench.WORKLOADS["llama2-7b"][k] for k in ("total", "sub")})
    assert len(s) == 68 and s[-1] == 38_415_616 and sum(s) == 6_738_415_616
    s = bench.subgroup_sizes(**{k: bench.WORKLOADS["20b"][k] for k in ("total", "sub")})
    assert len(s) == 200 and set(s) == {100_000_000}
    s = bench.subgroup_sizes(**{k: bench.WORKLOADS["ref-1b"][k] for k in ("total", "sub")})
    assert s == [125_000_000] * 8


def _meminfo(monkeypatch, avail_bytes):
    import builtins
    real_open = builtins.open

    def fake_open(path, *a, **k):
        if path == "/proc/meminfo":
            import io
            return io.StringIO(f"MemTotal: {avail_bytes // 1024} kB\nMemAvailable: {avail_bytes // 1024} kB\n")
        return real_open(path, *a, **k)
    monkeypatch.setattr(builtins, "open", fake_open)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_e2e_shard_fits_host_memory(monkeypatch, world):
    sizes = bench.subgroup_sizes(6_738_415_616, 100_000_000)
    avail = 205 * 2**30
    _meminfo(monkeypatch, avail)
    block = 12 * max(sizes) + 4096
    # mode 1: retained subgroups keep a slot, C <= pool - 3
    sub, pool, cache = bench.e2e_shard(sizes, world, 42, 29, 1)
    assert (pool + len(sub)) * block <= 0.7 * avail / world + block  # every pinned block fits
    assert 1 <= len(sub) <= len(sizes) and sub == sizes[:len(sub)]
    assert pool >= 4 and 0 <= cache <= max(0, pool - 3)
    if world == 1:
        assert (len(sub), pool, cache) == (68, 42, 29)
    # mode 2 (HBM cache, the bench default): C in HBM, no host block for it
    sub, pool, cache = bench.e2e_shard(sizes, world, 16, 29, 2)
    pinned = pool + bench.WRITEBACK_BLOCKS + len(sub) - cache
    assert pinned * block <= 0.7 * avail / world + block
    assert pool >= 4 and cache == min(len(sub) * 29 // 68, 3 * len(sub) // 7)  # the full shard's retained fraction
    if world == 1:
        assert (len(sub), pool) == (68, 16)


def test_e2e_shard_without_meminfo_keeps_request(monkeypatch):
    import builtins
    real_open = builtins.open

    def failing_open(path, *a, **k):
        if path == "/proc/meminfo":
            raise OSError("no procfs")
        return real_open(path, *a, **k)
    monkeypatch.setattr(builtins, "open", failing_open)
    sizes = [100] * 5
    assert bench.e2e_shard(sizes, 4, 16, 13) == (sizes, 16, 13)


def test_reference_arm_nonzero_rank_exits_quietly(monkeypatch, capsys):
    monkeypatch.setenv("RANK", "1")
    assert bench.main(["--impl", "reference"]) == 0
    assert capsys.readouterr().out == ""


def test_metric_is_baseline_metric():
    base = json.loads((ROOT / "BASELINE.json").read_text())
    assert bench.METRIC == base["metric"]
    assert bench.ALG_BYTES_PER_PARAM == 28


def test_llama2_70b_shape():
    # 68,976,648,192 params -> 690 subgroups @100M, the last 76,648,192
    s = bench.subgroup_sizes(**{k: bench.WORKLOADS["llama2-70b"][k] for k in ("total", "sub")})
    assert len(s) == 690 and s[-1] == 76_648_192 and sum(s) == 68_976_648_192
    from paper_2509_02480_b200.parallel import shard
    assert sorted({shard(690, 8, r)[1] for r in range(8)}) == [86, 87]  # uneven at N=8


def test_gpus_must_match_world_size(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    assert bench.main(["--gpus", "1", "--skip-e2e", "--skip-cpu"]) == 2


def test_gpus_n_without_torchrun_spawns_n_ranks(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    seen = {}

    def fake_call(cmd):
        seen["cmd"] = cmd
        return 0
    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    assert bench.main(["--gpus", "4", "--steps", "2", "--warmup", "3"]) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-6:] == ["--gpus", "4", "--steps", "2", "--warmup", "3"]


@pytest.mark.parametrize("world", [1, 2, 8])
def test_both_arms_report_the_same_config(world):
    wl = "llama2-7b" if world == 1 else "20b"
    a = bench.line_config(wl, world, "f16")
    assert a == bench.line_config(wl, world, "f16")
    assert a["subgroups_per_rank"] == (68 if world == 1 else 200 // world)
    assert a["survey_config"] == ("C2" if world == 1 else "C3")


@pytest.mark.parametrize("world,window", [(2, 4), (3, 4), (8, 4), (8, 1)])
def test_rolling_bucket_layout(world, window):
    from paper_2509_02480_b200.parallel import contribution_layout, shard
    sizes = bench.subgroup_sizes(20_000_000_000, 100_000_000)
    offs, total = contribution_layout(sizes, world, window)
    slot = 100_000_000
    assert total == window * world * slot
    for o in range(world):
        b, c = shard(len(sizes), world, o)
        for k in range(c):
            assert offs[b + k] == ((k % window) * world + o) * slot
    # within one bucket step every owner has its own slot: k-th subgroups of all owners never collide
    for k in range(min(shard(len(sizes), world, r)[1] for r in range(world))):
        ids = [shard(len(sizes), world, o)[0] + k for o in range(world)]
        assert len({offs[i] for i in ids}) == world
    offs0, total0 = contribution_layout([10, 3, 8], 2, 0)
    assert offs0 == [0, 16, 24] and total0 == 32
