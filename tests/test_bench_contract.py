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
