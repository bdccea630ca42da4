"""Turns the ncu outputs brought back in gpurun_out/ into committed
summaries under profiles/:
  launches.csv (gpu__time_duration per launch) -> profiles/<tag>_launches.md
  prof_adam.ncu-rep (--set full, fused kernel) -> profiles/ncu_adam_fused.json
                                                 + profiles/<tag>_ncu_adam_fused.txt

    python scripts/summarize_ncu.py <tag>
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
PROF.mkdir(exist_ok=True)

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}

launches = OUT / "launches.csv"
if launches.exists():
    rows = list(csv.reader(open(launches)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
    total = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list ({tag}): `ncu --metrics gpu__time_duration.sum --clock-control none "
             f"python bench.py --steps 2 --warmup 1 --skip-e2e --skip-cpu --skip-spill`",
             "", "Cold-cache, serialised per-launch times: compare shares, not absolutes.", "",
             "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{name}` | {c} | {t:.1f} | {t / c:.1f} | {100 * t / total:.2f}% |")
    (PROF / f"{tag}_launches.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))

import re  # noqa: E402


def summarize(rep: Path, label: str, alg_bytes_per_param: int) -> None:
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    get = {h: (vals[i], units[i]) for i, h in enumerate(hdr)}

    def num(key, scale=1.0):
        v, u = get.get(key, ("nan", ""))
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            return None
        x *= {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "usecond": 1e-6, "us": 1e-6, "nsecond": 1e-9, "ns": 1e-9,
              "msecond": 1e-3, "ms": 1e-3}.get(u, 1.0)
        return x * scale

    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
            "launch__func_cache_config", "smsp__inst_executed.sum"]
    text = [f"# ncu --set full, {label} ({tag}); scripts/profile_kernel.py (100M params, f16 grads)"]
    for k in keys:
        if k in get:
            text.append(f"{k} = {get[k][0]} {get[k][1]}")
    text.append("# warp stall reasons, warps stalled per issued instruction")
    stalls = sorted(((h, v) for h, v in get.items() if h.startswith("smsp__average_warps_issue_stalled_")
                     and h.endswith("_per_issue_active.ratio")), key=lambda x: -float(x[1][0] or 0))
    for h, (v, u) in stalls:
        text.append(f"{h} = {v}")
    name = get.get("Kernel Name", ("?", ""))[0]
    dur = num("gpu__time_duration.sum")
    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    n = 100_000_000
    alg = alg_bytes_per_param * n
    summary = {"kernel": name, "params_per_launch": n, "duration_s": dur, "dram_bytes_read": rd,
               "dram_bytes_write": wr, "dram_bytes_per_launch": (rd or 0) + (wr or 0),
               "algorithmic_bytes_per_launch": alg,
               "traffic_over_algorithmic": ((rd or 0) + (wr or 0)) / alg,
               "registers": num("launch__registers_per_thread"),
               "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
               "fp64_pipe_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
               "xu_pipe_pct": num("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
               "dram_throughput_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
               "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
               "tag": tag, "source": f"gpurun_out/{rep.name} (ncu --set full --clock-control none)"}
    stem = "adam_fused" if rep.stem == "prof_adam" else rep.stem.replace("prof_", "adam_")
    (PROF / f"ncu_{stem}.json").write_text(json.dumps(summary, indent=1) + "\n")
    (PROF / f"{tag}_ncu_{stem}.txt").write_text("\n".join(text) + "\n")
    print(json.dumps(summary, indent=1))


for rep in sorted(OUT.glob("prof_*.ncu-rep")):
    m = re.fullmatch(r"prof_multi(\d+)", rep.stem)
    if rep.stem == "prof_adam":
        summarize(rep, "fused Adam kernel", 28)
    elif m:
        k = int(m.group(1))
        summarize(rep, f"fused reduce + update kernel, {k} gradient sources", 26 + 2 * k)
