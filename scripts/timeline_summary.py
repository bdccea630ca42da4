"""Summarise a phase timeline dumped by bench.py (TFB_TIMELINE / TFB_TIMELINE_C0):
per-stream busy time, idle gaps on the H2D and D2H streams, slow tier transfers."""
import json
import sys


def busy(intervals):
    iv = sorted(i for i in intervals if i[1] > i[0])
    tot, gaps, cur = 0.0, [], None
    for s, e in iv:
        if cur is None:
            cur = [s, e]
        elif s <= cur[1]:
            cur[1] = max(cur[1], e)
        else:
            tot += cur[1] - cur[0]
            gaps.append((cur[1], s))
            cur = [s, e]
    if cur:
        tot += cur[1] - cur[0]
    return tot, gaps


def main(path):
    d = json.load(open(path))
    tl = d["timeline"]
    print(f"{path}: phase {d['ms']:.1f} ms, alloc {d.get('alloc')}")
    h2d = [(e["h2d_start"], e["h2d_end"]) for e in tl]
    d2h = [(e["d2h_start"], e["d2h_end"]) for e in tl if e["d2h_end"] - e["d2h_start"] > 0.5]
    for name, iv in (("h2d", h2d), ("d2h", d2h)):
        rates = [1.2e9 / ((b - a) * 1e6) for a, b in iv if b - a > 5]
        if rates:
            rates.sort()
            print(f"  {name}: per-copy GB/s (1.2 GB copies) min {rates[0]:.1f} median {rates[len(rates)//2]:.1f} "
                  f"max {rates[-1]:.1f}")
    for name, iv in (("h2d", h2d), ("d2h", d2h)):
        t, gaps = busy(iv)
        big = [(round(a, 1), round(b, 1)) for a, b in gaps if b - a > 5]
        print(f"  {name}: {len(iv)} copies, busy {t:.1f} ms; gaps > 5 ms: {big}")
    slow = [e for e in d.get("io", []) if e["read_s"] > 0.01 or e["write_s"] > 0.01]
    for e in slow:
        print(f"  tier io sg {e['id']}: read {e['read_s']*1e3:.0f} ms write {e['write_s']*1e3:.0f} ms")
    last = max(e["d2h_end"] for e in tl)
    print(f"  last d2h end {last:.1f} ms; last retire {max(e['host_retired'] for e in tl):.1f} ms")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
