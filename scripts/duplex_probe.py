"""PCIe duplex arbitration probe: how the link splits between concurrent H2D
and D2H streams, and whether pacing the H2D stream (chunked copies with spin
gaps on the same stream) buys the D2H stream a larger share. Pinned host
buffers, 1.2 GB copies (one 100M-param subgroup's P/m/v)."""
import json
import sys

import torch

GB = 1e9
SUB = 1_200_000_000
REPS = 8


def run(h2d_pace_gbs=None, chunk=64 << 20, d2h_streams=1, h2d=True, d2h=True):
    dev = torch.device("cuda:0")
    hs = run.hs
    dd = run.dd
    s_in = torch.cuda.Stream()
    s_out = [torch.cuda.Stream() for _ in range(d2h_streams)]
    ev = {}
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    start.record()
    for s in [s_in] + s_out:
        s.wait_event(start)
    cyc_per_ns = run.clock_ghz
    if h2d:
        with torch.cuda.stream(s_in):
            for r in range(REPS):
                src = hs[0]
                if h2d_pace_gbs is None:
                    dd[0].copy_(src, non_blocking=True)
                else:
                    for off in range(0, SUB, chunk):
                        n = min(chunk, SUB - off)
                        dd[0][off:off + n].copy_(src[off:off + n], non_blocking=True)
                        # spin so this chunk's slot in time is n / pace
                        gap_ns = n / h2d_pace_gbs - n / 55.0  # 55 GB/s: the copy itself
                        if gap_ns > 0:
                            torch.cuda._sleep(int(gap_ns * cyc_per_ns))
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            ev["h2d"] = e
    if d2h:
        for i, s in enumerate(s_out):
            with torch.cuda.stream(s):
                part = SUB // d2h_streams
                for r in range(REPS):
                    hs[1][i * part:(i + 1) * part].copy_(dd[1][i * part:(i + 1) * part], non_blocking=True)
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                ev[f"d2h{i}"] = e
    torch.cuda.synchronize()
    out = {}
    for k, e in ev.items():
        ms = start.elapsed_time(e)
        nbytes = REPS * SUB / (d2h_streams if k.startswith("d2h") else 1)
        out[k] = dict(ms=round(ms, 1), gbs=round(nbytes / ms / 1e6, 2))
    return out


def main():
    torch.cuda.init()
    run.hs = [torch.empty(SUB, dtype=torch.uint8).pin_memory() for _ in range(2)]
    run.dd = [torch.empty(SUB, dtype=torch.uint8, device="cuda") for _ in range(2)]
    # spin-kernel calibration: cycles per ns at the clock the copies run at
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        a.record()
        torch.cuda._sleep(20_000_000)
        b.record()
        torch.cuda.synchronize()
    run.clock_ghz = 20_000_000 / (a.elapsed_time(b) * 1e6)
    res = {"clock_ghz": run.clock_ghz}
    run(h2d=True, d2h=True)  # warm
    res["h2d_alone"] = run(d2h=False)
    res["d2h_alone"] = run(h2d=False)
    res["both"] = run()
    res["both_d2h_split2"] = run(d2h_streams=2)
    for pace in (50, 47, 44, 41, 38, 35):
        res[f"both_h2d_paced_{pace}"] = run(h2d_pace_gbs=pace)
    for k, v in res.items():
        print(k, v, flush=True)
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
