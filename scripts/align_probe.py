"""PCIe copy rate vs the host address offset of a pinned buffer (the engine's
host blocks carry the payload 32 bytes after a 4 KiB boundary, behind the v1
file header): alone and with both directions concurrent."""
import json
import sys

import torch

SUB = 1_200_000_000
REPS = 6


def main(out=None):
    dd = [torch.empty(SUB + 8192, dtype=torch.uint8, device="cuda") for _ in range(2)]
    hb = [torch.empty(SUB + 8192, dtype=torch.uint8).pin_memory() for _ in range(2)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for off in (0, 32, 64, 128, 256, 4096):
        for mode in ("h2d", "d2h", "both"):
            for dev_off in sorted({0, off}):
                torch.cuda.synchronize()
                a = torch.cuda.Event(enable_timing=True)
                a.record()
                for s in (s_in, s_out):
                    s.wait_event(a)
                ends = {}
                if mode in ("h2d", "both"):
                    with torch.cuda.stream(s_in):
                        for _ in range(REPS):
                            dd[0][dev_off:dev_off + SUB].copy_(hb[0][off:off + SUB], non_blocking=True)
                        ends["h2d"] = torch.cuda.Event(enable_timing=True)
                        ends["h2d"].record()
                if mode in ("d2h", "both"):
                    with torch.cuda.stream(s_out):
                        for _ in range(REPS):
                            hb[1][off:off + SUB].copy_(dd[1][dev_off:dev_off + SUB], non_blocking=True)
                        ends["d2h"] = torch.cuda.Event(enable_timing=True)
                        ends["d2h"].record()
                torch.cuda.synchronize()
                r = {k: round(REPS * SUB / a.elapsed_time(e) / 1e6, 2) for k, e in ends.items()}
                res[f"host+{off}_dev+{dev_off}_{mode}"] = r
                print(f"host+{off} dev+{dev_off} {mode}: {r}", flush=True)
    if out:
        open(out, "w").write(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
