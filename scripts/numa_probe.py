"""Host topology of the box and PCIe copy rates to pinned buffers first-touched
on each NUMA node (cudaHostAlloc touches the pages from the calling thread)."""
import glob
import json
import os
import subprocess
import sys

import torch


def cpus_of(node):
    s = open(f"/sys/devices/system/node/node{node}/cpulist").read().strip()
    out = []
    for part in s.split(","):
        a, _, b = part.partition("-")
        out += list(range(int(a), int(b or a) + 1))
    return out


def main():
    nodes = sorted(int(p.rsplit("node", 1)[1]) for p in glob.glob("/sys/devices/system/node/node[0-9]*"))
    info = {"nodes": {n: cpus_of(n) for n in nodes}, "ncpu": os.cpu_count()}
    try:
        bus = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"],
                             capture_output=True, text=True).stdout.strip().lower()
        bdf = bus[4:] if len(bus) > 12 else bus
        info["gpu_bdf"] = bdf
        info["gpu_numa_node"] = open(f"/sys/bus/pci/devices/{bdf}/numa_node").read().strip()
    except Exception as e:  # noqa: BLE001
        info["gpu_numa_err"] = str(e)
    info["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
    info["meminfo"] = open("/proc/meminfo").read().splitlines()[:3]
    print(json.dumps({k: v for k, v in info.items() if k != "topo"}, indent=1))
    print(info["topo"])
    SUB = 1_200_000_000
    dd = torch.empty(SUB, dtype=torch.uint8, device="cuda")
    res = {}
    for n in nodes:
        os.sched_setaffinity(0, cpus_of(n))
        hb = torch.empty(SUB, dtype=torch.uint8).pin_memory()
        os.sched_setaffinity(0, range(os.cpu_count()))
        for name, fn in (("h2d", lambda: dd.copy_(hb, non_blocking=True)),
                         ("d2h", lambda: hb.copy_(dd, non_blocking=True))):
            fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                fn()
            b.record()
            torch.cuda.synchronize()
            res[f"node{n}_{name}"] = round(5 * SUB / a.elapsed_time(b) / 1e6, 2)
        del hb
    print(res)
    if len(sys.argv) > 1:
        info["rates"] = res
        open(sys.argv[1], "w").write(json.dumps(info, indent=1))




def spread(nbuf=40, sub=1_200_000_000, out=None):
    """D2H/H2D rates cycling over nbuf distinct pinned buffers (the engine's
    ~100 GB of pinned slots and tier blobs) vs one buffer reused, alone and
    with both directions concurrent."""
    dd = [torch.empty(sub, dtype=torch.uint8, device="cuda") for _ in range(2)]
    hb = [torch.empty(sub, dtype=torch.uint8).pin_memory() for _ in range(nbuf)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for label, idx in (("one_buffer", [0] * nbuf), ("spread", list(range(nbuf)))):
        for mode in ("h2d", "d2h", "both"):
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            a.record()
            ends = {}
            for s in (s_in, s_out):
                s.wait_event(a)
            if mode in ("h2d", "both"):
                with torch.cuda.stream(s_in):
                    for i in idx:
                        dd[0].copy_(hb[i], non_blocking=True)
                    ends["h2d"] = torch.cuda.Event(enable_timing=True)
                    ends["h2d"].record()
            if mode in ("d2h", "both"):
                with torch.cuda.stream(s_out):
                    for i in (idx[::-1] if mode == "both" else idx):
                        hb[i].copy_(dd[1], non_blocking=True)
                    ends["d2h"] = torch.cuda.Event(enable_timing=True)
                    ends["d2h"].record()
            torch.cuda.synchronize()
            res[f"{label}_{mode}"] = {k: round(nbuf * sub / a.elapsed_time(e) / 1e6, 2) for k, e in ends.items()}
            print(label, mode, res[f"{label}_{mode}"], flush=True)
    if out:
        open(out, "w").write(json.dumps(res, indent=1))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "spread":
        spread(int(sys.argv[2]) if len(sys.argv) > 2 else 40, out=sys.argv[3] if len(sys.argv) > 3 else None)
    else:
        main()
