#!/bin/bash
# Inventory of the GPU box: host cores, DRAM, disks, PCIe and the B200 itself.
mkdir -p gpurun_out
{
echo "== nvidia-smi"; nvidia-smi; nvidia-smi -q | grep -iA3 -E "pci|link width|link gen|max clocks" | head -60
echo "== topo"; nvidia-smi topo -m
echo "== cpu"; nproc; lscpu | head -30
echo "== mem"; free -g; cat /proc/meminfo | head -5
echo "== numa"; (numactl --hardware 2>/dev/null || ls /sys/devices/system/node)
echo "== disks"; lsblk -o NAME,SIZE,TYPE,ROTA,MOUNTPOINT,MODEL 2>/dev/null; df -h; mount | grep -E "nvme|/ |tmp|root" | head -20
echo "== repo fs"; df -h "$GRAFT_REPO_ROOT" /tmp /dev/shm
echo "== ulimit"; ulimit -a
echo "== dd /tmp direct"; dd if=/dev/zero of=/tmp/ddprobe bs=16M count=128 oflag=direct 2>&1 | tail -1; dd if=/tmp/ddprobe of=/dev/null bs=16M iflag=direct 2>&1 | tail -1; rm -f /tmp/ddprobe
echo "== dd repo direct"; dd if=/dev/zero of=$GRAFT_REPO_ROOT/ddprobe bs=16M count=128 oflag=direct 2>&1 | tail -1; dd if=$GRAFT_REPO_ROOT/ddprobe of=/dev/null bs=16M iflag=direct 2>&1 | tail -1; rm -f $GRAFT_REPO_ROOT/ddprobe
echo "== dd shm"; dd if=/dev/zero of=/dev/shm/ddprobe bs=16M count=128 2>&1 | tail -1; rm -f /dev/shm/ddprobe
echo "== gds"; ls /usr/local/cuda/gds 2>/dev/null; ls /etc/cufile.json 2>/dev/null
echo "== torch pcie"
python - <<'PY'
import torch, time
print(torch.__version__, torch.cuda.get_device_name(0), torch.cuda.get_device_properties(0))
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): fn()
    e.record(); torch.cuda.synchronize()
    print(name, "GB/s", 5 * n / (s.elapsed_time(e) / 1e3) / 1e9)
# bidirectional
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print("bidir total GB/s", 10 * n / dt / 1e9)
PY
} > gpurun_out/probe_box.txt 2>&1
cat gpurun_out/probe_box.txt | tail -80
