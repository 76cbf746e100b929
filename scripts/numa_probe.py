"""PCIe copy bandwidth vs host CPU affinity (GPU-local NUMA node or not)."""
import os
import sys

import torch

dev = torch.device("cuda", 0)
bdf = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
print("torch props", torch.cuda.get_device_properties(0))
import subprocess
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
print(subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"], capture_output=True, text=True).stdout)
bus = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip().lower()
bus = bus[4:] if bus.startswith("0000") and len(bus) > 12 else bus
for cand in (bus, "0000" + bus[4:] if len(bus) > 12 else bus):
    p = f"/sys/bus/pci/devices/{cand.lower()}/local_cpulist"
    if os.path.exists(p):
        print(p, open(p).read().strip())
        print("numa_node", open(f"/sys/bus/pci/devices/{cand.lower()}/numa_node").read().strip())
print("cpus", os.cpu_count(), "affinity", sorted(os.sched_getaffinity(0))[:8], "...")
print(subprocess.run(["lscpu"], capture_output=True, text=True).stdout[:1500])


def bw():
    src = torch.empty((1700, 2400, 3), dtype=torch.float32, device=dev)
    dst = torch.empty(src.shape, dtype=torch.float32).pin_memory()
    h = torch.empty((3, 1700, 2400), dtype=torch.int16).pin_memory()
    d = torch.empty(h.shape, dtype=torch.int16, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        dst.copy_(src, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    d2h = src.numel() * 4 * 20 / (e0.elapsed_time(e1) / 1e3) / 1e9
    e0.record()
    for _ in range(20):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    h2d = h.numel() * 2 * 20 / (e0.elapsed_time(e1) / 1e3) / 1e9
    return d2h, h2d


print("default affinity: D2H %.1f GB/s, H2D %.1f GB/s" % bw())
