"""GPU NUMA locality and pinned-copy bandwidth with the host buffers first-touched on the GPU's local
node vs elsewhere.  Usage: python tools/numa_probe.py"""
import os

import torch

props = torch.cuda.get_device_properties(0)
bus = f"{props.pci_domain_id:04x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
base = f"/sys/bus/pci/devices/{bus}"
node = open(base + "/numa_node").read().strip() if os.path.exists(base + "/numa_node") else "?"
local = open(base + "/local_cpulist").read().strip() if os.path.exists(base + "/local_cpulist") else "?"
print("gpu", bus, "numa_node", node, "local_cpulist", local, "affinity", len(os.sched_getaffinity(0)), "cpus")
nodes = sorted(d for d in os.listdir("/sys/devices/system/node") if d.startswith("node"))
for nd in nodes:
    print(nd, open(f"/sys/devices/system/node/{nd}/cpulist").read().strip())


def parse(lst):
    out = set()
    for part in lst.split(","):
        if "-" in part:
            a, b = part.split("-")
            out |= set(range(int(a), int(b) + 1))
        elif part:
            out.add(int(part))
    return out


def bw(nbytes=256 << 20):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h.fill_(1)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    res = []
    for direction in ("h2d", "d2h"):
        for _ in range(2):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
        b.record()
        torch.cuda.synchronize()
        res.append(5 * nbytes / a.elapsed_time(b) / 1e6)
    return res


orig = os.sched_getaffinity(0)
print("default affinity: h2d %.1f GB/s d2h %.1f GB/s" % tuple(bw()))
for mb in (4, 8, 16, 33, 64):
    print(f"{mb} MB: h2d %.1f GB/s d2h %.1f GB/s" % tuple(bw(mb << 20)))
for nd in nodes:
    cpus = parse(open(f"/sys/devices/system/node/{nd}/cpulist").read().strip()) & orig
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    print(f"first touch on {nd}: h2d %.1f GB/s d2h %.1f GB/s" % tuple(bw()))
os.sched_setaffinity(0, orig)
