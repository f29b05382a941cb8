"""PCIe duplex probe: H2D alone, D2H alone, and both at once (two streams), pinned host buffers.
Also prints the host's NUMA layout and the GPU's NUMA node (sysfs)."""
import glob
import os
import time

import torch

GB = 1 << 30
n = int(float(os.environ.get("PROBE_GB", "2")) * GB)
nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
print("numa nodes:", [os.path.basename(p) + ":" + open(p + "/cpulist").read().strip() for p in nodes])
bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
for p in glob.glob("/sys/bus/pci/devices/*"):
    try:
        if open(p + "/vendor").read().strip() == "0x10de" and open(p + "/class").read().startswith("0x0302"):
            print("gpu", os.path.basename(p), "numa_node", open(p + "/numa_node").read().strip())
    except OSError:
        pass
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
hs = torch.empty(n, dtype=torch.uint8, pin_memory=True)
hd = torch.empty(n, dtype=torch.uint8, pin_memory=True)
hs.fill_(1)
hd.fill_(2)
ds = torch.empty(n, dtype=torch.uint8, device="cuda")
dd = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=3):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        t = time.perf_counter()
        if h2d:
            with torch.cuda.stream(s1):
                e[0].record(s1); ds.copy_(hs, non_blocking=True); e[1].record(s1)
        if d2h:
            with torch.cuda.stream(s2):
                e[2].record(s2); hd.copy_(dd, non_blocking=True); e[3].record(s2)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t
        r = (n / GB / (e[0].elapsed_time(e[1]) / 1e3) if h2d else 0.0,
             n / GB / (e[2].elapsed_time(e[3]) / 1e3) if d2h else 0.0, wall)
        best = r if best is None or r[2] < best[2] else best
    return best


for name, a, b in (("h2d alone", 1, 0), ("d2h alone", 0, 1), ("both", 1, 1)):
    h, d, w = run(a, b)
    print(f"{name:10s} H2D {h * GB / 1e9:6.1f} GB/s  D2H {d * GB / 1e9:6.1f} GB/s  wall {w * 1e3:7.1f} ms  "
          f"aggregate {(a + b) * n / w / 1e9:6.1f} GB/s")
