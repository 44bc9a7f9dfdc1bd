"""H2D bandwidth vs host NUMA placement of the pinned buffer: pin the process to
the GPU's local CPUs (sysfs local_cpulist) before allocating, then measure."""
import os, sys, subprocess
import torch

def local_cpus():
    p = torch.cuda.get_device_properties(0)
    bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    path = f"/sys/bus/pci/devices/{bus}/local_cpulist"
    txt = open(path).read().strip() if os.path.exists(path) else ""
    numa = open(f"/sys/bus/pci/devices/{bus}/numa_node").read().strip() if os.path.exists(f"/sys/bus/pci/devices/{bus}/numa_node") else "?"
    cpus = set()
    for part in txt.split(","):
        if "-" in part:
            a, b = part.split("-"); cpus.update(range(int(a), int(b) + 1))
        elif part:
            cpus.add(int(part))
    return bus, numa, txt, cpus

def t(fn, reps=30):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3

torch.cuda.init()
bus, numa, txt, cpus = local_cpus()
print("gpu", bus, "numa", numa, "local cpus", txt, "affinity", sorted(os.sched_getaffinity(0))[:8], "...", len(os.sched_getaffinity(0)))
nb = 13434880
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
for label in ("default", "local"):
    if label == "local" and cpus:
        os.sched_setaffinity(0, cpus & os.sched_getaffinity(0) or cpus)
    h = torch.empty(nb, dtype=torch.uint8).pin_memory()
    h.fill_(1)
    us = t(lambda: d.copy_(h, non_blocking=True))
    h2 = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    h2.fill_(1)
    us2 = t(lambda: d.copy_(h2, non_blocking=True))
    us3 = t(lambda: h2.copy_(d, non_blocking=True))
    print(label, f"H2D {nb/us/1e3:.1f} GB/s (pin_memory()), {nb/us2/1e3:.1f} GB/s (pin_memory=True); D2H {nb/us3/1e3:.1f} GB/s")
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[:1500])
