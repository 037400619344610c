"""Host<->device copy bandwidth with pinned 2 GB buffers: H2D, D2H, and both at once on two
streams (the e2e leg's bound). Dev probe."""
import os
import time

import torch

nb = 2 * 10**9 // 8
h_in = torch.empty(nb, dtype=torch.float64).pin_memory()
h_out = torch.empty(nb, dtype=torch.float64).pin_memory()
d_a = torch.empty(nb, dtype=torch.float64, device="cuda")
d_b = torch.empty(nb, dtype=torch.float64, device="cuda")
h_in.fill_(1.0)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


GB = nb * 8 / 1e9
a, b, c = t(h2d), t(d2h), t(both)
print(f"H2D {GB / a:.1f} GB/s  D2H {GB / b:.1f} GB/s  both {2 * GB / c:.1f} GB/s aggregate ({c * 1e3:.1f} ms per 2+2 GB)")
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    bus = pynvml.nvmlDeviceGetPciInfo(h).busId
    bus = bus.decode() if isinstance(bus, bytes) else bus
    path = f"/sys/bus/pci/devices/{bus.lower()[-12:]}"
    for f in ("numa_node", "local_cpulist", "current_link_speed", "current_link_width"):
        try:
            print(f, open(os.path.join(path, f)).read().strip())
        except Exception as e:
            print(f, "?", e)
    print("affinity", len(os.sched_getaffinity(0)), "cpus; nodes", os.listdir("/sys/devices/system/node")
          if os.path.exists("/sys/devices/system/node") else "?")
except Exception as e:
    print("nvml", e)
