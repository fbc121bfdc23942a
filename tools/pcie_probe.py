"""PCIe copy bandwidth of the box (pinned host <-> device), one direction and
both at once, for the e2e roofline: python tools/pcie_probe.py [MB]"""
import sys
import time

import torch

mb = int(sys.argv[1]) if len(sys.argv) > 1 else 839
n = mb * 1024 * 1024 // 8
h1 = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(up, down, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        if up:
            with torch.cuda.stream(s1):
                d1.copy_(h1, non_blocking=True)
        if down:
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best


B = n * 8
for name, u, d in (("H2D", 1, 0), ("D2H", 0, 1), ("both", 1, 1)):
    t = run(u, d)
    print(f"{name}: {t * 1e3:.2f} ms  {B * (u + d) / t / 1e9:.1f} GB/s total")

# the same bytes split over k streams per direction (k copy engines)
for k in (2, 4):
    su = [torch.cuda.Stream() for _ in range(k)]
    sd = [torch.cuda.Stream() for _ in range(k)]
    c = n // k

    def runk(up, down, reps=5):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            for i in range(k):
                sl = slice(i * c, (i + 1) * c)
                if up:
                    with torch.cuda.stream(su[i]):
                        d1[sl].copy_(h1[sl], non_blocking=True)
                if down:
                    with torch.cuda.stream(sd[i]):
                        h2[sl].copy_(d2[sl], non_blocking=True)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t)
        return best

    for name, u, d in (("H2D", 1, 0), ("D2H", 0, 1), ("both", 1, 1)):
        t = runk(u, d)
        print(f"{k} streams {name}: {t * 1e3:.2f} ms  {B * (u + d) / t / 1e9:.1f} GB/s total")
