"""PCIe floor of the C2 e2e leg: pinned H2D of the step inputs and D2H of its results, alone."""
import sys, time, numpy as np, torch
dev = torch.device("cuda", 0)
def med(fn, n=300):
    ts = []
    for i in range(n + 20):
        torch.cuda.synchronize()
        t0 = time.perf_counter(); fn(); t1 = time.perf_counter()
        if i >= 20: ts.append(t1 - t0)
    return np.median(ts) * 1e6
for nbytes in (266668, 695587, 4 << 20):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory(); d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    up = med(lambda: (d.copy_(h, non_blocking=True), torch.cuda.synchronize()))
    dn = med(lambda: (h.copy_(d, non_blocking=True), torch.cuda.synchronize()))
    print(f"{nbytes:>8} B: H2D {up:6.1f} us ({nbytes / up / 1e3:5.1f} GB/s)  D2H {dn:6.1f} us ({nbytes / dn / 1e3:5.1f} GB/s)")
print("empty sync", med(lambda: torch.cuda.synchronize()))
