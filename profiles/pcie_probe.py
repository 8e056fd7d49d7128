"""Pinned host <-> device copy bandwidth on this box (the e2e leg's ceiling)."""
import time
import torch

n = 1 << 30  # 1 GiB
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True)
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()


def timed(fn, reps=3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


t = timed(lambda: d.copy_(h, non_blocking=True))
print(f"H2D {n / t / 1e9:.1f} GB/s")
t = timed(lambda: h2.copy_(d2, non_blocking=True))
print(f"D2H {n / t / 1e9:.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


t = timed(both)
print(f"H2D+D2H concurrent {2 * n / t / 1e9:.1f} GB/s total")
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current", "--format=csv"],
                     capture_output=True, text=True).stdout)
