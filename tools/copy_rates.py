"""Host<->device copy rates on this box: pageable vs pinned (torch), host memcpy."""
import time
import numpy as np
import torch
import os

nb = 218 << 20
x = np.random.default_rng(0).integers(0, 255, nb, dtype=np.uint8)
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
pin = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
pin.numpy()[:] = x


def t(f, reps=3):
    f()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return nb / best / 1e9


print("cpus", os.cpu_count())
print("h2d pageable GB/s", t(lambda: d.copy_(torch.from_numpy(x))))
print("h2d pinned GB/s", t(lambda: d.copy_(pin, non_blocking=True)))
y = np.empty_like(x)
print("d2h pageable GB/s", t(lambda: torch.from_numpy(y).copy_(d)))
print("d2h pinned GB/s", t(lambda: pin.copy_(d, non_blocking=True)))
print("host memcpy 1 thread GB/s", t(lambda: np.copyto(y, x)))
z = np.empty_like(x)
print("host memcpy fresh dest GB/s", nb / (lambda: (lambda t0: (np.copyto(np.empty_like(x), x), time.perf_counter() - t0)[1])(time.perf_counter()))() / 1e9)
