"""Pageable vs pinned host->device bandwidth for 1 GiB (torch copies), and
the host's core count: sizing the chunked upload path."""
import os
import time

import numpy as np
import torch

n = 1 << 30
a = np.random.default_rng(0).integers(0, 255, n, dtype=np.uint8)
t = torch.from_numpy(a)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, src in (("pageable", t), ("pinned", t.pin_memory())):
    d.copy_(src)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        d.copy_(src)
    torch.cuda.synchronize()
    print(name, round(3 * n / (time.perf_counter() - t0) / 1e9, 1), "GB/s")
print("cores", os.cpu_count())
