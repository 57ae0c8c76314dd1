"""HBM ceilings by access mix on this B200 (GPU): read-only (sum), write-only (fill) and
copy (read+write) of 512 MiB with torch kernels, CUDA events, L2 flushed, best of 10.
Context for the kernels' mixes: K1 reads 4N and writes C (~80 % reads on NYX), K2 reads C
and writes 4N (~75 % writes).

    python tools/hbm_modes.py
"""
import json

import torch

n = 128 << 20  # 512 MiB of float32
a = torch.rand(n, device="cuda")
b = torch.empty_like(a)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def best(fn, reps=10):
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


r = best(lambda: a.sum())
w = best(lambda: b.fill_(1.0))
c = best(lambda: b.copy_(a))
nb = 4 * n
print(json.dumps({"read_only_gbs": round(nb / r / 1e6, 1), "write_only_gbs": round(nb / w / 1e6, 1),
                  "copy_gbs_read_plus_write": round(2 * nb / c / 1e6, 1)}))
