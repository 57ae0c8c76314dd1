"""Pinned host<->device copy bandwidth on this box (the e2e ceiling), GPU.

    python tools/pcie_bw.py
"""
import torch

nbytes = 512 << 20
h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def both():
    ev = torch.cuda.current_stream().record_event()
    s1.wait_event(ev)
    s2.wait_event(ev)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


ms = t(lambda: d.copy_(h, non_blocking=True))
print(f"H2D {nbytes / ms / 1e6:.1f} GB/s")
ms = t(lambda: h2.copy_(d2, non_blocking=True))
print(f"D2H {nbytes / ms / 1e6:.1f} GB/s")
ms = t(both)
print(f"H2D+D2H concurrent: {2 * nbytes / ms / 1e6:.1f} GB/s total ({ms:.2f} ms for 2 x 512 MiB)")
