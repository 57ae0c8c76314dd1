"""Per-phase cycle counters of the bs=128 compress kernel on a NYX-sized field (GPU).

    python tools/compress_stats.py [n_values]
"""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2201_13020_b200 import _abi, _device, synth  # noqa: E402
from paper_2201_13020_b200.pipeline import _Pools, compress_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512 ** 3
kind = sys.argv[2] if len(sys.argv) > 2 else "smooth_ridges"
L = _abi.lib()
L.szx_set_compress_variant(1)
x = synth.field(kind, n, seed=1)
e = 1e-3 * float(x.max() - x.min())
pools = _Pools(n, 128)
small = torch.zeros(8, dtype=torch.int64, device="cuda")
sp = _device.stream_ptr()
for _ in range(3):
    compress_device(x, n, 128, e, pools, small, sp)
torch.cuda.synchronize()
st = (ctypes.c_uint64 * 8)()
L.szx_debug_stats(st, 1)
reps = 5
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for _ in range(reps):
    compress_device(x, n, 128, e, pools, small, sp)
ev1.record()
torch.cuda.synchronize()
ms = ev0.elapsed_time(ev1) / reps
L.szx_debug_stats(st, 1)
s = [v / reps for v in st]
tiles = s[3]
names = ["look-back warp: scan", "compute: encode (load..counts)", "compute: wait group counts",
         "tiles", "compute: ring release", "compute: wait input",
         "compute: staging", "write-out warp: write-out"]
print(f"{kind}: compress {ms:.3f} ms  ({4 * n / ms / 1e6:.1f} GB/s input)")
for i, nm in enumerate(names):
    if i == 3:
        continue
    print(f"  {nm:32s} {s[i] / max(tiles, 1):10.0f} cycles/tile")
print(f"  tiles per launch {tiles:.0f}")
