"""Per-phase cycle counters of compress128v3_kernel (K1 v3) on a BASELINE-shaped field (GPU,
profiling build: SZX_NVCC_FLAGS=-DSZX_STATS).

    python tools/v3_stats.py [kind] [n_values] [rel]
"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2201_13020_b200 import _abi, _device, synth  # noqa: E402
from paper_2201_13020_b200.pipeline import _Pools, compress_device  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "smooth_ridges"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 512 ** 3
rel = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-3
L = _abi.lib()
L.szx_set_compress_variant(3)
x = synth.field(kind, n, seed=1)
e = rel * float(x.max() - x.min())
pools = _Pools(n, 128)
small = torch.zeros(8, dtype=torch.int64, device="cuda")
sp = _device.stream_ptr()
for _ in range(3):
    compress_device(x, n, 128, e, pools, small, sp)
torch.cuda.synchronize()
st = (ctypes.c_uint64 * 16)()
L.szx_debug_stats(st, 1 | (4 << 1))
reps = 5
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for _ in range(reps):
    compress_device(x, n, 128, e, pools, small, sp)
ev1.record()
torch.cuda.synchronize()
ms = ev0.elapsed_time(ev1) / reps
L.szx_debug_stats(st, 1 | (4 << 1))
s = [v / reps for v in st]
print(f"{kind} n={n} rel={rel}: compress {ms:.3f} ms ({4 * n / ms / 1e6:.1f} GB/s input)")
ws, ls = max(s[6], 1), max(s[12], 1)
for i, nm in ((0, "input wait"), (1, "encode..counts"), (2, "ring-room write-outs"),
              (3, "staging"), (4, "record-forced write-outs"), (5, "opportunistic write-outs")):
    print(f"  compute {nm:26s} {s[i] / ws:9.0f} cycles/warp-tile")
print(f"  write-outs per warp-tile: blocking {s[7] / ws:.3f}, opportunistic {s[8] / ws:.3f}; "
      f"mean pending at write-out {s[9] / max(s[7] + s[8], 1):.2f} tiles")
for i, nm in ((10, "look-back scan"), (11, "counts wait")):
    print(f"  look-back {nm:24s} {s[i] / ls:9.0f} cycles/tile")
print(f"  warp-tiles {s[6]:.0f}, tiles {s[12]:.0f}")
