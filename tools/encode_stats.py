"""Per-phase cycle counters of encode128_kernel (K1v2) on a BASELINE-shaped field (GPU,
profiling build: SZX_NVCC_FLAGS=-DSZX_STATS).

    python tools/encode_stats.py [kind] [n_values] [rel]
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
L.szx_set_compress_variant(2)
x = synth.field(kind, n, seed=1)
e = rel * float(x.max() - x.min())
pools = _Pools(n, 128)
small = torch.zeros(8, dtype=torch.int64, device="cuda")
sp = _device.stream_ptr()
for _ in range(3):
    compress_device(x, n, 128, e, pools, small, sp)
torch.cuda.synchronize()
st = (ctypes.c_uint64 * 16)()
L.szx_debug_stats(st, 1 | (3 << 1))
reps = 5
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for _ in range(reps):
    compress_device(x, n, 128, e, pools, small, sp)
ev1.record()
torch.cuda.synchronize()
ms = ev0.elapsed_time(ev1) / reps
L.szx_debug_stats(st, 1 | (3 << 1))
s = [v / reps for v in st]
print(f"{kind} n={n} rel={rel}: compress {ms:.3f} ms ({4 * n / ms / 1e6:.1f} GB/s input)")
ws, ls = max(s[4], 1), max(s[7], 1)
for i, nm in ((0, "compute: input wait"), (1, "compute: encode"), (2, "compute: offsets wait"),
              (3, "compute: write-out")):
    print(f"  {nm:28s} {s[i] / ws:9.0f} cycles/warp-step")
for i, nm in ((5, "look-back warp: counts wait"), (6, "look-back warp: look-back")):
    print(f"  {nm:28s} {s[i] / ls:9.0f} cycles/step")
print(f"  warp steps {s[4]:.0f}, super-tile steps {s[7]:.0f}")
print(f"  look-back: windows/step {s[8] / ls:.2f}, polls/step {s[9] / ls:.2f}, "
      f"waiting polls/step {s[11] / ls:.2f}, mean distance to prefix {s[10] / max(s[8], 1):.1f}")
