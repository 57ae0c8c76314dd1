"""Per-tile pipeline timeline of the K1 v1 compress kernel (GPU, profiling build
SZX_NVCC_FLAGS=-DSZX_TRACE): median / p90 latencies between a tile's events.

    python tools/k1_trace.py [kind] [n_values] [rel]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2201_13020_b200 import _abi, _device, synth  # noqa: E402
from paper_2201_13020_b200.pipeline import _Pools, compress_device  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "smooth_ridges"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 512 ** 3
rel = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-3
L = _abi.lib()
L.szx_set_compress_variant(1)
x = synth.field(kind, n, seed=1)
e = rel * float(x.max() - x.min())
pools = _Pools(n, 128)
small = torch.zeros(8, dtype=torch.int64, device="cuda")
sp = _device.stream_ptr()
ntiles = -(-n // 8192)
buf = torch.zeros(8 * ntiles, dtype=torch.int64, device="cuda")
for _ in range(3):
    compress_device(x, n, 128, e, pools, small, sp)
L.szx_debug_trace(ctypes_ptr := buf.data_ptr())
compress_device(x, n, 128, e, pools, small, sp)
torch.cuda.synchronize()
L.szx_debug_trace(None)
raw = buf.view(ntiles, 8).cpu().numpy()
import os
os.makedirs("gpurun_out", exist_ok=True)
np.save(f"gpurun_out/k1_trace_{kind}.npy", raw)
t = raw.astype(np.float64)
t0 = t[t > 0].min()
t = (t - t0) / 1e3  # us from the first event
names = ["claim", "tma", "seen", "agg", "lbscan", "incl", "wo_start", "wo_end"]
print(f"{kind} n={n} rel={rel}: {ntiles} tiles, span {t.max():.1f} us")
pairs = [(0, 1), (1, 2), (2, 3), (0, 3), (0, 4), (3, 5), (4, 5), (5, 6), (6, 7), (3, 7), (0, 7)]
for a, b in pairs:
    d = t[:, b] - t[:, a]
    print(f"  {names[a]:>8s} -> {names[b]:<8s} median {np.median(d):7.2f} us  p10 {np.percentile(d, 10):7.2f}"
          f"  p90 {np.percentile(d, 90):7.2f}")
# look-back diagnosis: when was the window (the G tiles below t) fully aggregated, and when
# did this CTA's previous tile get its inclusive prefix (the look-back warp is serial)?
G = 148
agg = t[:, 3]
from numpy.lib.stride_tricks import sliding_window_view
win = np.full(ntiles, np.nan)
w = sliding_window_view(agg, G - 1)  # w[i] = agg[i : i + G - 1]
win[G:] = w[1: ntiles - G + 1].max(axis=1)  # tiles t-G+1 .. t-1
d1 = t[G:, 4] - win[G:]
prev_incl = np.full(ntiles, np.nan)
prev_incl[G:] = t[:-G, 5]
d2 = t[G:, 4] - prev_incl[G:]
for nm, d in (("lbscan - window aggregated", d1), ("scan duration (static)", t[G:, 4] - t[G:, 0]),
              ("scan start - own prev incl", t[G:, 0] - prev_incl[G:]), ("lbscan - own prev incl", d2),
              ("window aggregated - own agg", win[G:] - agg[G:])):
    print(f"  {nm:30s} median {np.nanmedian(d):7.2f}  p10 {np.nanpercentile(d, 10):7.2f}  p90 {np.nanpercentile(d, 90):7.2f}")
# steady-state rate: tiles claimed per us in the middle half
mid = np.sort(t[:, 0])[ntiles // 4: 3 * ntiles // 4]
print(f"  claim rate (middle half) {len(mid) / (mid[-1] - mid[0]):.1f} tiles/us")
