"""Time single compress launches of one bs == 128 variant on NYX 1e-3, synchronizing after
each (GPU; a probe for experimental variants -- stops at the first failing launch).

    python tools/k1_once.py variant [launches] [config]
"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2201_13020_b200 import _abi, synth  # noqa: E402
from paper_2201_13020_b200.pipeline import _Pools, compress_device  # noqa: E402

CFG = {"nyx": ("smooth_ridges", 512 ** 3), "hacc": ("random_walk", 280_953_867),
       "noise": ("white_noise", 512 ** 3)}
var = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
kind, n = CFG[sys.argv[3] if len(sys.argv) > 3 else "nyx"]
L = _abi.lib()
x = synth.field(kind, n, seed=1)
e = 1e-3 * (float(x.max()) - float(x.min()))
L.szx_set_compress_variant(var)
p = _Pools(n, 128)
small = torch.zeros(8, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
sp = int(st.cuda_stream)
ts = []
for i in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    compress_device(x, n, 128, e, p, small, sp)
    b.record(st)
    b.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
    print(f"launch {i}: {ts[-1]:.1f} us", flush=True)
print("median", sorted(ts)[len(ts) // 2], "totals", small.cpu().tolist()[:3])
