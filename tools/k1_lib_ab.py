"""A/B of the K1 kernel from two builds of the library (GPU): times compress on NYX 1e-3
with the library at the given path (one process per library).

    python tools/k1_lib_ab.py path/to/libszx.so [reps]
"""
import ctypes
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2201_13020_b200 import _abi  # noqa: E402

L = ctypes.CDLL(sys.argv[1])
for name, (res, args) in _abi._SIGS.items():
    if hasattr(L, name):
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
_abi._lib = L
from paper_2201_13020_b200 import synth  # noqa: E402
from paper_2201_13020_b200.pipeline import _Pools, compress_device  # noqa: E402

reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
n = 512 ** 3
x = synth.field("smooth_ridges", n, seed=1)
e = 1e-3 * float(x.max() - x.min())
pools = _Pools(n, 128)
small = torch.zeros(8, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
sp = int(st.cuda_stream)
flush = torch.empty(2 * 126 * 2**20 // 4, dtype=torch.float32, device="cuda")
for _ in range(3):
    compress_device(x, n, 128, e, pools, small, sp)
evs = []
for _ in range(reps):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    compress_device(x, n, 128, e, pools, small, sp)
    b.record(st)
    evs.append((a, b))
torch.cuda.synchronize()
print(sys.argv[1].split("/")[-1], round(statistics.median(a.elapsed_time(b) for a, b in evs) * 1e3, 1), "us")
