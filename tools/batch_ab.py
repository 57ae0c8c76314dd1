"""Batched compress (77 CESM-shaped fields) with and without the decode-index output: device
time per launch pair (GPU).

    python tools/batch_ab.py
"""
import ctypes
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2201_13020_b200 as szx  # noqa: E402
from paper_2201_13020_b200 import _abi, _device, synth  # noqa: E402

nf, dims = 77, (1800, 3600)
n = dims[0] * dims[1]
xs = [synth.field("smooth_ridges", n, seed=1000 + i) for i in range(nf)]
fs = szx.datafields(xs, [dims] * nf)
cfg = szx.CompressorConfig(szx.ErrorBound("rel", 1e-3))
st = szx.compress_batch(fs, cfg)
L = _abi.lib()
P = _device.ptr
vp = ctypes.c_void_p
arr = lambda t, vals: (t * nf)(*vals)  # noqa: E731
ns = arr(ctypes.c_uint64, [n] * nf)
c_args = (nf, arr(vp, [P(f.device_values) for f in fs]), ns,
          arr(ctypes.c_double, [s.error_bound for s in st]),
          arr(vp, [P(s._map) for s in st]), arr(vp, [P(s._mu) for s in st]),
          arr(vp, [P(s._req) for s in st]), arr(vp, [P(s._codes) for s in st]),
          arr(vp, [P(s._mid_buf) for s in st]))
idx = arr(vp, [P(s._index) for s in st])
tot = torch.zeros(4 * nf, dtype=torch.int64, device="cuda")
err = torch.zeros(2, dtype=torch.int64, device="cuda")
sc = _device.empty_u8(L.szx_compress_batch_scratch_bytes(nf, ns))
sp = _device.stream_ptr()
runs = {
    "plain": lambda: L.szx_compress_batch_f32(*c_args, P(tot), P(err), P(sc), sc.numel(), sp),
    "indexed": lambda: L.szx_compress_batch_indexed_f32(*c_args, idx, P(tot), P(err), P(sc),
                                                        sc.numel(), sp),
}
for rnd in range(2):
    for name, fn in runs.items():
        for _ in range(3):
            assert fn() == 0
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        print(f"{name:8s} {statistics.median(ts):8.1f} us  ({4 * n * nf / statistics.median(ts) / 1e3:.0f} GB/s)")
