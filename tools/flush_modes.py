"""K1 / K2 device time on NYX under three L2 states before each timed launch (GPU):
`write` = 252 MiB zero-fill (the L2 is left full of dirty lines the kernel must write back),
`write+read` = the same then a 252 MiB read of another buffer (L2 cold AND clean), `none`.

    python tools/flush_modes.py
"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2201_13020_b200 as szx  # noqa: E402
from paper_2201_13020_b200 import _abi, _device, synth  # noqa: E402
from paper_2201_13020_b200.pipeline import (_Pools, compress_device, decompress_device,  # noqa: E402
                                            index_buffer)

n = 512 ** 3
L = _abi.lib()
x = synth.field("smooth_ridges", n, seed=1)
e = 1e-3 * float(x.max() - x.min())
pools = _Pools(n, 128)
small = torch.zeros(8, dtype=torch.int64, device="cuda")
sp = _device.stream_ptr()
idx = index_buffer(n, 128)
compress_device(x, n, 128, e, pools, small, sp, idx)
h = small.cpu().numpy()
s = szx.CompressedStream._from_device(128, e, (n,), pools.map, pools.mu[: 4 * (-(-n // 128))].view(torch.float32),
                                      pools.req, pools.codes, pools.mid, int(h[0]), int(h[1]), int(h[2]))
s._index = idx
out = torch.empty(n, dtype=torch.float32, device="cuda")
dsmall = torch.zeros(8, dtype=torch.int64, device="cuda")
dsc = _device.Scratch.get("decompress", L.szx_decompress_scratch_bytes(n, 128))
fw = torch.empty(252 << 18, dtype=torch.float32, device="cuda")
fr = torch.ones(252 << 18, dtype=torch.float32, device="cuda")
acc = torch.zeros(1, dtype=torch.float32, device="cuda")
modes = {"write": lambda: fw.zero_(),
         "write+read": lambda: (fw.zero_(), acc.copy_(fr.sum())),
         "none": lambda: None}
kern = {"K1": lambda: compress_device(x, n, 128, e, pools, small, sp, idx),
        "K2": lambda: decompress_device(s, out, dsmall, dsc, sp)}
for rnd in range(2):
    for mname, flush in modes.items():
        res = {}
        for kname, fn in kern.items():
            ts = []
            for _ in range(20):
                flush()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                ts.append((a, b))
            torch.cuda.synchronize()
            res[kname] = statistics.median(a.elapsed_time(b) * 1e3 for a, b in ts)
        print(f"{mname:11s} K1 {res['K1']:6.1f} us  K2 {res['K2']:6.1f} us", flush=True)
