"""Host-buffer path (szx_compress_host / szx_decompress_host) on the NYX field from pinned
host memory (GPU): wall time per call for several decompress pipeline part counts, the
CUDA-event timeline of each stage, and the pinned PCIe ceilings beside it.

    python tools/e2e_pipeline.py [parts ...]
"""
import ctypes
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2201_13020_b200 import _abi, synth  # noqa: E402

n = 512 ** 3
dims = (512, 512, 512)
L = _abi.lib()
x = synth.field("smooth_ridges", n, seed=1)
xh = torch.empty(n, dtype=torch.float32, pin_memory=True)
xh.copy_(x)
cap = int(L.szx_compress_bound(n, 3, 128))
blob = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
outh = torch.empty(n, dtype=torch.float32, pin_memory=True)
dims_c = (ctypes.c_uint64 * 3)(*dims)
olen = ctypes.c_uint64()
N4 = 4 * n


def comp():
    assert L.szx_compress_host(xh.data_ptr(), dims_c, 3, 128, 1, 1e-3, blob.data_ptr(), cap,
                               ctypes.byref(olen)) == 0, _abi.last_error()


def decomp():
    assert L.szx_decompress_host(blob.data_ptr(), olen.value, outh.data_ptr(), n) == 0, \
        _abi.last_error()


def wall(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


comp()
decomp()
assert torch.equal(outh[:1000], outh[:1000])  # touch
tc = wall(comp)
print(f"compress host: {1e3 * tc:.3f} ms  ({N4 / tc / 1e9:.2f} GB/s), blob {olen.value} B")
for parts in [int(v) for v in sys.argv[1:]] or [4, 8, 16, 32]:
    L.szx_set_host_pipeline(parts, 0)
    decomp()
    td = wall(decomp)
    print(f"decompress host parts={parts}: {1e3 * td:.3f} ms  ({N4 / td / 1e9:.2f} GB/s); "
          f"round trip {2 * N4 / (tc + td) / 1e9:.2f} GB/s", flush=True)
L.szx_set_host_pipeline(8, 1)
comp()
decomp()
L.szx_set_host_pipeline(8, 0)
