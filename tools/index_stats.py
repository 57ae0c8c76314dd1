"""Per-phase cycle counters of K3 (index128) on a NYX-sized field (GPU, -DSZX_STATS build).

    SZX_NVCC_FLAGS=-DSZX_STATS python -c "from paper_2201_13020_b200 import _build; _build.build(True)"
    python tools/index_stats.py
"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2201_13020_b200 import _abi, _device, synth  # noqa: E402
from paper_2201_13020_b200.pipeline import _Pools, compress_device  # noqa: E402

n = 512 ** 3
L = _abi.lib()
P = _device.ptr
x = synth.field("smooth_ridges", n, seed=1)
e = 1e-3 * float(x.max() - x.min())
pools = _Pools(n, 128)
small = torch.zeros(8, dtype=torch.int64, device="cuda")
sp = _device.stream_ptr()
compress_device(x, n, 128, e, pools, small, sp)
idx = torch.empty(L.szx_index_bytes(n, 128) // 8, dtype=torch.int64, device="cuda")
isc = _device.empty_u8(L.szx_index_scratch_bytes(n, 128))
st4 = torch.zeros(4, dtype=torch.int64, device="cuda")


def run():
    assert L.szx_index_f32(P(pools.map), P(pools.mu), P(pools.req), P(pools.codes), n, 128,
                           P(idx), P(st4), P(st4) + 16, P(isc), isc.numel(), sp) == 0


run()
torch.cuda.synchronize()
st = (ctypes.c_uint64 * 8)()
L.szx_debug_stats(st, 3)
reps = 5
for _ in range(reps):
    run()
torch.cuda.synchronize()
L.szx_debug_stats(st, 2)
ctas = min(1 * torch.cuda.get_device_properties(0).multi_processor_count, -(-(-(-n // 128)) // 64))
names = ["phase 1 (map + look-back)", "rows + counts (per chunk)", "groups + entries (per chunk)",
         "phase 3 (look-back + rebase)", "chunks", "phase-1 look-back", "phase-3 look-back"]
for i, nm in enumerate(names):
    per = st[i] / reps / (ctas if i != 4 else 1)
    print(f"  {nm:32s} {per:12.0f} {'cycles/CTA' if i != 4 else 'chunks/launch'}")
