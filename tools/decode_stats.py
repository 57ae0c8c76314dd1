"""Compute-warp wait / busy cycles of K2 (decode128) on a NYX-sized field (-DSZX_STATS build)."""
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
h = small.cpu().numpy()
mid_len = int(h[2])
idx = torch.empty(L.szx_index_bytes(n, 128) // 8, dtype=torch.int64, device="cuda")
isc = _device.empty_u8(L.szx_index_scratch_bytes(n, 128))
st4 = torch.zeros(4, dtype=torch.int64, device="cuda")
out = torch.empty(n, dtype=torch.float32, device="cuda")
assert L.szx_index_f32(P(pools.map), P(pools.mu), P(pools.req), P(pools.codes), n, 128, P(idx),
                       P(st4), P(st4) + 16, P(isc), isc.numel(), sp) == 0


def run():
    assert L.szx_decompress_indexed_f32(P(pools.map), P(pools.mu), P(pools.req), P(pools.codes),
                                        P(pools.mid), mid_len, n, 128, P(idx), P(out),
                                        P(st4) + 24, sp) == 0


run()
torch.cuda.synchronize()
st = (ctypes.c_uint64 * 8)()
L.szx_debug_stats(st, 4 | 1)
reps = 5
for _ in range(reps):
    run()
torch.cuda.synchronize()
L.szx_debug_stats(st, 4)
tiles = st[1] / reps
print(f"warp-tiles/launch {tiles:.0f}: wait {st[0] / reps / tiles:.0f} busy {st[2] / reps / tiles:.0f} cycles per warp-tile")
