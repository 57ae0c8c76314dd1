"""K0 (range_kernel: DataField finite check + global min/max) on the NYX-shaped field, for
ncu captures and a device-event timing (GPU).

    python tools/k0_probe.py            # prints the median K0 time and achieved GB/s
"""
import json
import statistics
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2201_13020_b200 import _abi, _device, synth  # noqa: E402

n = 512 ** 3
x = synth.field("smooth_ridges", n, seed=1)
L = _abi.lib()
scratch = _device.empty_u8(L.szx_range_scratch_bytes(n))
small = torch.zeros(16, dtype=torch.int32, device="cuda")
flush = torch.empty(2 * 126 * 2**20 // 4, dtype=torch.float32, device="cuda")
sp = _device.stream_ptr()
st = torch.cuda.current_stream()


def k0():
    rc = L.szx_range_f32(_device.ptr(x), n, _device.ptr(small), _device.ptr(small) + 8,
                         _device.ptr(scratch), scratch.numel(), sp)
    assert rc == 0


for _ in range(3):
    k0()
ts = []
for _ in range(20):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    k0()
    b.record(st)
    ts.append((a, b))
torch.cuda.synchronize()
ms = statistics.median(a.elapsed_time(b) for a, b in ts)
mm = small[:2].view(torch.float32).cpu()
assert float(mm[0]) == float(x.min()) and float(mm[1]) == float(x.max())
print(json.dumps({"kernel": "range_kernel", "n": n, "ms": round(ms, 4),
                  "gbs": round(4 * n / ms / 1e6, 1)}))
