"""Run the bs == 128 compress kernel a few times on a BASELINE-shaped field (for ncu).

    python tools/k1_probe.py [variant] [kind] [n] [rel]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2201_13020_b200 import _abi, _device, synth  # noqa: E402
from paper_2201_13020_b200.pipeline import _Pools, compress_device  # noqa: E402

var = int(sys.argv[1]) if len(sys.argv) > 1 else 2
kind = sys.argv[2] if len(sys.argv) > 2 else "smooth_ridges"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 512 ** 3
rel = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-3
L = _abi.lib()
L.szx_set_compress_variant(var)
x = synth.field(kind, n, seed=1)
e = rel * float(x.max() - x.min())
pools = _Pools(n, 128)
small = torch.zeros(8, dtype=torch.int64, device="cuda")
for _ in range(4):
    compress_device(x, n, 128, e, pools, small, _device.stream_ptr())
torch.cuda.synchronize()
print("ok", small.cpu().tolist()[:3])
