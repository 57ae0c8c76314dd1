"""Device times of K1 (compress), K3 (index) and K2 (decode) on a NYX-sized field (GPU).

    python tools/kernel_times.py [n_values] [rel]
"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2201_13020_b200 import _abi, _device, synth  # noqa: E402
from paper_2201_13020_b200.pipeline import _Pools, compress_device, index_buffer  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512 ** 3
rel = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-3
import os  # noqa: E402
if os.environ.get("SZX_LIB"):  # A/B: time another build of the library
    L = ctypes.CDLL(os.environ["SZX_LIB"])
    for name, (res, args) in _abi._SIGS.items():
        if hasattr(L, name):
            getattr(L, name).restype = res
            getattr(L, name).argtypes = args
    _abi._lib = L
L = _abi.lib()
if os.environ.get("SZX_DIRECT_LIMIT"):
    L.szx_set_index_direct_limit(int(os.environ["SZX_DIRECT_LIMIT"]))
P = _device.ptr
x = synth.field("smooth_ridges", n, seed=1)
e = rel * float(x.max() - x.min())
pools = _Pools(n, 128)
small = torch.zeros(8, dtype=torch.int64, device="cuda")
sp = _device.stream_ptr()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")


def timed(fn, reps=10):
    evs = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    return ts[len(ts) // 2]


k1_idx = index_buffer(n, 128)  # K1 also writes the decode index (as in the bench step)
for _ in range(3):
    compress_device(x, n, 128, e, pools, small, sp, k1_idx)
tc = timed(lambda: compress_device(x, n, 128, e, pools, small, sp, k1_idx))
h = small.cpu().numpy()
n_nc, m, mid_len = int(h[0]), int(h[1]), int(h[2])
nb = -(-n // 128)
C = 17 + 24 + -(-nb // 8) + 4 * nb + n_nc + -(-2 * m // 8) + mid_len
idx = torch.empty(L.szx_index_bytes(n, 128) // 8, dtype=torch.int64, device="cuda")
isc = _device.empty_u8(L.szx_index_scratch_bytes(n, 128))
stats = torch.zeros(4, dtype=torch.int64, device="cuda")
out = torch.empty(n, dtype=torch.float32, device="cuda")


def run_index():
    rc = L.szx_index_f32(P(pools.map), P(pools.mu), P(pools.req), P(pools.codes), n, 128, P(idx),
                         P(stats), P(stats) + 16, P(isc), isc.numel(), sp)
    assert rc == 0


def run_decode():
    rc = L.szx_decompress_indexed_f32(P(pools.map), P(pools.mu), P(pools.req), P(pools.codes),
                                      P(pools.mid), mid_len, n, 128, P(idx), P(out),
                                      P(stats) + 24, sp)
    assert rc == 0


run_index()
run_decode()
ti = timed(run_index)
td = timed(run_decode)
err = float((x.double() - out.double()).abs().max())
assert err <= e or "ABL" in os.environ.get("SZX_NVCC_FLAGS", ""), (err, e)  # ablations: wrong output
assert int(stats[1].item()) == mid_len or "ABL" in os.environ.get("SZX_NVCC_FLAGS", "")
peak = 6544.3
for name, t, by in (("compress K1", tc, 4 * n + C), ("index K3", ti, C // 4),
                    ("decode K2", td, 4 * n + C)):
    print(f"{name:12s} {t * 1e3:8.1f} us  {by / t / 1e6:8.1f} GB/s  frac {by / t / 1e6 / peak:.3f}")
print(f"CR {4 * n / C:.3f}  compress input {4 * n / tc / 1e6:.1f} GB/s  "
      f"decompress (K3+K2) output {4 * n / (ti + td) / 1e6:.1f} GB/s")
