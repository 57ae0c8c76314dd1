"""Device times of the generic block-size kernels (bs != 128) on the NYX field (GPU):
compress_generic_kernel and decompress_generic_kernel, vs the bs == 128 path.

    python tools/generic_times.py [bs ...]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2201_13020_b200 import _abi, _device, synth  # noqa: E402
from paper_2201_13020_b200.pipeline import _Pools, compress_device, index_buffer  # noqa: E402

n = 512 ** 3
L = _abi.lib()
P = _device.ptr
x = synth.field("smooth_ridges", n, seed=1)
e = 1e-3 * float(x.max() - x.min())
sp = _device.stream_ptr()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
peak = 6547.5


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


for bs in [int(v) for v in sys.argv[1:]] or [64, 128, 256]:
    pools = _Pools(n, bs)
    small = torch.zeros(8, dtype=torch.int64, device="cuda")
    compress_device(x, n, bs, e, pools, small, sp)
    tc = timed(lambda: compress_device(x, n, bs, e, pools, small, sp))
    h = small.cpu().numpy()
    n_nc, m, mid_len = int(h[0]), int(h[1]), int(h[2])
    nb = -(-n // bs)
    C = 17 + 24 + -(-nb // 8) + 4 * nb + n_nc + -(-2 * m // 8) + mid_len
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    dsc = _device.empty_u8(L.szx_decompress_scratch_bytes(n, bs))
    st = torch.zeros(8, dtype=torch.int64, device="cuda")

    def dec():
        assert L.szx_decompress_f32(P(pools.map), P(pools.mu), P(pools.req), P(pools.codes),
                                    P(pools.mid), mid_len, n, bs, P(out), P(st), P(st) + 32,
                                    P(dsc), dsc.numel(), sp) == 0

    dec()
    td = timed(dec)
    err = float((x.double() - out.double()).abs().max())
    assert err <= e
    # the device round trip: K1 writes the decode index, K2 decodes through it
    idx = index_buffer(n, bs)
    tdi = None
    if idx is not None:
        compress_device(x, n, bs, e, pools, small, sp, idx)

        def deci():
            assert L.szx_decompress_indexed_f32(P(pools.map), P(pools.mu), P(pools.req),
                                                P(pools.codes), P(pools.mid), mid_len, n, bs,
                                                P(idx), P(out), P(st) + 32, sp) == 0
        out.zero_()
        deci()
        tdi = timed(deci)
        assert float((x.double() - out.double()).abs().max()) <= e
    print(json.dumps({"bs": bs, "cr": round(4 * n / C, 3), "compress_us": round(tc * 1e3, 1),
                      "compress_frac": round((4 * n + C) / tc / 1e6 / peak, 3),
                      "decompress_us": round(td * 1e3, 1),
                      "decompress_frac": round((4 * n + C) / td / 1e6 / peak, 3),
                      "indexed_decode_us": None if tdi is None else round(tdi * 1e3, 1),
                      "indexed_decode_frac": None if tdi is None else
                      round((4 * n + C) / tdi / 1e6 / peak, 3)}))
    del pools
