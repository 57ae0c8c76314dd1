"""A/B device timing of the bs == 128 compress kernels (szx_set_compress_variant) on the
BASELINE configs; both variants must produce identical pools (GPU).

    python tools/k1_ab.py [config ...]     configs: nyx1e-3 nyx1e-2 nyx1e-4 hurricane hacc
"""
import json
import statistics
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2201_13020_b200 as szx  # noqa: E402
from paper_2201_13020_b200 import _abi, synth  # noqa: E402
from paper_2201_13020_b200.pipeline import _Pools, compress_device  # noqa: E402

CFG = {"nyx1e-3": ("smooth_ridges", 512 ** 3, 1e-3), "nyx1e-2": ("smooth_ridges", 512 ** 3, 1e-2),
       "nyx1e-4": ("smooth_ridges", 512 ** 3, 1e-4),
       "hurricane": ("smooth_ridges", 100 * 500 * 500, 1e-3),
       "hacc": ("random_walk", 280_953_867, 1e-3),
       "hacc_ridges": ("smooth_ridges", 280_953_867, 1e-3),
       "noise": ("white_noise", 512 ** 3, 1e-3)}
L = _abi.lib()
import os  # noqa: E402
VARIANTS = [int(v) for v in os.environ.get("K1_VARIANTS", "1,2").split(",")]
flush = torch.empty(2 * 126 * 2**20 // 4, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()
sp = int(st.cuda_stream)
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if len(sys.argv) else 6548.5
for name in (sys.argv[1:] or ["nyx1e-3"]):
    kind, n, rel = CFG[name]
    x = synth.field(kind, n, seed=1)
    e = rel * (float(x.max()) - float(x.min()))
    res = {}
    pools = {}
    for var in VARIANTS:
        L.szx_set_compress_variant(var)
        p = _Pools(n, 128)
        small = torch.zeros(8, dtype=torch.int64, device="cuda")
        for _ in range(3):
            compress_device(x, n, 128, e, p, small, sp)
        evs = []
        for _ in range(20):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            compress_device(x, n, 128, e, p, small, sp)
            b.record(st)
            evs.append((a, b))
        torch.cuda.synchronize()
        ms = statistics.median(a.elapsed_time(b) for a, b in evs)
        h = small.cpu().tolist()
        nb = -(-n // 128)
        c = 17 + 8 + -(-nb // 8) + 4 * nb + h[0] + -(-2 * h[1] // 8) + h[2]
        res[var] = {"ms": round(ms, 4), "frac": round((4 * n + c) / ms / 1e6 / peak, 4),
                    "cr": round(4 * n / c, 3)}
        pools[var] = (p, h)
    (p1, h1), (p2, h2) = pools[VARIANTS[0]], pools[VARIANTS[-1]]
    same = h1[:3] == h2[:3]
    if same:
        s1 = szx.CompressedStream._from_device(128, e, (n,), p1.map, p1.mu[: 4 * nb].view(torch.float32),
                                               p1.req, p1.codes, p1.mid, h1[0], h1[1], h1[2])
        s2 = szx.CompressedStream._from_device(128, e, (n,), p2.map, p2.mu[: 4 * nb].view(torch.float32),
                                               p2.req, p2.codes, p2.mid, h2[0], h2[1], h2[2])
        same = s1 == s2
    print(json.dumps({"config": name, **{f"v{v}": res[v] for v in VARIANTS},
                      "identical": bool(same)}), flush=True)
    del pools, x
    torch.cuda.empty_cache()
L.szx_set_compress_variant(1)
