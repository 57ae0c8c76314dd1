"""CESM-ATM-shaped batch (BASELINE configs[2]): 77 float32 fields of 1800 x 3600, each with
its own value-range-relative bound (1e-3), compressed + decompressed through the batched API
vs one call per field.  Wall time around the API calls (host syncs included) -- this config
measures the launch / synchronisation overhead path, not kernel bandwidth.

    python tools/bench_batch.py [--fields 77] [--reps 3]
"""
import argparse
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2201_13020_b200 as szx  # noqa: E402
from paper_2201_13020_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--fields", type=int, default=77)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
dims = (1800, 3600)
n = dims[0] * dims[1]
xs = [synth.field("smooth_ridges", n, seed=i) for i in range(args.fields)]
cfg = szx.CompressorConfig(szx.ErrorBound("rel", 1e-3))
torch.cuda.synchronize()


def batched():
    fs = szx.datafields(xs, [dims] * len(xs))
    st = szx.compress_batch(fs, cfg)
    outs = szx.decompress_batch(st)
    torch.cuda.synchronize()
    return st, outs


def looped():
    st = [szx.compress(szx.DataField(x, dims), cfg) for x in xs]
    outs = [szx.decompress(s) for s in st]
    torch.cuda.synchronize()
    return st, outs


res = {}
for name, fn in (("batched", batched), ("per_field", looped)):
    fn()
    ts = []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        st, outs = fn()
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    cbytes = sum(len(szx.serialize(s)) for s in st[:4]) * len(st) / 4
    res[name] = {"seconds": round(t, 5), "gbs_round_trip": round(2 * 4 * n * len(xs) / t / 1e9, 2)}
res["workload"] = f"{args.fields} x {dims} float32 smooth_ridges, rel 1e-3 per field, bs 128"
res["cr"] = round(4 * n * len(xs) / cbytes, 3)
print(json.dumps(res))
