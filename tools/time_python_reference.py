"""Time the reference AS SHIPPED (the pure-Python/NumPy ufzx package) on a sample of the
NYX workload, in the build container (the GPU box has no /root/reference).  Records
MB/s of field data for compress (-> serialize) and deserialize -> decompress, single
process, next to this repo's C restatement of the same algorithm on the same sample.

    python tools/time_python_reference.py [n_values] > profiles/r02_python_reference.json
"""
import json
import os
import platform
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import ufzx  # noqa: E402

import fields  # noqa: E402
import oracle  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 21
x = fields.smooth_ridges(np.random.default_rng(1), n)
rel = 1e-3
field = ufzx.DataField(x, (n,))
cfg = ufzx.CompressorConfig(ufzx.ErrorBound("rel", rel))
t0 = time.perf_counter()
s = ufzx.compress(field, cfg)
blob = ufzx.serialize(s)
t1 = time.perf_counter()
y = ufzx.decompress(ufzx.deserialize(blob)).values
t2 = time.perf_counter()
ref_blob = oracle.compress(x, (n,), 128, "rel", rel)
t3 = time.perf_counter()
for _ in range(3):
    oracle.compress(x, (n,), 128, "rel", rel)
t4 = time.perf_counter()
for _ in range(3):
    oracle.decompress(ref_blob)
t5 = time.perf_counter()
assert blob == ref_blob, "oracle disagrees with the shipped reference"
assert np.array_equal(np.asarray(y, np.float32).view(np.uint32), oracle.decompress(ref_blob).view(np.uint32))
mb = 4 * n / 1e6
print(json.dumps({
    "what": "reference as shipped (ufzx, pure Python/NumPy), single process, build container",
    "host": platform.processor() or platform.machine(), "sample_values": n,
    "workload": "NYX-shaped smooth_ridges (tests/fields.py == ufzx/synth.py), rel 1e-3, bs 128",
    "python_compress_MBps": round(mb / (t1 - t0), 2),
    "python_decompress_MBps": round(mb / (t2 - t1), 2),
    "oracle_c_1thread_compress_MBps": round(mb / ((t4 - t3) / 3), 1),
    "oracle_c_1thread_decompress_MBps": round(mb / ((t5 - t4) / 3), 1),
    "streams_identical": True,
}))
