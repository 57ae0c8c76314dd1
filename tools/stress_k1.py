"""Repeated K1 launches on race-prone shapes, bit-exact against the oracle (GPU).

    python tools/stress_k1.py [reps]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle  # noqa: E402
import paper_2201_13020_b200 as szx  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
rng = np.random.default_rng(12)
cases = []
for nb in (64 * 5 + 7, 64 * 148 + 3, 64 * 148 * 6 + 50):
    x = np.cumsum(rng.normal(0, 1, nb * 128 - int(rng.integers(0, 128)))).astype(np.float32)
    cases.append((x, 1e-3))
x = rng.standard_normal(64 * 148 * 8 * 128).astype(np.float32)  # 4-byte tiles: ring full
cases.append((x, 1e-9))
bad = 0
for x, e in cases:
    blob = oracle.compress(x, (x.size,), 128, "abs", e)
    f = szx.DataField(x, (x.size,))
    cfg = szx.CompressorConfig(szx.ErrorBound("abs", e))
    for _ in range(reps):
        bad += szx.serialize(szx.compress(f, cfg)) != blob
print(f"stress_k1: {len(cases)} shapes x {reps} launches, mismatches {bad}")
sys.exit(1 if bad else 0)
