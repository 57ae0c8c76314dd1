"""Small compress/decompress round trips for compute-sanitizer runs (GPU).

    compute-sanitizer --tool memcheck python tools/sanitize_small.py [decode]

`decode`: only the read side (deserialize -> K3 index + K2 decode of oracle-made streams,
block sizes 128 / 64 / 256), for tools that cannot follow K1's polled tagged words
(racecheck).
"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle  # noqa: E402
import paper_2201_13020_b200 as szx  # noqa: E402

rng = np.random.default_rng(5)
if len(sys.argv) > 1 and sys.argv[1] == "decode":
    for bs in (128, 64, 256):
        for n, e in ((64 * 128 * 40 + 77, 1e-3), (64 * 128 * 3 + 5, 1e-6), (1000, 1e-2)):
            x = np.cumsum(rng.normal(0, 1, n)).astype(np.float32)
            blob = oracle.compress(x, (n,), bs, "abs", e)
            out = szx.decompress(szx.deserialize(blob)).values
            assert np.array_equal(out.view(np.uint32), oracle.decompress(blob).view(np.uint32)), n
    print("sanitize_small decode ok")
    sys.exit(0)
for n, e in ((64 * 128 * 40 + 77, 1e-3), (64 * 128 * 3 + 5, 1e-6), (1000, 1e-2)):
    x = np.cumsum(rng.normal(0, 1, n)).astype(np.float32)
    blob = oracle.compress(x, (n,), 128, "abs", e)
    s = szx.compress(szx.DataField(x, (n,)), szx.CompressorConfig(szx.ErrorBound("abs", e)))
    assert szx.serialize(s) == blob, n
    # device stream: K2 through the index K1 wrote; bytes: K3 then K2
    out = szx.decompress(s).values
    assert np.array_equal(out.view(np.uint32), oracle.decompress(blob).view(np.uint32)), n
    out = szx.decompress(szx.deserialize(blob)).values
    assert np.array_equal(out.view(np.uint32), oracle.decompress(blob).view(np.uint32)), n
print("sanitize_small ok")
