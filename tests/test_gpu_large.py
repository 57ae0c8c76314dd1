"""BASELINE configs at full size that the other suites only sample.

* configs[4]: one 12.5 GB-per-GPU shard of the ~100 GB field -- 24,414,080 blocks x 128 =
  3,125,002,240 values on ONE B200 (the per-rank work of the 8-GPU run; the shards are
  independent streams, sharded.py).  Its pools need 64-bit offsets everywhere: the mid pool
  of the white-noise leg is ~7 GB (offsets past 4 GiB), and the index/look-back payloads
  carry > 2^32 byte counts.  Every byte of every pool and every reconstructed value is
  compared with the oracle window by window (tests/streamcheck.py).
* configs[2]: the whole CESM-shaped batch, 77 fields of 1800x3600 with their own relative
  bounds, through compress_batch / decompress_batch, each stream byte-equal to the oracle's.
"""
import numpy as np
import pytest

from streamcheck import check_stream
import paper_2201_13020_b200 as szx

pytestmark = pytest.mark.gpu

SHARD_VALUES = 24_414_080 * 128  # 3,125,002,240


def _max_err(x, out, chunk=1 << 27):
    """max |x - x'| in float64 without a 25 GB temporary."""
    m = 0.0
    for c0 in range(0, x.numel(), chunk):
        a = x[c0: c0 + chunk].double()
        b = out[c0: c0 + chunk].double()
        m = max(m, float((a - b).abs().max()))
    return m


@pytest.mark.parametrize("kind", ["smooth_ridges", "white_noise"])
def test_configs4_shard_full_stream(cuda, kind):
    torch = cuda
    from paper_2201_13020_b200 import synth

    n = SHARD_VALUES
    x = synth.field(kind, n, seed=5)
    field = szx.DataField(x, (n,))
    s = szx.compress(field, szx.CompressorConfig(szx.ErrorBound("rel", 1e-3)))
    assert s.n_blocks == 24_414_080
    assert s.error_bound == 1e-3 * (float(x.max()) - float(x.min()))
    if kind == "white_noise":
        assert s.mid_len > 1 << 32  # mid-pool offsets beyond 4 GiB are exercised
    out = szx.decompress(s)
    assert _max_err(x, out.device_values) <= s.error_bound
    st = check_stream(s, x, out.device_values, window_blocks=1 << 20)
    assert st["mid_end"] == s.mid_len
    # the serialized length is the container's size formula (container.py:255-266)
    nb = s.n_blocks
    assert s.compressed_size_bytes() == (17 + 8 + -(-nb // 8) + 4 * nb + s.n_nonconstant_blocks
                                         + -(-2 * s.n_nonconstant_elements // 8) + s.mid_len)
    del out, s, field, x
    torch.cuda.empty_cache()


def test_cesm_full_batch(cuda):
    """77 x (1800, 3600) smooth-ridges fields, each with its own relative bound."""
    torch = cuda
    from paper_2201_13020_b200 import synth

    dims = (1800, 3600)
    n = dims[0] * dims[1]
    xs = [synth.field("smooth_ridges", n, seed=i) for i in range(77)]
    cfg = szx.CompressorConfig(szx.ErrorBound("rel", 1e-3))
    fs = szx.datafields(xs, [dims] * 77)
    streams = szx.compress_batch(fs, cfg)
    outs = szx.decompress_batch(streams)
    for i, (x, s, o) in enumerate(zip(xs, streams, outs)):
        assert s.error_bound == 1e-3 * (float(x.max()) - float(x.min())), i
        check_stream(s, x, o.device_values)
    del xs, fs, streams, outs
    torch.cuda.empty_cache()
