"""Batched small-field path (BASELINE configs[2], CESM-ATM-shaped fields): every batched
stream and reconstruction must equal the one-field-at-a-time API bit for bit, and the
oracle on small fields; errors surface as the reference raises them."""
import numpy as np
import pytest

import fields
import oracle
import paper_2201_13020_b200 as szx

pytestmark = pytest.mark.gpu


def test_batch_equals_single_calls(cuda):
    rng = np.random.default_rng(0)
    xs = [fields.smooth_ridges(np.random.default_rng(i), int(rng.integers(1000, 70_000)))
          for i in range(9)]
    dims = [(x.size,) for x in xs]
    cfg = szx.CompressorConfig(szx.ErrorBound("rel", 1e-3))
    batch = szx.compress_batch(szx.datafields(xs, dims), cfg)
    for x, d, s in zip(xs, dims, batch):
        blob = szx.serialize(s)
        assert blob == szx.serialize(szx.compress(szx.DataField(x, d), cfg))
        assert blob == oracle.compress(x, d, 128, "rel", 1e-3)
    outs = szx.decompress_batch(batch)
    for x, s, o in zip(xs, batch, outs):
        ref = oracle.decompress(szx.serialize(s))
        assert np.array_equal(o.values.view(np.uint32), ref.view(np.uint32))


def test_cesm_shaped_batch(cuda):
    """A few 1800x3600 fields with their own relative bounds (device-generated)."""
    from paper_2201_13020_b200 import synth

    n = 1800 * 3600
    xs = [synth.field("smooth_ridges", n, seed=i) for i in range(4)]
    cfg = szx.CompressorConfig(szx.ErrorBound("rel", 1e-3))
    fs = szx.datafields(xs, [(1800, 3600)] * 4)
    batch = szx.compress_batch(fs, cfg)
    outs = szx.decompress_batch(batch)
    for x, f, s, o in zip(xs, fs, batch, outs):
        assert s.error_bound == 1e-3 * (f.global_max - f.global_min)
        assert s == szx.compress(szx.DataField(x, (1800, 3600)), cfg)
        assert float((x.double() - o.device_values.double()).abs().max()) <= s.error_bound


def test_batch_errors(cuda):
    good = np.linspace(0, 1, 4096, dtype=np.float32)
    bad = good.copy()
    bad[7] = np.nan
    with pytest.raises(ValueError):
        szx.datafields([good, bad], [(4096,), (4096,)])
    with pytest.raises(ValueError):
        szx.datafields([good], [(4095,)])
    flat = np.full(4096, 2.5, np.float32)
    fs = szx.datafields([good, flat], [(4096,), (4096,)])
    with pytest.raises(szx.ZeroRangeError):
        szx.compress_batch(fs, szx.CompressorConfig(szx.ErrorBound("rel", 1e-3)))
    s = szx.compress_batch(fs, szx.CompressorConfig(szx.ErrorBound("abs", 1e-3)))
    assert len(s) == 2 and s[1].n_values == 4096
