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


def test_batched_kernel_mixed_sizes(cuda):
    """One K1 launch over fields of every size class (shorter than a block, than a 32-value
    TMA row, than a tile; exact tiles; partial tiles; a CESM-sized field): each stream equals
    the oracle's, over repeated launches (the per-field look-back segments and tile-0 starts)."""
    from test_gpu_parity import TestWarpPaths

    rng = np.random.default_rng(11)
    sizes = [1, 7, 31, 128, 129, 8191, 8192, 8193, 8192 * 3 + 5, 100_000, 1800 * 3600, 33,
             8192 * 17]
    xs = []
    for i, n in enumerate(sizes):
        if i % 3 == 0:
            xs.append(fields.smooth_ridges(np.random.default_rng(i), n))
        elif i % 3 == 1:
            xs.append(TestWarpPaths._mixed_q_field(rng, -(-n // 128), 1e-3)[:n])
        else:
            xs.append(rng.standard_normal(n).astype(np.float32))
    dims = [(x.size,) for x in xs]
    cfg = szx.CompressorConfig(szx.ErrorBound("rel", 1e-3))
    refs = [oracle.compress(x, d, 128, "rel", 1e-3) if np.ptp(x) > 0 else None
            for x, d in zip(xs, dims)]
    keep = [i for i, r in enumerate(refs) if r is not None]
    fs = szx.datafields([xs[i] for i in keep], [dims[i] for i in keep])
    for _ in range(5):
        batch = szx.compress_batch(fs, cfg)
        for i, s in zip(keep, batch):
            assert szx.serialize(s) == refs[i], (i, sizes[i])
    outs = szx.decompress_batch(batch)
    for i, o in zip(keep, outs):
        assert np.array_equal(o.values.view(np.uint32), oracle.decompress(refs[i]).view(np.uint32))


def test_batch_index_equals_k3(cuda):
    """compress_batch writes every field's decode index from the per-group offsets its K1
    launch records: resolved entry for entry it equals what K3 computes from the field's
    pools (every size class, incl. partial tiles and fields shorter than a group), and
    decompress_batch through it (K2 only) equals the K3 path bit for bit."""
    import torch

    from paper_2201_13020_b200 import _abi, _device
    from test_gpu_parity import TestK1Index, TestWarpPaths

    L = _abi.lib()
    rng = np.random.default_rng(12)
    sizes = [1000, 100, 129, 8191, 8192, 8193, 8192 * 3 + 5, 9216 * 7 + 11, 100_000,
             1800 * 3600, 8192 * 17]
    xs = []
    for i, n in enumerate(sizes):
        x = (fields.smooth_ridges(np.random.default_rng(i), n) if i % 2 == 0
             else TestWarpPaths._mixed_q_field(rng, -(-n // 128), 1e-3)[:n])
        if np.ptp(x) == 0:
            x = x + np.arange(n, dtype=np.float32)
        xs.append(x)
    cfg = szx.CompressorConfig(szx.ErrorBound("rel", 1e-3))
    batch = szx.compress_batch(szx.datafields(xs, [(x.size,) for x in xs]), cfg)
    P = _device.ptr
    for x, s in zip(xs, batch):
        n = s.n_values
        nt = -(-n // 8192)
        p = s.device_pools
        idx3 = torch.empty_like(s._index)
        isc = _device.empty_u8(L.szx_index_scratch_bytes(n, 128))
        st = torch.zeros(4, dtype=torch.int64, device="cuda")
        assert L.szx_index_f32(P(p["constant_map"]), P(p["mu"]), P(s._req), P(s._codes), n, 128,
                               P(idx3), P(st), P(st) + 16, P(isc), isc.numel(),
                               _device.stream_ptr()) == 0
        a = TestK1Index._resolved(s._index.cpu().numpy().view(np.uint64), nt)
        b = TestK1Index._resolved(idx3.cpu().numpy().view(np.uint64), nt)
        for u, v in zip(a, b):
            assert np.array_equal(u, v), n
    fast = szx.decompress_batch(batch)
    for s in batch:
        s._index = None
    slow = szx.decompress_batch(batch)
    for x, s, f, g in zip(xs, batch, fast, slow):
        ref = oracle.decompress(szx.serialize(s))
        assert np.array_equal(f.values.view(np.uint32), ref.view(np.uint32))
        assert np.array_equal(g.values.view(np.uint32), ref.view(np.uint32))
