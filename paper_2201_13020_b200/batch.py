"""Batched small-field path (BASELINE.json configs[2]: CESM-ATM-shaped 77 x 1800x3600 fields).

The reference compresses one field per call (``cli.py:113-165`` per file,
``pipeline.compress`` per ``DataField``).  Called in a loop, every field pays the DataField
finite check + range readback (``container.py:84-87``), the bound resolution
(``pipeline.py:34-43``), the pool-size readback after compress and -- on the GPU -- a
persistent-kernel ramp for a field of only a few tiles per SM.  Here the same steps run for
the whole batch:

1. ``datafields``: ONE batched K0 launch (a CTA grid per field, ``range_batch_kernel``),
   ONE readback, then the per-field checks (non-finite -> ValueError, exactly as DataField);
2. ``compress_batch``: bounds resolved on the host from those stats (same float64
   arithmetic as ``resolve_bound``); for block size 128 ONE K1 launch over the tiles of all
   fields (``compress128v3_kernel<true>``: per-field descriptors and TMA tensor maps, the
   decoupled look-back segmented per field) into one pool arena, ONE readback of all pool
   totals; other block sizes one launch per field;
3. ``decompress_batch``: for block size 128 ONE K3 launch indexing every stream (each field
   its own CTA ranges) and ONE K2 launch over the decode tiles of all fields, ONE readback of
   all flags; other block sizes K3/K2 per stream back to back.

Every stream is bit-identical to ``compress(DataField(x, dims), cfg)`` on the same field
(tests/test_gpu_batch.py) -- batching changes when the host waits, not what is computed.
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _abi, _device
from .container import CompressedStream, DataField
from .errors import InconsistentLengthError, PoolUnderrunError
from .pipeline import (
    CompressorConfig,
    _Pools,
    compress_device,
    decompress_device,
    resolve_bound,
)


def datafields(values_list, dims_list) -> list[DataField]:
    """``[DataField(v, d) for v, d in zip(...)]`` with one device synchronisation."""
    torch = _device.torch_cuda()
    L = _abi.lib()
    if len(values_list) != len(dims_list):
        raise ValueError("values and dims lists differ in length")
    devs, hosts = [], []
    for v, dims in zip(values_list, dims_list):
        dims = tuple(int(d) for d in dims)
        if isinstance(v, torch.Tensor):
            dev = v.detach().to(torch.float32).reshape(-1)
            if not dev.is_cuda:
                dev = dev.cuda()
            if not dev.is_contiguous() or dev.data_ptr() % 16:
                dev = dev.clone()
            host = None
        else:
            host = np.ascontiguousarray(v, dtype=np.float32).ravel()
            dev = torch.from_numpy(host).to("cuda", non_blocking=False)
        n = int(dev.numel())
        if n == 0:  # container.py:75-76
            raise ValueError("empty dataset")
        if not dims or any(d <= 0 for d in dims):  # container.py:77-78
            raise ValueError(f"dims must be positive, got {dims}")
        if math.prod(dims) != n:  # container.py:79-83
            raise ValueError(f"product(dims) = {math.prod(dims)} != {n} values")
        devs.append((dev, dims))
        hosts.append(host)
    k = len(devs)
    table = torch.zeros(4 * max(k, 1), dtype=torch.int32, device="cuda")  # [mn, mx] | err
    if k:
        ns = (ctypes.c_uint64 * k)(*[int(d.numel()) for d, _ in devs])
        xs = (ctypes.c_void_p * k)(*[_device.ptr(d) for d, _ in devs])
        scratch = _device.Scratch.get("range_batch", L.szx_range_batch_scratch_bytes(k, ns))
        rc = L.szx_range_batch_f32(k, xs, ns, _device.ptr(table), _device.ptr(table) + 8 * k,
                                   _device.ptr(scratch), scratch.numel(), _device.stream_ptr())
        _device.check(rc, "szx_range_batch_f32")
    t = table.cpu().numpy()
    h = np.zeros((max(k, 1), 4), np.int32)
    h[:k, :2] = t[: 2 * k].reshape(-1, 2)
    h[:k, 2] = t[2 * k: 3 * k]
    out = []
    for i, (dev, dims) in enumerate(devs):
        if h[i, 2] & _abi.FLAG_NONFINITE:  # container.py:84-85
            raise ValueError(f"non-finite value in dataset (field {i})")
        mn, mx = h[i, :2].view(np.float32)
        f = DataField._from_device(dev, dims, float(mn), float(mx))
        f._host = hosts[i]
        out.append(f)
    return out


def _arena(ns, bs):
    """One device allocation for the worst-case pools of every field (include/szx_b200.h
    sizes, 256-byte aligned pieces): offsets of (map, mu, req, codes, mid) per field."""
    L = _abi.lib()
    al = lambda v: -(-v // 256) * 256  # noqa: E731
    offs, off = [], 0
    for n in ns:
        nb = -(-n // bs)
        sizes = (L.szx_map_bytes(n, bs) + 8, 4 * nb + 16, nb + 16,
                 L.szx_codes_capacity(n) + 64, 4 * n + 64)
        o = []
        for sz in sizes:
            o.append((off, sz))
            off += al(sz)
        offs.append(o)
    return _device.empty_u8(off), offs


def compress_batch(fields, cfg: CompressorConfig) -> list[CompressedStream]:
    """``[compress(f, cfg) for f in fields]`` with one device synchronisation (block size
    128: one K1 launch for the whole batch)."""
    torch = _device.torch_cuda()
    L = _abi.lib()
    bs = cfg.block_size
    es = [resolve_bound(cfg.bound, f) for f in fields]  # ZeroRangeError before any launch
    k = len(fields)
    if k == 0:
        return []
    small = torch.zeros(8 * k, dtype=torch.int64, device="cuda")
    sp = _device.stream_ptr()
    if bs == 128:
        ns = [f.n for f in fields]
        arena, offs = _arena(ns, bs)
        P = lambda o: _device.ptr(arena) + o[0]  # noqa: E731
        arr = lambda t, vals: (t * k)(*vals)  # noqa: E731
        vp = ctypes.c_void_p
        n_arr = arr(ctypes.c_uint64, ns)
        totals = torch.zeros(4 * k, dtype=torch.int64, device="cuda")
        scratch = _device.Scratch.get("compress_batch", L.szx_compress_batch_scratch_bytes(k, n_arr))
        # every stream also gets its decode index (what deserialize's K3 would compute), so
        # decompress_batch of these streams runs K2 only
        idxs = [torch.empty(L.szx_index_bytes(n, bs) // 8, dtype=torch.int64, device="cuda")
                for n in ns]
        rc = L.szx_compress_batch_indexed_f32(
            k, arr(vp, [_device.ptr(f.device_values) for f in fields]), n_arr,
            arr(ctypes.c_double, es), arr(vp, [P(o[0]) for o in offs]),
            arr(vp, [P(o[1]) for o in offs]), arr(vp, [P(o[2]) for o in offs]),
            arr(vp, [P(o[3]) for o in offs]), arr(vp, [P(o[4]) for o in offs]),
            arr(vp, [_device.ptr(i) for i in idxs]),
            _device.ptr(totals), _device.ptr(small), _device.ptr(scratch), scratch.numel(), sp)
        _device.check(rc, "szx_compress_batch_indexed_f32")
        h = totals.cpu().numpy().reshape(-1, 4)
        err = int(small[0].item())
        if err & _abi.FLAG_BAD_REQ:  # container.py:206-207
            raise InconsistentLengthError("required bit length outside 1..32")
        out = []
        for f, e, o, t, ix in zip(fields, es, offs, h, idxs):
            nb = -(-f.n // bs)
            sl = lambda oo: arena[oo[0]: oo[0] + oo[1]]  # noqa: E731
            s = CompressedStream._from_device(
                bs, e, f.dims, sl(o[0]), sl(o[1])[: 4 * nb].view(torch.float32), sl(o[2]),
                sl(o[3]), sl(o[4]), int(t[0]), int(t[1]), int(t[2]))
            s._index = ix
            out.append(s)
        return out
    pools = []
    for i, (f, e) in enumerate(zip(fields, es)):
        p = _Pools(f.n, bs)
        compress_device(f.device_values, f.n, bs, e, p, small[8 * i: 8 * i + 8], sp)
        pools.append(p)
    h = small.cpu().numpy().reshape(-1, 8)
    out = []
    for i, (f, e, p) in enumerate(zip(fields, es, pools)):
        n_nc, m, mid_len, err = (int(v) for v in h[i, [0, 1, 2, 4]])
        if err & _abi.FLAG_BAD_REQ:  # container.py:206-207
            raise InconsistentLengthError(f"required bit length outside 1..32 (field {i})")
        nb = -(-f.n // bs)
        out.append(CompressedStream._from_device(bs, e, f.dims, p.map,
                                                 p.mu[: 4 * nb].view(torch.float32), p.req,
                                                 p.codes, p.mid, n_nc, m, mid_len))
    return out


def decompress_batch(streams) -> list[DataField]:
    """``[decompress(s) for s in streams]`` with one device synchronisation (block size 128:
    one K3 launch indexing every stream and one K2 launch decoding all of them)."""
    torch = _device.torch_cuda()
    L = _abi.lib()
    k = len(streams)
    if k == 0:
        return []
    sp = _device.stream_ptr()
    outs = [torch.empty(s.n_values, dtype=torch.float32, device="cuda") for s in streams]
    if all(s.block_size == 128 for s in streams):
        vp = ctypes.c_void_p
        arr = lambda t, vals: (t * k)(*vals)  # noqa: E731
        P = _device.ptr
        ns = arr(ctypes.c_uint64, [s.n_values for s in streams])
        pools = [s.device_pools for s in streams]
        stats = torch.zeros(2 * k, dtype=torch.int64, device="cuda")
        errs = torch.zeros(k, dtype=torch.int32, device="cuda")
        scratch = _device.Scratch.get("decompress_batch",
                                      L.szx_decompress_batch_scratch_bytes(k, ns))
        pool_args = (arr(vp, [P(p["constant_map"]) for p in pools]),
                     arr(vp, [P(p["mu"]) for p in pools]), arr(vp, [P(s._req) for s in streams]),
                     arr(vp, [P(s._codes) for s in streams]),
                     arr(vp, [P(s._mid_buf) for s in streams]),
                     arr(ctypes.c_uint64, [s.mid_len for s in streams]), ns)
        if all(s._index is not None for s in streams):
            # every stream carries its decode index (compress_batch or deserialize's K3)
            rc = L.szx_decompress_batch_indexed_f32(
                k, *pool_args, arr(vp, [P(s._index) for s in streams]),
                arr(vp, [P(o) for o in outs]), P(errs), P(scratch), scratch.numel(), sp)
            _device.check(rc, "szx_decompress_batch_indexed_f32")
        else:
            rc = L.szx_decompress_batch_f32(
                k, *pool_args, arr(vp, [P(o) for o in outs]), P(stats), P(errs), P(scratch),
                scratch.numel(), sp)
            _device.check(rc, "szx_decompress_batch_f32")
        errv = errs.cpu().numpy().astype(np.int64)
    else:
        small = torch.zeros(8 * k, dtype=torch.int64, device="cuda")
        for i, (s, out) in enumerate(zip(streams, outs)):
            scratch = _device.Scratch.get("decompress",
                                          L.szx_decompress_scratch_bytes(s.n_values, s.block_size))
            decompress_device(s, out, small[8 * i: 8 * i + 8], scratch, sp)
        errv = small.cpu().numpy().reshape(-1, 8)[:, 4]
    res = []
    for i, (s, out) in enumerate(zip(streams, outs)):
        err = int(errv[i])
        if err & _abi.FLAG_UNDERRUN:  # blockcodec.py:155-158
            raise PoolUnderrunError(f"mid pool exhausted during decode (field {i})")
        if err & _abi.FLAG_MU_NONFINITE:  # container.py:198-199
            raise InconsistentLengthError(f"non-finite mu (field {i})")
        if err & _abi.FLAG_NONFINITE:  # pipeline.py:224 -> container.py:84-85
            raise ValueError(f"non-finite value in dataset (field {i})")
        res.append(DataField._from_device(out, s.dims))
    return res
