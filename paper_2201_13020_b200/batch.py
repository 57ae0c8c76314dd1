"""Batched small-field path (BASELINE.json configs[2]: CESM-ATM-shaped 77 x 1800x3600 fields).

The reference compresses one field per call (``cli.py:113-165`` per file,
``pipeline.compress`` per ``DataField``).  Called in a loop, every field pays the DataField
finite check + range readback (``container.py:84-87``), the bound resolution
(``pipeline.py:34-43``) and the pool-size readback after compress -- three host round trips
per field.  Here the same steps run for the whole batch with two synchronisations in total:

1. ``datafields``: one K0 launch per field into a shared device table, ONE readback, then
   the per-field checks (non-finite -> ValueError, exactly as DataField);
2. ``compress_batch``: bounds resolved on the host from those stats (same float64
   arithmetic as ``resolve_bound``), one K1 launch per field back to back, ONE readback of
   all pool totals;
3. ``decompress_batch``: K3 + K2 per stream back to back, ONE readback of all flags.

Every stream is bit-identical to ``compress(DataField(x, dims), cfg)`` on the same field
(tests/test_gpu_batch.py) -- batching changes when the host waits, not what is computed.
"""
from __future__ import annotations

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
    table = torch.zeros(4 * max(k, 1), dtype=torch.int32, device="cuda")  # [mn, mx, err, -]
    nmax = max((int(d.numel()) for d, _ in devs), default=1)
    scratch = _device.Scratch.get("range", L.szx_range_scratch_bytes(nmax))
    sp = _device.stream_ptr()
    for i, (dev, _) in enumerate(devs):  # stream-ordered: the scratch is reused in turn
        rc = L.szx_range_f32(_device.ptr(dev), int(dev.numel()), _device.ptr(table) + 16 * i,
                             _device.ptr(table) + 16 * i + 8, _device.ptr(scratch),
                             scratch.numel(), sp)
        _device.check(rc, "szx_range_f32")
    h = table.cpu().numpy().reshape(-1, 4)
    out = []
    for i, (dev, dims) in enumerate(devs):
        if h[i, 2] & _abi.FLAG_NONFINITE:  # container.py:84-85
            raise ValueError(f"non-finite value in dataset (field {i})")
        mn, mx = h[i, :2].view(np.float32)
        f = DataField._from_device(dev, dims, float(mn), float(mx))
        f._host = hosts[i]
        out.append(f)
    return out


def compress_batch(fields, cfg: CompressorConfig) -> list[CompressedStream]:
    """``[compress(f, cfg) for f in fields]`` with one device synchronisation."""
    torch = _device.torch_cuda()
    L = _abi.lib()
    bs = cfg.block_size
    es = [resolve_bound(cfg.bound, f) for f in fields]  # ZeroRangeError before any launch
    small = torch.zeros(8 * max(len(fields), 1), dtype=torch.int64, device="cuda")
    sp = _device.stream_ptr()
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
    """``[decompress(s) for s in streams]`` with one device synchronisation."""
    torch = _device.torch_cuda()
    L = _abi.lib()
    small = torch.zeros(8 * max(len(streams), 1), dtype=torch.int64, device="cuda")
    sp = _device.stream_ptr()
    outs = []
    for i, s in enumerate(streams):
        n = s.n_values
        out = torch.empty(n, dtype=torch.float32, device="cuda")
        scratch = _device.Scratch.get("decompress", L.szx_decompress_scratch_bytes(n, s.block_size))
        decompress_device(s, out, small[8 * i: 8 * i + 8], scratch, sp)
        outs.append(out)
    h = small.cpu().numpy().reshape(-1, 8)
    res = []
    for i, (s, out) in enumerate(zip(streams, outs)):
        err = int(h[i, 4])
        if err & _abi.FLAG_UNDERRUN:  # blockcodec.py:155-158
            raise PoolUnderrunError(f"mid pool exhausted during decode (field {i})")
        if err & _abi.FLAG_MU_NONFINITE:  # container.py:198-199
            raise InconsistentLengthError(f"non-finite mu (field {i})")
        if err & _abi.FLAG_NONFINITE:  # pipeline.py:224 -> container.py:84-85
            raise ValueError(f"non-finite value in dataset (field {i})")
        res.append(DataField._from_device(out, s.dims))
    return res
