"""Whole-dataset compress / decompress on the B200 (mirrors ``ufzx/pipeline.py``).

``compress`` is one K1 launch per chunk (compress.cu) and ``decompress`` one K2 launch per
chunk (decompress.cu); both execution modes of the reference ("sequential",
"parallel-sim") select the same kernels because the kernels ARE the data-parallel
strategy the reference simulates (parallel.py:1-6) and produce the identical bytes.
"""
from __future__ import annotations

import numpy as np

from . import _abi, _device
from .container import CompressedStream, DataField, ErrorBound
from .errors import InconsistentLengthError, PoolUnderrunError, ZeroRangeError

__all__ = ["CompressorConfig", "ZeroRangeError", "resolve_bound", "block_partition",
           "compress", "compress_with_accounting", "decompress"]

EXECUTION_MODES = ("sequential", "parallel-sim")


class CompressorConfig:
    """pipeline.py:21-31."""

    def __init__(self, bound: ErrorBound, block_size: int = 128, execution: str = "sequential"):
        self.bound = bound
        self.block_size = block_size
        self.execution = execution
        if not 8 <= self.block_size <= 65535:
            raise ValueError(f"block size {self.block_size} outside 8..65535")
        if self.execution not in EXECUTION_MODES:
            raise ValueError(f"unknown execution mode {self.execution!r}")

    def __repr__(self):
        return (f"CompressorConfig(bound={self.bound!r}, block_size={self.block_size}, "
                f"execution={self.execution!r})")


def resolve_bound(bound: ErrorBound, field: DataField) -> float:
    """Absolute bound recorded in the header (pipeline.py:34-43)."""
    if bound.mode == "abs":
        return float(bound.magnitude)
    e = float(bound.magnitude) * field.value_range
    if e == 0:
        raise ZeroRangeError(
            "relative bound on a zero-range dataset resolves to 0; use an absolute bound")
    return e


def block_partition(n: int, block_size: int):
    """pipeline.py:46-51."""
    nb = -(-n // block_size)
    counts = np.full(nb, block_size, dtype=np.int64)
    counts[-1] = n - (nb - 1) * block_size
    return nb, counts


class _Pools:
    """Worst-case device pools for one compress call (include/szx_b200.h sizes)."""

    def __init__(self, n: int, bs: int):
        L = _abi.lib()
        nb = -(-n // bs)
        self.map = _device.empty_u8(L.szx_map_bytes(n, bs) + 8)
        self.mu = _device.empty_u8(4 * nb + 16)
        self.req = _device.empty_u8(nb + 16)
        # the decoder stages whole 32-byte code rows (+16 B alignment slack) per NC block
        self.codes = _device.empty_u8(L.szx_codes_capacity(n) + 64)
        self.mid = _device.empty_u8(4 * n + 64)
        self.scratch = _device.Scratch.get("compress", L.szx_compress_scratch_bytes(n, bs))


def compress_device(x, n: int, bs: int, e: float, pools: _Pools, small, stream_ptr: int,
                    index=None):
    """Launch K1 on device-resident values (stream-ordered, no sync).  With `index` (a
    device buffer of szx_index_bytes, only when szx_compress_emits_index(bs)) K1 also writes
    the decode index the decoder would otherwise compute with K3."""
    L = _abi.lib()
    P = _device.ptr
    if index is not None:
        rc = L.szx_compress_indexed_f32(P(x), n, bs, float(e), P(pools.map), P(pools.mu),
                                        P(pools.req), P(pools.codes), P(pools.mid), P(small),
                                        P(small) + 32, P(pools.scratch), pools.scratch.numel(),
                                        P(index), stream_ptr)
        _device.check(rc, "szx_compress_indexed_f32")
        return
    rc = L.szx_compress_f32(P(x), n, bs, float(e), P(pools.map), P(pools.mu), P(pools.req),
                            P(pools.codes), P(pools.mid), P(small), P(small) + 32,
                            P(pools.scratch), pools.scratch.numel(), stream_ptr)
    _device.check(rc, "szx_compress_f32")


def index_buffer(n: int, bs: int):
    """Device buffer for the decode index K1 emits, or None when it does not (bs != 128 or a
    non-default kernel variant)."""
    L = _abi.lib()
    if not L.szx_compress_emits_index(bs):
        return None
    torch = _device.torch_cuda()
    return torch.empty(L.szx_index_bytes(n, bs) // 8, dtype=torch.int64, device="cuda")


def compress(field: DataField, cfg: CompressorConfig) -> CompressedStream:
    """pipeline.py:177-183 (both execution modes)."""
    torch = _device.torch_cuda()
    e = resolve_bound(cfg.bound, field)
    n, bs = field.n, cfg.block_size
    pools = _Pools(n, bs)
    small = torch.zeros(8, dtype=torch.int64, device="cuda")  # totals[4] | err
    index = index_buffer(n, bs)
    compress_device(field.device_values, n, bs, e, pools, small, _device.stream_ptr(), index)
    h = small.cpu().numpy()
    n_nc, m, mid_len, err = int(h[0]), int(h[1]), int(h[2]), int(h[4])
    if err & _abi.FLAG_BAD_REQ:  # container.py:206-207 at CompressedStream construction
        raise InconsistentLengthError("required bit length outside 1..32")
    nb = -(-n // bs)
    stream = CompressedStream._from_device(bs, e, field.dims, pools.map,
                                           pools.mu[: 4 * nb].view(torch.float32), pools.req,
                                           pools.codes, pools.mid, n_nc, m, mid_len)
    stream._index = index  # decode index from K1 (None: the decoder runs K3)
    return stream


def compress_with_accounting(field: DataField, cfg: CompressorConfig):
    """pipeline.py:186-190: the stream plus its ShiftAccounting.

    K1 produces the stream (bits_shifted_scheme = 8 * mid bytes, pipeline.py:125); the
    unshifted shadow scheme (pipeline.py:119-129) is summed by A1 (``accounting_kernel``,
    csrc/analysis.cu) over the same resident values with the same block classification,
    enqueued behind K1 on the same stream -- one host sync for both.
    """
    from .metrics import ShiftAccounting

    torch = _device.torch_cuda()
    L = _abi.lib()
    e = resolve_bound(cfg.bound, field)
    n, bs = field.n, cfg.block_size
    pools = _Pools(n, bs)
    small = torch.zeros(8, dtype=torch.int64, device="cuda")  # totals[4] | err | bits
    sp = _device.stream_ptr()
    index = index_buffer(n, bs)
    compress_device(field.device_values, n, bs, e, pools, small, sp, index)
    rc = L.szx_accounting_f32(_device.ptr(field.device_values), n, bs, float(e),
                              _device.ptr(small) + 40, sp)
    _device.check(rc, "szx_accounting_f32")
    h = small.cpu().numpy()
    n_nc, m, mid_len, err = int(h[0]), int(h[1]), int(h[2]), int(h[4])
    if err & _abi.FLAG_BAD_REQ:
        raise InconsistentLengthError("required bit length outside 1..32")
    nb = -(-n // bs)
    stream = CompressedStream._from_device(bs, e, field.dims, pools.map,
                                           pools.mu[: 4 * nb].view(torch.float32), pools.req,
                                           pools.codes, pools.mid, n_nc, m, mid_len)
    stream._index = index
    acct = ShiftAccounting(bits_shifted_scheme=8 * mid_len,
                           bits_unshifted_scheme=int(h[5]),
                           compressed_size_bytes=stream.compressed_size_bytes())
    return stream, acct


def decompress_device(stream: CompressedStream, out, small, scratch, stream_ptr: int):
    """Launch K2 into a device float32 buffer (stream-ordered, no sync)."""
    L = _abi.lib()
    P = _device.ptr
    p = stream.device_pools
    if stream._index is not None and stream.block_size in (64, 128, 256, 512):
        # the index exists (K1 emitted it, or deserialize ran K3): decode only
        rc = L.szx_decompress_indexed_f32(
            P(p["constant_map"]), P(p["mu"]), P(stream._req), P(stream._codes),
            P(stream._mid_buf), stream.mid_len, stream.n_values, stream.block_size,
            P(stream._index), P(out), P(small) + 32, stream_ptr)
        _device.check(rc, "szx_decompress_indexed_f32")
        return
    rc = L.szx_decompress_f32(P(p["constant_map"]), P(p["mu"]), P(stream._req),
                              P(stream._codes), P(stream._mid_buf), stream.mid_len,
                              stream.n_values,
                              stream.block_size, P(out), P(small), P(small) + 32, P(scratch),
                              scratch.numel(), stream_ptr)
    _device.check(rc, "szx_decompress_f32")


def decompress(stream: CompressedStream) -> DataField:
    """pipeline.py:227-260 (== parallel.parallel_decompress, parallel.py:143-180)."""
    torch = _device.torch_cuda()
    L = _abi.lib()
    n = stream.n_values
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    scratch = _device.Scratch.get("decompress", L.szx_decompress_scratch_bytes(n, stream.block_size))
    small = torch.zeros(8, dtype=torch.int64, device="cuda")
    decompress_device(stream, out, small, scratch, _device.stream_ptr())
    err = int(small[4].item())
    if err & _abi.FLAG_UNDERRUN:  # blockcodec.py:155-158
        raise PoolUnderrunError("mid pool exhausted during decode")
    if err & _abi.FLAG_MU_NONFINITE:  # container.py:198-199
        raise InconsistentLengthError("non-finite mu")
    if err & _abi.FLAG_NONFINITE:  # pipeline.py:224 -> container.py:84-85
        raise ValueError("non-finite value in dataset")
    return DataField._from_device(out, stream.dims)
