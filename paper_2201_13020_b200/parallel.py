"""The data-parallel strategy, executed for real (mirrors ``ufzx/parallel.py``).

The reference simulates a GPU design: two-phase compression with prefix-scanned mid-byte
destinations, and decompression with logarithmic index propagation (parallel.py:1-6).
On the B200 that design IS the codec: K1 (compress.cu) classifies, encodes and places mid
bytes through a device-wide decoupled look-back, and K2 (decompress.cu) resolves leading
bytes with a warp-scan form of the same index propagation.  ``parallel_compress`` /
``parallel_decompress`` therefore run the same kernels as ``compress`` / ``decompress``
and are bit-identical to them, as the reference requires (test_parallel.py:146-200).

The simulation's building blocks are exported as device passes too (csrc/analysis.cu):
``prefix_scan`` (A4, exclusive int64 scan) and ``propagate_round`` / ``propagate_indices``
(A5, the per-column running maximum the stride-doubling rounds converge to), so code
written against the reference's parallel module runs unchanged.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _abi, _device
from .container import CompressedStream, DataField
from .pipeline import CompressorConfig, compress, decompress

__all__ = ["SCAN_GROUP", "prefix_scan", "BlockByteLayout", "ReadPosition", "propagate_round",
           "propagate_indices", "parallel_compress", "parallel_decompress"]

SCAN_GROUP = 32  # warp width of the scans (parallel.py:18)


def _to_device_i64(a):
    torch = _device.torch_cuda()
    if isinstance(a, torch.Tensor):
        t = a.detach().reshape(-1).to(torch.int64)
        return (t if t.is_cuda else t.cuda()).contiguous(), True
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.int64).ravel())
    return torch.from_numpy(arr).cuda(), False


def prefix_scan(lengths):
    """Exclusive prefix scan, int64 (parallel.py:21-44); equals the naive running sum.

    NumPy / array-like in -> NumPy int64 out (as the reference); a torch tensor in -> a CUDA
    int64 tensor out."""
    torch = _device.torch_cuda()
    L = _abi.lib()
    d_in, is_torch = _to_device_i64(lengths)
    n = int(d_in.numel())
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    if n:
        scratch = _device.Scratch.get("scan", L.szx_prefix_scan_scratch_bytes(n))
        rc = L.szx_prefix_scan_i64(_device.ptr(d_in), n, _device.ptr(out), _device.ptr(scratch),
                                   scratch.numel(), _device.stream_ptr())
        _device.check(rc, "szx_prefix_scan_i64")
    return out if is_torch else out.cpu().numpy()


@dataclass
class BlockByteLayout:
    """Byte-kind layout of one non-constant block: element i has min(code, q) leading bytes
    followed by q - min(code, q) mid bytes (parallel.py:47-67)."""

    leading_codes: np.ndarray  # uint8 per element
    required_byte_count: int
    count: int

    def __post_init__(self):
        self.leading_codes = np.ascontiguousarray(self.leading_codes, dtype=np.uint8)
        if len(self.leading_codes) != self.count:
            raise ValueError("one code per element required")
        if not 1 <= self.required_byte_count <= 4:
            raise ValueError(f"bad byte count {self.required_byte_count}")

    def is_mid(self) -> np.ndarray:
        """(count, q) bool matrix: True where the byte is a mid byte."""
        q = self.required_byte_count
        cols = np.arange(q, dtype=np.uint8)
        clamped = np.minimum(self.leading_codes, q)
        return cols[None, :] >= clamped[:, None]


@dataclass
class ReadPosition:
    """Resolved read positions per byte: 1-based source element index, 0 = zero word
    (parallel.py:70-74)."""

    positions: np.ndarray  # (count, q) int64
    rounds: int


def propagate_round(positions: np.ndarray, stride: int) -> np.ndarray:
    """One interleaved-addressing round (parallel.py:74-80): a row adopts the row `stride`
    back when that one is greater; positions never decrease."""
    torch = _device.torch_cuda()
    L = _abi.lib()
    if int(stride) < 1:  # the reference's slices positions[:-0] fail to broadcast
        raise ValueError(f"stride must be positive, got {stride}")
    p = np.ascontiguousarray(np.asarray(positions, dtype=np.int64))
    shape = p.shape
    rows = shape[0] if p.ndim else 1
    cols = int(np.prod(shape[1:])) if p.ndim > 1 else 1
    if p.size == 0:
        return p.copy()
    d_in = torch.from_numpy(p.reshape(-1)).cuda()
    d_out = torch.empty_like(d_in)
    rc = L.szx_propagate_round(_device.ptr(d_in), rows, cols, int(stride),
                               _device.ptr(d_out), _device.stream_ptr())
    _device.check(rc, "szx_propagate_round")
    return d_out.cpu().numpy().reshape(shape)


def propagate_indices(layout: BlockByteLayout) -> ReadPosition:
    """Assign every byte the element index of the mid byte it reads from (parallel.py:83-101):
    mid bytes start at their own 1-based index, leading bytes at the zero word (0), and
    ceil(log2 n) stride-doubling rounds make each position the running maximum -- which A5
    computes directly as a per-column max-scan on the device."""
    torch = _device.torch_cuda()
    L = _abi.lib()
    n, q = layout.count, layout.required_byte_count
    rounds = max(0, math.ceil(math.log2(n))) if n > 1 else 0
    if n == 0:
        return ReadPosition(np.zeros((0, q), np.int64), rounds)
    codes = torch.from_numpy(layout.leading_codes).cuda()
    pos = torch.empty(n * q, dtype=torch.int64, device="cuda")
    rc = L.szx_propagate_indices(_device.ptr(codes), n, q, _device.ptr(pos),
                                 _device.stream_ptr())
    _device.check(rc, "szx_propagate_indices")
    return ReadPosition(pos.cpu().numpy().reshape(n, q), rounds)


def parallel_compress(field: DataField, cfg: CompressorConfig) -> CompressedStream:
    """parallel.py:104-140."""
    return compress(field, cfg)


def parallel_decompress(stream: CompressedStream) -> DataField:
    """parallel.py:143-180."""
    return decompress(stream)
