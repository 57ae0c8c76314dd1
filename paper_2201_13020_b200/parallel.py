"""The data-parallel strategy, executed for real (mirrors ``ufzx/parallel.py``).

The reference simulates a GPU design: two-phase compression with prefix-scanned mid-byte
destinations, and decompression with logarithmic index propagation (parallel.py:1-6).
On the B200 that design IS the codec: K1 (compress.cu) classifies, encodes and places mid
bytes through a device-wide decoupled look-back, and K2 (decompress.cu) resolves leading
bytes with a warp-scan form of the same index propagation.  ``parallel_compress`` /
``parallel_decompress`` therefore run the same kernels as ``compress`` / ``decompress``
and are bit-identical to them, as the reference requires (test_parallel.py:146-200).
"""
from __future__ import annotations

from .container import CompressedStream, DataField
from .pipeline import CompressorConfig, compress, decompress

__all__ = ["SCAN_GROUP", "parallel_compress", "parallel_decompress"]

SCAN_GROUP = 32  # warp width of the scans (parallel.py:18)


def parallel_compress(field: DataField, cfg: CompressorConfig) -> CompressedStream:
    """parallel.py:104-140."""
    return compress(field, cfg)


def parallel_decompress(stream: CompressedStream) -> DataField:
    """parallel.py:143-180."""
    return decompress(stream)
