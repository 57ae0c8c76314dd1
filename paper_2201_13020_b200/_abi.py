"""ctypes binding of libszx_b200.so (the C ABI declared in include/szx_b200.h).

There is no CPU implementation behind this module: if the shared library is missing or no
CUDA device is visible, every codec call raises.  Device buffers are torch CUDA tensors
(plumbing only); pointers and the current torch stream are passed as plain integers.
"""
from __future__ import annotations

import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libszx_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "szx_b200.h")

# status codes (include/szx_b200.h)
OK = 0
ERR_INVALID_ARG = 1
ERR_CUDA = 2
ERR_ALIGN = 3
ERR_NONFINITE = 4
ERR_ZERO_RANGE = 5
ERR_BAD_REQ = 6
ERR_UNDERRUN = 7
ERR_TRUNCATED = 8
ERR_MAGIC = 9
ERR_VERSION = 10
ERR_DTYPE = 11
ERR_INCONSISTENT = 12
ERR_CAPACITY = 13
ERR_NO_DEVICE = 14

FLAG_BAD_REQ = 1
FLAG_NONFINITE = 2
FLAG_UNDERRUN = 4
FLAG_MU_NONFINITE = 8
FLAG_CODE_PADDING = 16

_lib = None


class NativeLibraryError(RuntimeError):
    """libszx_b200.so is missing or unusable; there is no fallback path."""


class Totals(ctypes.Structure):
    _fields_ = [("n_nc", ctypes.c_uint64), ("m", ctypes.c_uint64),
                ("mid_len", ctypes.c_uint64), ("pad", ctypes.c_uint64)]


_SIGS = {
    "szx_version": (ctypes.c_char_p, []),
    "szx_last_error": (ctypes.c_char_p, []),
    "szx_bound_exponent": (ctypes.c_int32, [ctypes.c_double]),
    "szx_set_max_chunk_blocks": (ctypes.c_uint64, [ctypes.c_uint64]),
    "szx_set_index_direct_limit": (ctypes.c_uint64, [ctypes.c_uint64]),
    "szx_set_compress_variant": (ctypes.c_int, [ctypes.c_int]),
    "szx_debug_stats": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "szx_debug_trace": (ctypes.c_int, [ctypes.c_void_p]),
    "szx_set_index_kernel": (ctypes.c_int, [ctypes.c_int]),
    "szx_set_host_pipeline": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "szx_range_scratch_bytes": (ctypes.c_size_t, [ctypes.c_uint64]),
    "szx_range_f32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                     ctypes.c_void_p]),
    "szx_num_blocks": (ctypes.c_uint64, [ctypes.c_uint64, ctypes.c_uint32]),
    "szx_map_bytes": (ctypes.c_uint64, [ctypes.c_uint64, ctypes.c_uint32]),
    "szx_codes_capacity": (ctypes.c_uint64, [ctypes.c_uint64]),
    "szx_compress_scratch_bytes": (ctypes.c_size_t, [ctypes.c_uint64, ctypes.c_uint32]),
    "szx_compress_emits_index": (ctypes.c_int, [ctypes.c_uint32]),
    "szx_compress_indexed_f32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32,
                                                ctypes.c_double] + [ctypes.c_void_p] * 8
                                 + [ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p]),
    "szx_compress_f32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32,
                                        ctypes.c_double] + [ctypes.c_void_p] * 7
                         + [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "szx_validate_f32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                        ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64,
                                        ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p]),
    "szx_index_bytes": (ctypes.c_uint64, [ctypes.c_uint64, ctypes.c_uint32]),
    "szx_index_scratch_bytes": (ctypes.c_size_t, [ctypes.c_uint64, ctypes.c_uint32]),
    "szx_index_f32": (ctypes.c_int, [ctypes.c_void_p] * 4 + [
        ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
        ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "szx_decompress_indexed_f32": (ctypes.c_int, [ctypes.c_void_p] * 5 + [
        ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
        ctypes.c_void_p, ctypes.c_void_p]),
    "szx_decompress_scratch_bytes": (ctypes.c_size_t, [ctypes.c_uint64, ctypes.c_uint32]),
    "szx_decompress_f32": (ctypes.c_int, [ctypes.c_void_p] * 5 + [
        ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "szx_accounting_f32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32,
                                          ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p]),
    "szx_quality_scratch_bytes": (ctypes.c_size_t, [ctypes.c_uint64]),
    "szx_quality_f32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                       ctypes.c_void_p]),
    "szx_block_range_counts_f32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64,
                                                  ctypes.c_uint32, ctypes.c_double,
                                                  ctypes.c_void_p, ctypes.c_uint32,
                                                  ctypes.c_void_p, ctypes.c_void_p]),
    "szx_prefix_scan_scratch_bytes": (ctypes.c_size_t, [ctypes.c_uint64]),
    "szx_prefix_scan_i64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "szx_propagate_indices": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32,
                                             ctypes.c_void_p, ctypes.c_void_p]),
    "szx_propagate_round": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32,
                                           ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]),
    "szx_range_batch_scratch_bytes": (ctypes.c_size_t, [ctypes.c_uint32, ctypes.c_void_p]),
    "szx_range_batch_f32": (ctypes.c_int, [ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_size_t, ctypes.c_void_p]),
    "szx_compress_batch_scratch_bytes": (ctypes.c_size_t, [ctypes.c_uint32, ctypes.c_void_p]),
    "szx_compress_batch_f32": (ctypes.c_int, [ctypes.c_uint32] + [ctypes.c_void_p] * 9
                               + [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                  ctypes.c_void_p]),
    "szx_decompress_batch_scratch_bytes": (ctypes.c_size_t, [ctypes.c_uint32, ctypes.c_void_p]),
    "szx_decompress_batch_f32": (ctypes.c_int, [ctypes.c_uint32] + [ctypes.c_void_p] * 10
                                 + [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "szx_compress_batch_indexed_f32": (ctypes.c_int, [ctypes.c_uint32] + [ctypes.c_void_p] * 10
                                       + [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                          ctypes.c_void_p]),
    "szx_decompress_batch_indexed_f32": (ctypes.c_int, [ctypes.c_uint32] + [ctypes.c_void_p] * 10
                                         + [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "szx_compress_bound": (ctypes.c_uint64, [ctypes.c_uint64, ctypes.c_uint32,
                                             ctypes.c_uint32]),
    "szx_compress_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32,
                                         ctypes.c_uint32, ctypes.c_int32, ctypes.c_double,
                                         ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]),
    "szx_stream_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32,
                                       ctypes.c_void_p, ctypes.c_void_p]),
    "szx_decompress_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                           ctypes.c_uint64]),
}


def declared_symbols() -> list[str]:
    """Function names declared in include/szx_b200.h."""
    text = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"\b(szx_[a-z0-9_]+)\s*\(", text)))


def lib():
    """Load the native library, (re)building it first when it is missing or was built from
    other sources than the ones in the tree (content digest, _build.source_digest)."""
    global _lib
    if _lib is not None:
        return _lib
    from . import _build

    if _build._stale():
        try:
            _build.build()
        except Exception as exc:  # pragma: no cover - build environment specific
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryError(f"{LIB_PATH} missing and build failed: {exc}") from exc
            raise NativeLibraryError(f"{LIB_PATH} is stale and the rebuild failed: {exc}") from exc
    try:
        L = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, (res, args) in _SIGS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def last_error() -> str:
    msg = lib().szx_last_error()
    return msg.decode() if msg else ""


def require_cuda():
    """The codec runs only on a CUDA device; fail loudly otherwise."""
    import torch

    lib()
    if not torch.cuda.is_available():
        raise NativeLibraryError("no CUDA device visible: the SZx B200 codec has no CPU path")
    return torch
