"""Device plumbing: torch CUDA buffers, the current stream, and checked ABI calls."""
from __future__ import annotations

import ctypes

from . import _abi


def torch_cuda():
    return _abi.require_cuda()


def stream_ptr() -> int:
    torch = torch_cuda()
    return int(torch.cuda.current_stream().cuda_stream)


def empty_u8(nbytes: int, align: int = 256):
    """Uninitialised device bytes; torch allocations are >= 256-byte aligned."""
    torch = torch_cuda()
    t = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device="cuda")
    assert t.data_ptr() % align == 0
    return t


def ptr(t) -> int:
    return int(t.data_ptr())


def check(rc: int, what: str):
    if rc != _abi.OK:
        from .errors import error_for_status

        raise error_for_status(rc, f"{what}: {_abi.last_error()}")


class Scratch:
    """Grow-only device scratch per (purpose) key, reused across calls on one device."""

    _pool: dict = {}

    @classmethod
    def get(cls, key: str, nbytes: int):
        torch = torch_cuda()
        dev = torch.cuda.current_device()
        t = cls._pool.get((key, dev))
        if t is None or t.numel() < nbytes:
            t = empty_u8(max(nbytes, 256) + max(nbytes, 256) // 8)
            cls._pool[(key, dev)] = t
        return t


def small_host():
    """Pinned 256-byte host buffer for flag / totals readback."""
    torch = torch_cuda()
    return torch.empty(256, dtype=torch.uint8, pin_memory=True)


def totals_from(t_u8_cpu) -> _abi.Totals:
    raw = bytes(t_u8_cpu[:32].numpy().tobytes())
    return _abi.Totals.from_buffer_copy(raw)


def c_u64_array(values):
    arr = (ctypes.c_uint64 * len(values))(*[int(v) for v in values])
    return arr
