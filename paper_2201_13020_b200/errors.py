"""Exception taxonomy of the reference (container.py:38-59, blockcodec.py:25-26,
pipeline.py:17-18), plus the mapping from C-ABI status codes onto it."""
from __future__ import annotations

from . import _abi


class FormatError(ValueError):
    """Base class for container format violations."""


class MalformedMagicError(FormatError):
    pass


class VersionMismatchError(FormatError):
    pass


class UnsupportedDtypeError(FormatError):
    pass


class TruncatedStreamError(FormatError):
    pass


class InconsistentLengthError(FormatError):
    pass


class PoolUnderrunError(FormatError):
    """Mid-byte pool exhausted during decode: the stream is corrupt."""


class ZeroRangeError(ValueError):
    """Relative bound on a zero-range (flat) dataset resolves to e = 0."""


_STATUS = {
    _abi.ERR_INVALID_ARG: ValueError,
    _abi.ERR_CUDA: RuntimeError,
    _abi.ERR_ALIGN: ValueError,
    _abi.ERR_NONFINITE: ValueError,
    _abi.ERR_ZERO_RANGE: ZeroRangeError,
    _abi.ERR_BAD_REQ: InconsistentLengthError,
    _abi.ERR_UNDERRUN: PoolUnderrunError,
    _abi.ERR_TRUNCATED: TruncatedStreamError,
    _abi.ERR_MAGIC: MalformedMagicError,
    _abi.ERR_VERSION: VersionMismatchError,
    _abi.ERR_DTYPE: UnsupportedDtypeError,
    _abi.ERR_INCONSISTENT: InconsistentLengthError,
    _abi.ERR_CAPACITY: ValueError,
    _abi.ERR_NO_DEVICE: _abi.NativeLibraryError,
}


def error_for_status(rc: int, msg: str) -> Exception:
    return _STATUS.get(rc, RuntimeError)(msg)
