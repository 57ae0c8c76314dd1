"""Domain types and the bit-exact UFZX container, device-resident.

Mirrors ``ufzx/container.py`` (reference file:line cited per item).  Pools of a
``CompressedStream`` live in HBM as the kernels wrote them (constant map and leading codes
PACKED exactly as they appear in the container), so ``serialize`` is a gather of five
device ranges into one host buffer and ``deserialize`` is one host->device copy plus a
device pass that derives the mid-pool length.  The reference's unpacked NumPy views
(``constant_map``, ``leading_codes``, ...) are materialised on first access.

Layout (container.py:3-21, all multi-byte integers little-endian):
    "UFZX" | version 1 | dtype 0 | block_size u16 | error_bound f64 | ndims u8 |
    dims u64 x ndims | constant map | mu f32 x nb | req u8 x n_nc | 2-bit codes | mid bytes
"""
from __future__ import annotations

import math
import struct
import warnings

import numpy as np

from . import _abi, _device
from .errors import (
    FormatError,
    InconsistentLengthError,
    MalformedMagicError,
    PoolUnderrunError,
    TruncatedStreamError,
    UnsupportedDtypeError,
    VersionMismatchError,
    ZeroRangeError,
)

__all__ = [
    "MAGIC", "VERSION", "DTYPE_F32", "DTYPE_F64", "DataField", "ErrorBound",
    "CompressedStream", "serialize", "deserialize", "FormatError", "MalformedMagicError",
    "VersionMismatchError", "UnsupportedDtypeError", "TruncatedStreamError",
    "InconsistentLengthError", "PoolUnderrunError", "ZeroRangeError",
]

MAGIC = b"UFZX"          # container.py:30-33
VERSION = 1
DTYPE_F32 = 0x00
DTYPE_F64 = 0x01
_HEAD = struct.Struct("<4sBBHdB")  # container.py:35 (17 bytes)


def _ceil(a: int, b: int) -> int:
    return -(-a // b)


def _nc_elements(n: int, bs: int, n_nc: int, last_is_nc: bool) -> int:
    """Non-constant element count: every NC block is full except possibly the last block
    (container.py:232-239)."""
    if n_nc == 0:
        return 0
    nb = _ceil(n, bs)
    tail = n - (nb - 1) * bs
    return n_nc * bs - ((bs - tail) if last_is_nc else 0)


# --------------------------------------------------------------------------------------
# DataField / ErrorBound
# --------------------------------------------------------------------------------------
class DataField:
    """A flat float32 dataset plus its logical dimensions and global value stats
    (container.py:62-99).

    ``values`` may be array-like (kept on the host and uploaded once) or a torch tensor;
    the finite check and global min/max run on the GPU (K0, range_validate.cu).
    """

    element_size_bytes = 4

    def __init__(self, values, dims):
        torch = _device.torch_cuda()
        self._host = None
        if isinstance(values, torch.Tensor):
            dev = values.detach()
            if dev.dtype != torch.float32:
                dev = dev.to(torch.float32)
            dev = dev.reshape(-1)
            if not dev.is_cuda:
                dev = dev.cuda()
            if not dev.is_contiguous() or dev.data_ptr() % 16:
                dev = dev.clone()
        else:
            host = np.ascontiguousarray(values, dtype=np.float32).ravel()
            self._host = host
            dev = None
        self.dims = tuple(int(d) for d in dims)
        n = int(dev.numel()) if dev is not None else int(self._host.size)
        if n == 0:  # container.py:75-76
            raise ValueError("empty dataset")
        if not self.dims or any(d <= 0 for d in self.dims):  # container.py:77-78
            raise ValueError(f"dims must be positive, got {self.dims}")
        if math.prod(self.dims) != n:  # container.py:79-83
            raise ValueError(f"product(dims) = {math.prod(self.dims)} != {n} values")
        if dev is None:
            dev = torch.from_numpy(self._host).to("cuda", non_blocking=False)
        self._dev = dev
        self._n = n
        mn, mx, bad = _device_range(dev)
        if bad:  # container.py:84-85
            raise ValueError("non-finite value in dataset")
        self.global_min = mn  # container.py:86-87
        self.global_max = mx

    @classmethod
    def _from_device(cls, dev, dims, global_min=None, global_max=None):
        """Wrap decoded device values (stats computed lazily when not supplied)."""
        self = cls.__new__(cls)
        self._host = None
        self._dev = dev
        self._n = int(dev.numel())
        self.dims = tuple(int(d) for d in dims)
        self._gmin, self._gmax = global_min, global_max
        return self

    def _stats(self):
        if getattr(self, "_gmin", None) is None:
            mn, mx, bad = _device_range(self._dev)
            if bad:
                raise ValueError("non-finite value in dataset")
            self._gmin, self._gmax = mn, mx
        return self._gmin, self._gmax

    @property
    def global_min(self) -> float:
        return self._stats()[0]

    @global_min.setter
    def global_min(self, v):
        self._gmin = v

    @property
    def global_max(self) -> float:
        return self._stats()[1]

    @global_max.setter
    def global_max(self, v):
        self._gmax = v

    @property
    def values(self) -> np.ndarray:
        """Host float32 view (container.py:66); device results are copied once."""
        if self._host is None:
            self._host = self._dev.cpu().numpy()
        return self._host

    @property
    def device_values(self):
        """The float32 values as a CUDA tensor (resident in HBM)."""
        return self._dev

    @property
    def n(self) -> int:
        return self._n

    @property
    def value_range(self) -> float:
        return self.global_max - self.global_min

    @property
    def nbytes(self) -> int:
        return self.n * self.element_size_bytes

    def __repr__(self):
        return f"DataField(n={self.n}, dims={self.dims})"


def _device_range(dev):
    """(min, max, nonfinite) of a device float32 vector via K0."""
    torch = _device.torch_cuda()
    L = _abi.lib()
    n = int(dev.numel())
    scratch = _device.Scratch.get("range", L.szx_range_scratch_bytes(n))
    small = torch.zeros(16, dtype=torch.int32, device="cuda")  # [mn, mx, err]
    rc = L.szx_range_f32(_device.ptr(dev), n, _device.ptr(small), _device.ptr(small) + 8,
                         _device.ptr(scratch), scratch.numel(), _device.stream_ptr())
    _device.check(rc, "szx_range_f32")
    h = small.cpu().numpy()
    mn, mx = h[:2].view(np.float32)
    return float(mn), float(mx), bool(h[2] & _abi.FLAG_NONFINITE)


class ErrorBound:
    """User-facing bound: absolute, or relative to the dataset's global value range
    (container.py:102-114)."""

    __slots__ = ("mode", "magnitude")

    def __init__(self, mode: str, magnitude: float):
        if mode not in ("abs", "rel"):
            raise ValueError(f"unknown bound mode {mode!r}")
        m = float(magnitude)
        if not (m > 0 and math.isfinite(m)):
            raise ValueError(f"bound magnitude must be positive and finite, got {m}")
        object.__setattr__(self, "mode", mode)
        object.__setattr__(self, "magnitude", magnitude)

    def __setattr__(self, k, v):  # frozen dataclass semantics
        raise AttributeError("ErrorBound is immutable")

    def __eq__(self, other):
        return isinstance(other, ErrorBound) and (self.mode, self.magnitude) == (
            other.mode, other.magnitude)

    def __hash__(self):
        return hash((self.mode, self.magnitude))

    def __repr__(self):
        return f"ErrorBound(mode={self.mode!r}, magnitude={self.magnitude!r})"


# --------------------------------------------------------------------------------------
# CompressedStream
# --------------------------------------------------------------------------------------
class CompressedStream:
    """Parsed container contents (container.py:160-283), pools resident on the device.

    Constructing it from host arrays (the reference signature) uploads and validates the
    pools with the same checks and error classes as container.py:182-219.
    """

    def __init__(self, block_size, error_bound, dims, constant_map, mu_array, req_len_array,
                 leading_codes, mid_bytes):
        torch = _device.torch_cuda()
        self.block_size = int(block_size)
        self.error_bound = float(error_bound)
        self.dims = tuple(int(d) for d in dims)
        self._host = {}
        self._check_header_fields()
        nb = self.n_blocks
        cmap = np.ascontiguousarray(constant_map, dtype=bool)
        mu = np.ascontiguousarray(mu_array, dtype=np.float32)
        req = np.ascontiguousarray(req_len_array, dtype=np.uint8)
        codes = np.ascontiguousarray(leading_codes, dtype=np.uint8)
        mid = np.ascontiguousarray(mid_bytes, dtype=np.uint8)
        if len(cmap) != nb:  # container.py:190-193
            raise InconsistentLengthError(f"constant map has {len(cmap)} bits for {nb} blocks")
        if len(mu) != nb:  # container.py:194-197
            raise InconsistentLengthError(f"mu array has {len(mu)} entries for {nb} blocks")
        # pools get the same slack as compress output (_Pools): the decoders read 16-byte
        # supersets and whole 32-byte code rows
        d_mu = _padded(torch.from_numpy(mu.view(np.uint8))).view(torch.float32)[:nb]
        if not bool(torch.isfinite(d_mu).all()):  # container.py:198-199
            raise InconsistentLengthError("non-finite mu")
        n_nc = int((~cmap).sum())
        if len(req) != n_nc:  # container.py:200-205
            raise InconsistentLengthError(
                f"req_len array has {len(req)} entries for {n_nc} non-constant blocks")
        d_req = _padded(torch.from_numpy(req))
        if n_nc and not bool(((d_req[:n_nc] >= 1) & (d_req[:n_nc] <= 32)).all()):  # 206-207
            raise InconsistentLengthError("required bit length outside 1..32")
        m = _nc_elements(self.n_values, self.block_size, n_nc, bool(not cmap[-1]))
        if len(codes) != m:  # container.py:208-212
            raise InconsistentLengthError(f"{len(codes)} leading codes for {m} non-constant elements")
        d_codes_u = torch.from_numpy(codes).cuda()
        if m and int(d_codes_u.max()) > 3:  # container.py:213-214
            raise InconsistentLengthError("leading code > 3")
        d_map = _pack_bits_device(torch.from_numpy(cmap.astype(np.uint8)).cuda(), 1)
        d_codes = _pack_bits_device(d_codes_u, 2)
        self._set_pools(d_map, d_mu, d_req, d_codes, n_nc, m)
        self._mid_buf, self._mid_len = _device.empty_u8(64), 0
        expected = self.expected_mid_bytes()
        if len(mid) != expected:  # container.py:215-219
            raise InconsistentLengthError(
                f"mid pool has {len(mid)} bytes, expected {expected}")
        d_mid = _device.empty_u8(len(mid) + 48)
        if len(mid):
            d_mid[: len(mid)].copy_(torch.from_numpy(mid))
        self._mid_buf = d_mid
        self._mid_len = len(mid)

    # ---- construction from device pools (compress / deserialize) -----------------------
    @classmethod
    def _from_device(cls, block_size, error_bound, dims, d_map, d_mu, d_req, d_codes, d_mid_buf,
                     n_nc, m, mid_len):
        self = cls.__new__(cls)
        self.block_size = int(block_size)
        self.error_bound = float(error_bound)
        self.dims = tuple(int(d) for d in dims)
        self._host = {}
        self._set_pools(d_map, d_mu, d_req, d_codes, int(n_nc), int(m))
        self._mid_buf = d_mid_buf
        self._mid_len = int(mid_len)
        self._expected_mid = int(mid_len)
        return self

    def _set_pools(self, d_map, d_mu, d_req, d_codes, n_nc, m):
        self._map = d_map          # u8, ceil(nb/8) used bytes (buffer may be longer)
        self._mu = d_mu            # f32, nb
        self._req = d_req          # u8, n_nc
        self._codes = d_codes      # u8, ceil(2m/8) used bytes, packed LSB-first
        self._index = None         # bs 64/128/256/512: the decode index (K1 or K3)
        self._n_nc = int(n_nc)
        self._m = int(m)
        self._expected_mid = None

    def _check_header_fields(self):
        if not 8 <= self.block_size <= 65535:  # container.py:183-184
            raise InconsistentLengthError(f"block size {self.block_size} out of range")
        if not (self.error_bound > 0 and math.isfinite(self.error_bound)):  # 185-186
            raise InconsistentLengthError(f"error bound {self.error_bound} not positive finite")
        if not self.dims or any(d <= 0 for d in self.dims):  # 187-188
            raise InconsistentLengthError(f"bad dims {self.dims}")

    # ---- sizes ---------------------------------------------------------------------------
    @property
    def n_values(self) -> int:
        return math.prod(self.dims)

    @property
    def n_blocks(self) -> int:
        return _ceil(self.n_values, self.block_size)

    def block_counts(self) -> np.ndarray:
        counts = np.full(self.n_blocks, self.block_size, dtype=np.int64)
        counts[-1] = self.n_values - (self.n_blocks - 1) * self.block_size
        return counts

    @property
    def n_nonconstant_blocks(self) -> int:
        return self._n_nc

    @property
    def n_nonconstant_elements(self) -> int:
        return self._m

    @property
    def mid_len(self) -> int:
        return self._mid_len

    def byte_counts_per_block(self) -> np.ndarray:
        """q per non-constant block, in block order (container.py:241-244)."""
        req = self.req_len_array.astype(np.int64)
        return (req + (8 - req % 8) % 8) // 8

    def expected_mid_bytes(self) -> int:
        """Mid length the codes imply (container.py:246-253), derived on the device."""
        if self._expected_mid is None:
            total, flags = _validate_device(self)
            self._expected_mid = total
        return self._expected_mid

    def compressed_size_bytes(self) -> int:
        """container.py:255-266."""
        nb = self.n_blocks
        return (_HEAD.size + 8 * len(self.dims) + _ceil(nb, 8) + 4 * nb + self._n_nc
                + _ceil(2 * self._m, 8) + self._mid_len)

    # ---- device views ----------------------------------------------------------------------
    @property
    def device_pools(self) -> dict:
        """Exact-length device views of the five pools (packed as in the container)."""
        nb = self.n_blocks
        return {
            "constant_map": self._map[: _ceil(nb, 8)],
            "mu": self._mu[:nb],
            "req": self._req[: self._n_nc],
            "codes": self._codes[: _ceil(2 * self._m, 8)],
            "mid": self._mid_buf[: self._mid_len],
        }

    # ---- reference-compatible host views (container.py:167-171) ------------------------------
    def _h(self, key, fn):
        if key not in self._host:
            self._host[key] = fn()
        return self._host[key]

    @property
    def constant_map(self) -> np.ndarray:
        nb = self.n_blocks
        return self._h("map", lambda: np.unpackbits(
            self.device_pools["constant_map"].cpu().numpy(), bitorder="little")[:nb].astype(bool))

    @property
    def mu_array(self) -> np.ndarray:
        return self._h("mu", lambda: self.device_pools["mu"].cpu().numpy().astype(np.float32))

    @property
    def req_len_array(self) -> np.ndarray:
        return self._h("req", lambda: self.device_pools["req"].cpu().numpy().astype(np.uint8))

    @property
    def leading_codes(self) -> np.ndarray:
        def unpack():
            raw = self.device_pools["codes"].cpu().numpy()
            spread = np.stack([(raw >> (2 * j)) & 3 for j in range(4)], axis=1).reshape(-1)
            return spread[: self._m].astype(np.uint8)
        return self._h("codes", unpack)

    @property
    def mid_bytes(self) -> np.ndarray:
        return self._h("mid", lambda: self.device_pools["mid"].cpu().numpy().astype(np.uint8))

    def __eq__(self, other):
        """Bitwise equality of every pool (container.py:268-283), compared on the device."""
        if not isinstance(other, CompressedStream):
            return NotImplemented
        if (self.block_size, self.error_bound, self.dims, self._n_nc, self._m, self._mid_len) != (
                other.block_size, other.error_bound, other.dims, other._n_nc, other._m,
                other._mid_len):
            return False
        torch = _device.torch_cuda()
        a, b = self.device_pools, other.device_pools
        return all(torch.equal(a[k].view(torch.uint8) if k != "mu" else a[k].view(torch.int32),
                               b[k].view(torch.uint8) if k != "mu" else b[k].view(torch.int32))
                   for k in a)

    __hash__ = None

    def __repr__(self):
        return (f"CompressedStream(n={self.n_values}, block_size={self.block_size}, "
                f"n_nc={self._n_nc}, mid={self._mid_len}, bytes={self.compressed_size_bytes()})")


def _padded(host_u8, slack: int = 64):
    """Device copy of a host byte tensor with `slack` zero bytes after it."""
    buf = _device.empty_u8(host_u8.numel() + slack)
    buf.zero_()
    if host_u8.numel():
        buf[: host_u8.numel()].copy_(host_u8)
    return buf


def _pack_bits_device(vals_u8, width: int):
    """Pack 1- or 2-bit values LSB-first into bytes on the device (container.py:286-294,
    321).  64 bytes of zero slack follow (the decoders read whole code rows)."""
    torch = _device.torch_cuda()
    per = 8 // width
    k = vals_u8.numel()
    nbytes = _ceil(k * width, 8)
    buf = _device.empty_u8(nbytes + 64)
    buf.zero_()
    if k:
        padded = torch.zeros(nbytes * per, dtype=torch.uint8, device="cuda")
        padded[:k] = vals_u8
        sh = torch.arange(per, dtype=torch.uint8, device="cuda") * width
        packed = (padded.view(-1, per) << sh).sum(dim=1, dtype=torch.int32).to(torch.uint8)
        buf[:nbytes] = packed
    return buf


def _validate_device(stream: CompressedStream):
    """K3: mid length implied by req + codes, plus device-side pool flags."""
    torch = _device.torch_cuda()
    L = _abi.lib()
    p = stream.device_pools
    small = torch.zeros(4, dtype=torch.int64, device="cuda")  # [mid_total, err]
    rc = L.szx_validate_f32(_device.ptr(p["req"]) if stream._n_nc else 0, stream._n_nc,
                            _device.ptr(p["codes"]) if stream._m else 0, stream._m,
                            _device.ptr(p["mu"]), stream.n_blocks, stream.block_size,
                            _device.ptr(small), _device.ptr(small) + 8, _device.stream_ptr())
    _device.check(rc, "szx_validate_f32")
    h = small.cpu().numpy()
    return int(h[0]), int(h[1])


def _index_device(stream: CompressedStream):
    """K3 for block sizes 64/128/256/512: tile index (cached on the stream) + mid length + flags."""
    torch = _device.torch_cuda()
    L = _abi.lib()
    n, bs = stream.n_values, stream.block_size
    p = stream.device_pools
    idx = torch.empty(L.szx_index_bytes(n, bs) // 8, dtype=torch.int64, device="cuda")
    scratch = _device.Scratch.get("index", L.szx_index_scratch_bytes(n, bs))
    small = torch.zeros(4, dtype=torch.int64, device="cuda")  # nc_total, mid_total, err
    P = _device.ptr
    rc = L.szx_index_f32(P(p["constant_map"]), P(p["mu"]), P(stream._req), P(stream._codes), n,
                         bs, P(idx), P(small), P(small) + 16, P(scratch), scratch.numel(),
                         _device.stream_ptr())
    _device.check(rc, "szx_index_f32")
    h = small.cpu().numpy()
    stream._index = idx
    return int(h[1]), int(h[2])


# --------------------------------------------------------------------------------------
# serialize / deserialize
# --------------------------------------------------------------------------------------
def _header(stream: CompressedStream) -> bytes:
    return _HEAD.pack(MAGIC, VERSION, DTYPE_F32, stream.block_size, stream.error_bound,
                      len(stream.dims)) + struct.pack(f"<{len(stream.dims)}Q", *stream.dims)


def serialize(stream: CompressedStream) -> bytes:
    """Emit the container bytes (container.py:309-326): one device->host gather of the
    five pools into a pinned buffer at their container offsets."""
    torch = _device.torch_cuda()
    head = _header(stream)
    total = stream.compressed_size_bytes()
    out = torch.empty(total, dtype=torch.uint8, pin_memory=True)
    out[: len(head)] = torch.frombuffer(bytearray(head), dtype=torch.uint8)
    pos = len(head)
    for key in ("constant_map", "mu", "req", "codes", "mid"):
        src = stream.device_pools[key]
        nbytes = src.numel() * src.element_size()
        if nbytes:
            out[pos: pos + nbytes].copy_(src.view(torch.uint8).reshape(-1), non_blocking=True)
        pos += nbytes
    torch.cuda.current_stream().synchronize()
    return out.numpy().tobytes()


def _take(pos: int, n: int, length: int, what: str) -> int:
    if pos + n > length:  # container.py:334-339
        raise TruncatedStreamError(
            f"stream ends inside {what}: need {n} bytes at offset {pos}, have {length - pos}")
    return pos + n


def deserialize(data) -> CompressedStream:
    """Parse container bytes (container.py:349-416) into device pools.

    Header, map, req and code-padding checks run on the host in the reference's order; the
    bytes are then copied to the device once, where K3 derives the mid-pool length and
    checks mu, before the remaining length checks.
    """
    buf = np.frombuffer(bytes(data) if not isinstance(data, (bytes, bytearray)) else data,
                        dtype=np.uint8)
    length = buf.size
    pos = _take(0, _HEAD.size, length, "header")
    magic, version, dtype, block_size, bound, ndims = _HEAD.unpack(buf[: _HEAD.size].tobytes())
    if magic != MAGIC:
        raise MalformedMagicError(f"bad magic {magic!r}")
    if version != VERSION:
        raise VersionMismatchError(f"unsupported version {version}")
    if dtype == DTYPE_F64:
        raise UnsupportedDtypeError("float64 payloads are reserved and not supported")
    if dtype != DTYPE_F32:
        raise UnsupportedDtypeError(f"unknown dtype code {dtype:#x}")
    if ndims < 1:
        raise InconsistentLengthError("ndims must be >= 1")
    p0 = pos
    pos = _take(pos, 8 * ndims, length, "dims")
    dims = struct.unpack(f"<{ndims}Q", buf[p0:pos].tobytes())
    if any(d == 0 for d in dims):
        raise InconsistentLengthError(f"zero dimension in {dims}")
    if not 8 <= block_size <= 65535:
        raise InconsistentLengthError(f"block size {block_size} out of range")
    if not (bound > 0 and math.isfinite(bound)):
        raise InconsistentLengthError(f"error bound {bound} not positive finite")
    n = math.prod(dims)
    nb = _ceil(n, block_size)

    o_map = pos
    pos = _take(pos, _ceil(nb, 8), length, "constant map")
    map_bytes = buf[o_map:pos]
    if nb % 8 and int(map_bytes[-1]) >> (nb % 8):  # container.py:379-380
        raise InconsistentLengthError("nonzero padding bits in constant map")
    n_const = int(np.unpackbits(map_bytes).sum())
    o_mu = pos
    pos = _take(pos, 4 * nb, length, "mu array")
    n_nc = nb - n_const
    o_req = pos
    pos = _take(pos, n_nc, length, "req_len array")
    req = buf[o_req:pos]
    if n_nc and not ((req >= 1) & (req <= 32)).all():  # container.py:389-390
        raise InconsistentLengthError("required bit length outside 1..32")
    last_is_nc = not ((int(map_bytes[(nb - 1) >> 3]) >> ((nb - 1) & 7)) & 1)
    m = _nc_elements(n, block_size, n_nc, last_is_nc)
    o_codes = pos
    pos = _take(pos, _ceil(2 * m, 8), length, "leading code pool")
    if m % 4 and int(buf[pos - 1]) >> (2 * (m % 4)):  # container.py:304-305
        raise InconsistentLengthError("nonzero padding bits in leading code pool")
    o_mid = pos
    remaining = length - o_mid

    # one host->device copy, placed so the mid pool starts 16-byte aligned
    torch = _device.torch_cuda()
    lead = (-o_mid) % 16
    dev = _device.empty_u8(lead + length + 64)
    dev[lead + length:].zero_()
    with warnings.catch_warnings():  # read-only bytes are only read by the copy
        warnings.simplefilter("ignore")
        src = torch.from_numpy(buf) if buf.size else torch.empty(0, dtype=torch.uint8)
    dev[lead: lead + length].copy_(src)
    blob = dev[lead:]

    def aligned_view(off, nbytes, align):
        v = blob[off: off + nbytes]
        if (blob.data_ptr() + off) % align:
            c = _device.empty_u8(nbytes + 32)  # bulk copies read 16-byte supersets
            c[:nbytes].copy_(v)
            return c
        return blob[off:]

    d_map = aligned_view(o_map, _ceil(nb, 8), 4)
    d_mu = aligned_view(o_mu, 4 * nb, 4)[: 4 * nb].view(torch.float32)
    d_req = blob[o_req:]
    d_codes = blob[o_codes:]
    d_mid_buf = blob[o_mid:]
    stream = CompressedStream._from_device(block_size, bound, dims, d_map, d_mu, d_req, d_codes,
                                           d_mid_buf, n_nc, m, 0)
    if block_size in (64, 128, 256, 512):  # K3 index: the scan of the stored sizes, kept
        mid_len, flags = _index_device(stream)
    else:
        mid_len, flags = _validate_device(stream)
    if mid_len > remaining:  # container.py:403
        raise TruncatedStreamError(
            f"stream ends inside mid byte pool: need {mid_len} bytes at offset {o_mid}, "
            f"have {remaining}")
    if remaining > mid_len:  # container.py:404-405
        raise InconsistentLengthError(f"{remaining - mid_len} trailing bytes after mid pool")
    if flags & _abi.FLAG_MU_NONFINITE:  # container.py:198-199 (CompressedStream._validate)
        raise InconsistentLengthError("non-finite mu")
    stream._mid_len = mid_len
    stream._expected_mid = mid_len
    return stream
