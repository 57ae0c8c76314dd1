"""One UFZX stream from a field sharded across GPUs.

Blocks are independent once the bound e is fixed (``prev`` restarts at every block,
``pipeline.py:108-111``; decode state is per block, ``pipeline.py:212-213``), so each rank
compresses a contiguous, block-aligned shard of the field with the same absolute e and the
per-rank pools are byte ranges of the single-stream pools.  Shards hold a multiple of 8 blocks
(map bytes stay whole) and, for block sizes divisible by 4, every shard's codes start on a byte.

Collectives (NCCL over NVLink on GPUs, gloo in the CPU tests): one all-reduce of the shard
range for a relative bound, one all-gather of the per-shard pool sizes.  The payload never
crosses GPUs: every rank writes its own pools at its offsets in the shared output.

Decompression mirrors it: every rank reads the header and the constant
map of the one stream, locates its shard's map / mu / req / code ranges from the map alone (the
NC blocks before the shard come from map popcounts; every NC block but the field's last is
full), derives its shard's mid-byte total from its own codes and req bytes on the device (K3),
and one all-gather of those totals gives every rank its mid-pool offset.  Each rank then reads
only its own byte ranges of the stream and decodes its shard.
"""
from __future__ import annotations

import math
import os
import struct
from dataclasses import dataclass

import numpy as np

_HEAD = struct.Struct("<4sBBHdB")  # container.py:35


def shard_plan(n: int, block_size: int, world: int, align_blocks: int = 8):
    """Contiguous block-aligned value ranges [v0, v1) per rank; every shard but the last
    holds a multiple of `align_blocks` blocks."""
    nb = -(-n // block_size)
    per = -(-nb // world)
    per = -(-per // align_blocks) * align_blocks
    out = []
    for r in range(world):
        b0 = min(nb, r * per)
        b1 = min(nb, b0 + per)
        out.append((min(n, b0 * block_size), min(n, b1 * block_size)))
    return out


@dataclass(frozen=True)
class ShardSizes:
    nb: int        # blocks
    n_nc: int      # non-constant blocks (req bytes)
    m: int         # non-constant elements (2-bit codes)
    mid_len: int   # mid bytes

    def as_list(self):
        return [self.nb, self.n_nc, self.m, self.mid_len]


@dataclass(frozen=True)
class ShardOffsets:
    header_len: int
    total_len: int
    map_off: int
    mu_off: int
    req_off: int
    codes_off: int
    mid_off: int


def header_bytes(dims, block_size: int, e: float) -> bytes:
    """container.py:312-320."""
    dims = tuple(int(d) for d in dims)
    return _HEAD.pack(b"UFZX", 1, 0, block_size, float(e), len(dims)) + struct.pack(
        f"<{len(dims)}Q", *dims)


def shard_offsets(sizes: list[ShardSizes], rank: int, ndims: int) -> ShardOffsets:
    """Byte offsets of rank `rank`'s pools inside the single stream (container.py:255-266)."""
    H = _HEAD.size + 8 * ndims
    nb = sum(s.nb for s in sizes)
    n_nc = sum(s.n_nc for s in sizes)
    m = sum(s.m for s in sizes)
    mid = sum(s.mid_len for s in sizes)
    map0 = H
    mu0 = map0 + -(-nb // 8)
    req0 = mu0 + 4 * nb
    codes0 = req0 + n_nc
    mid0 = codes0 + -(-2 * m // 8)
    total = mid0 + mid
    before = sizes[:rank]
    b_nb = sum(s.nb for s in before)
    b_m = sum(s.m for s in before)
    if b_nb % 8:
        raise ValueError("shard block counts must be multiples of 8 (map bytes)")
    if b_m % 4:
        raise ValueError("shard code pools must start on a byte (block size % 4 == 0)")
    return ShardOffsets(
        header_len=H, total_len=total, map_off=map0 + b_nb // 8, mu_off=mu0 + 4 * b_nb,
        req_off=req0 + sum(s.n_nc for s in before), codes_off=codes0 + b_m // 4,
        mid_off=mid0 + sum(s.mid_len for s in before))


def gather_sizes(local: ShardSizes, group=None, device=None) -> list[ShardSizes]:
    """All-gather of the 4 x u64 per-shard sizes (the one collective of the assembly)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    t = torch.tensor(local.as_list(), dtype=torch.int64, device=device)
    out = torch.empty(world * 4, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out, t, group=group)
    v = out.cpu().tolist()
    return [ShardSizes(*v[4 * r: 4 * r + 4]) for r in range(world)]


def global_range(lo: float, hi: float, nonfinite: bool, group=None, device=None):
    """All-reduce MIN/MAX of the shard ranges plus the non-finite flag (container.py:84-87)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([-lo, hi, 1.0 if nonfinite else 0.0], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    v = t.cpu().tolist()
    return -v[0], v[1], v[2] > 0


def write_pools(path: str, off: ShardOffsets, header: bytes | None, pools: dict, rank: int):
    """Write this rank's pools (host byte arrays) at their offsets of the shared output file.
    Rank 0 also writes the header and sizes the file."""
    flags = os.O_RDWR | os.O_CREAT
    fd = os.open(path, flags, 0o644)
    try:
        if rank == 0:
            os.ftruncate(fd, off.total_len)
            if header is not None:
                os.pwrite(fd, header, 0)
        for key, pos in (("constant_map", off.map_off), ("mu", off.mu_off), ("req", off.req_off),
                         ("codes", off.codes_off), ("mid", off.mid_off)):
            data = np.ascontiguousarray(pools[key]).view(np.uint8)
            if data.size:
                os.pwrite(fd, data.tobytes(), pos)
    finally:
        os.close(fd)


@dataclass
class ShardResult:
    stream: object          # local CompressedStream (device pools)
    sizes: list             # ShardSizes of every rank
    offsets: ShardOffsets   # this rank's offsets in the single stream
    header: bytes
    error_bound: float


def compress_sharded(local_values, dims, cfg, v0: int, group=None) -> ShardResult:
    """Compress this rank's shard (device tensor of values [v0, v0+len)) of a field of shape
    `dims`; collective over `group` (NCCL)."""
    import torch
    import torch.distributed as dist

    from . import _abi, _device
    from .container import CompressedStream, DataField, _device_range
    from .errors import InconsistentLengthError, ZeroRangeError
    from .pipeline import _Pools, compress_device

    rank = dist.get_rank(group)
    if cfg.block_size % 4:  # checked on every rank before any collective (no rank blocks)
        raise ValueError("sharded streams need block_size % 4 == 0 (byte-aligned code pools)")
    dev = torch.device("cuda", torch.cuda.current_device())
    cdev = dev if dist.get_backend(group) == "nccl" else torch.device("cpu")  # collectives
    x = local_values.reshape(-1).to(torch.float32).contiguous()
    n_local = int(x.numel())
    bs = cfg.block_size
    if n_local:
        lo, hi, bad = _device_range(x)
    else:
        lo, hi, bad = math.inf, -math.inf, False
    gmin, gmax, gbad = global_range(lo, hi, bad, group=group, device=cdev)
    if gbad:
        raise ValueError("non-finite value in dataset")
    if cfg.bound.mode == "abs":
        e = float(cfg.bound.magnitude)
    else:
        e = float(cfg.bound.magnitude) * (gmax - gmin)  # pipeline.py:38
        if e == 0:
            raise ZeroRangeError("relative bound on a zero-range dataset resolves to 0")
    stream = None
    nb_local = -(-n_local // bs)
    if n_local:
        pools = _Pools(n_local, bs)
        small = torch.zeros(8, dtype=torch.int64, device=dev)
        compress_device(x, n_local, bs, e, pools, small, _device.stream_ptr())
        h = small.cpu().numpy()
        if int(h[4]) & _abi.FLAG_BAD_REQ:
            raise InconsistentLengthError("required bit length outside 1..32")
        stream = CompressedStream._from_device(
            bs, e, (n_local,), pools.map, pools.mu[: 4 * nb_local].view(torch.float32), pools.req,
            pools.codes, pools.mid, int(h[0]), int(h[1]), int(h[2]))
        local = ShardSizes(nb_local, int(h[0]), int(h[1]), int(h[2]))
    else:
        local = ShardSizes(0, 0, 0, 0)
    sizes = gather_sizes(local, group=group, device=cdev)
    off = shard_offsets(sizes, rank, len(dims))
    return ShardResult(stream, sizes, off, header_bytes(dims, bs, e), e)


def write_sharded(result: ShardResult, path: str, group=None):
    """Every rank writes its pools into the shared stream file (D2H of its own pools only)."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    pools = {}
    if result.stream is not None:
        for k, v in result.stream.device_pools.items():
            pools[k] = v.contiguous().view(-1).cpu().numpy().view(np.uint8)
    else:
        pools = {k: np.zeros(0, np.uint8) for k in ("constant_map", "mu", "req", "codes", "mid")}
    write_pools(path, result.offsets, result.header, pools, rank)
    dist.barrier(group=group)


# --------------------------------------------------------------------------------------
# decompression of one stream across ranks
# --------------------------------------------------------------------------------------
@dataclass
class ShardPools:
    """One rank's view of a UFZX stream: header fields and its shard's pool byte ranges."""
    dims: tuple
    block_size: int
    error_bound: float
    n: int                 # values of the whole field
    v0: int                # this shard: values [v0, v1), blocks [b0, b1)
    v1: int
    b0: int
    b1: int
    nc_before: int         # NC blocks before the shard
    n_nc: int              # NC blocks in the shard
    m: int                 # NC elements in the shard
    map_bytes: np.ndarray  # the shard's constant-map bytes (b0 is a multiple of 8)
    mu_range: tuple        # (offset, length) in the stream
    req_range: tuple
    codes_range: tuple
    mid0: int              # stream offset of the mid pool
    total_len: int         # stream length


def _read_at(src, off: int, n: int) -> bytes:
    if isinstance(src, (bytes, bytearray, memoryview)):
        return bytes(src[off: off + n])
    return os.pread(src, n, off)


def read_shard(src, rank: int, world: int, align_blocks: int = 8) -> ShardPools:
    """Parse the header and constant map of a UFZX stream (bytes, or an open file descriptor)
    and locate rank `rank`'s pools (container.py:349-402 checks, in the reference's order)."""
    from .container import _HEAD as CHEAD, _take, _nc_elements
    from .errors import (InconsistentLengthError, MalformedMagicError, UnsupportedDtypeError,
                         VersionMismatchError)

    total = len(src) if isinstance(src, (bytes, bytearray, memoryview)) else os.fstat(src).st_size
    _take(0, CHEAD.size, total, "header")
    magic, version, dtype, bs, e, ndims = CHEAD.unpack(_read_at(src, 0, CHEAD.size))
    if magic != b"UFZX":
        raise MalformedMagicError(f"bad magic {magic!r}")
    if version != 1:
        raise VersionMismatchError(f"unsupported version {version}")
    if dtype != 0:
        raise UnsupportedDtypeError(f"unsupported dtype code {dtype:#x}")
    if ndims < 1:
        raise InconsistentLengthError("ndims must be >= 1")
    pos = _take(CHEAD.size, 8 * ndims, total, "dims")
    dims = struct.unpack(f"<{ndims}Q", _read_at(src, CHEAD.size, 8 * ndims))
    if any(d == 0 for d in dims):
        raise InconsistentLengthError(f"zero dimension in {dims}")
    if not 8 <= bs <= 65535:
        raise InconsistentLengthError(f"block size {bs} out of range")
    if not (e > 0 and math.isfinite(e)):
        raise InconsistentLengthError(f"error bound {e} not positive finite")
    if bs % 4:
        raise ValueError("sharded streams need block_size % 4 == 0 (byte-aligned code pools)")
    n = math.prod(dims)
    nb = -(-n // bs)
    o_map = pos
    pos = _take(pos, -(-nb // 8), total, "constant map")
    cmap = np.frombuffer(_read_at(src, o_map, -(-nb // 8)), np.uint8)
    if nb % 8 and int(cmap[-1]) >> (nb % 8):
        raise InconsistentLengthError("nonzero padding bits in constant map")
    o_mu = pos
    pos = _take(pos, 4 * nb, total, "mu array")
    bits = np.unpackbits(cmap, bitorder="little")[:nb]
    n_nc_all = int(nb - bits.sum())
    o_req = pos
    pos = _take(pos, n_nc_all, total, "req_len array")
    last_nc = not bits[-1]
    m_all = _nc_elements(n, bs, n_nc_all, bool(last_nc))
    o_codes = pos
    pos = _take(pos, -(-2 * m_all // 8), total, "leading code pool")
    mid0 = pos
    v0, v1 = shard_plan(n, bs, world, align_blocks)[rank]
    b0, b1 = -(-v0 // bs), -(-v1 // bs)
    nc_before = int(b0 - bits[:b0].sum())
    n_nc = int((b1 - b0) - bits[b0:b1].sum())
    m = _nc_elements(v1 - v0, bs, n_nc, bool(b1 > b0 and not bits[b1 - 1])) if b1 > b0 else 0
    m_before = nc_before * bs  # every NC block before the shard is full
    return ShardPools(
        dims=tuple(int(d) for d in dims), block_size=bs, error_bound=float(e), n=n, v0=v0, v1=v1,
        b0=b0, b1=b1, nc_before=nc_before, n_nc=n_nc, m=m,
        map_bytes=cmap[b0 // 8: -(-b1 // 8)].copy(),
        mu_range=(o_mu + 4 * b0, 4 * (b1 - b0)),
        req_range=(o_req + nc_before, n_nc),
        codes_range=(o_codes + m_before // 4, -(-2 * m // 8)),
        mid0=mid0, total_len=total)


def mid_offsets(local_mid: int, group=None, device=None):
    """All-gather of the per-shard mid totals (the one collective of sharded decode): returns
    (mid bytes before this rank's shard, mid bytes of the whole stream)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    t = torch.tensor([int(local_mid)], dtype=torch.int64, device=device)
    out = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out, t, group=group)
    v = out.cpu().tolist()
    return sum(v[:rank]), sum(v)


def check_mid_total(sp: ShardPools, mid_total: int):
    """container.py:403-405 on the whole stream, identically on every rank."""
    from .errors import InconsistentLengthError, TruncatedStreamError

    remaining = sp.total_len - sp.mid0
    if mid_total > remaining:
        raise TruncatedStreamError(
            f"stream ends inside mid byte pool: need {mid_total} bytes at offset {sp.mid0}, "
            f"have {remaining}")
    if remaining > mid_total:
        raise InconsistentLengthError(f"{remaining - mid_total} trailing bytes after mid pool")


def decompress_sharded(src, group=None):
    """Decode this rank's shard of ONE UFZX stream (bytes, or an open file descriptor that
    every rank can read).  Returns (values [v0, v1) of the field as a CUDA float32 tensor, v0,
    v1).  Collective over `group`: one all-gather of the shard mid totals."""
    import torch
    import torch.distributed as dist

    from . import _device
    from .container import CompressedStream, _index_device, _validate_device
    from .errors import InconsistentLengthError
    from .pipeline import decompress

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    cdev = dev if dist.get_backend(group) == "nccl" else torch.device("cpu")
    sp = read_shard(src, rank, world)
    n_local = sp.v1 - sp.v0
    stream = None
    local_mid, flags = 0, 0
    if n_local:
        def up(rng, slack=64):  # a pool range onto the device with the decoders' slack
            off, ln = rng
            buf = _device.empty_u8(ln + slack)
            buf.zero_()
            if ln:
                buf[:ln].copy_(torch.frombuffer(bytearray(_read_at(src, off, ln)), dtype=torch.uint8))
            return buf

        d_map = _device.empty_u8(sp.map_bytes.size + 64)
        d_map.zero_()
        d_map[: sp.map_bytes.size].copy_(torch.from_numpy(sp.map_bytes))
        nbl = sp.b1 - sp.b0
        d_mu = up(sp.mu_range).view(torch.float32)[:nbl]  # 4 nbl + 64 bytes: whole floats
        stream = CompressedStream._from_device(
            sp.block_size, sp.error_bound, (n_local,), d_map, d_mu, up(sp.req_range),
            up(sp.codes_range), _device.empty_u8(64), sp.n_nc, sp.m, 0)
        if sp.block_size == 128:  # K3: the shard's tile index + its mid total + checks
            local_mid, flags = _index_device(stream)
        else:
            local_mid, flags = _validate_device(stream)
    before, total_mid = mid_offsets(local_mid, group=group, device=cdev)
    check_mid_total(sp, total_mid)  # every rank raises the same error
    if stream is None:
        return torch.empty(0, dtype=torch.float32, device=dev), sp.v0, sp.v1
    from . import _abi
    if flags & _abi.FLAG_MU_NONFINITE:  # container.py:198-199
        raise InconsistentLengthError("non-finite mu")
    mid = _device.empty_u8(local_mid + 64)
    mid.zero_()
    if local_mid:
        mid[:local_mid].copy_(torch.frombuffer(
            bytearray(_read_at(src, sp.mid0 + before, local_mid)), dtype=torch.uint8))
    stream._mid_buf = mid
    stream._mid_len = local_mid
    stream._expected_mid = local_mid
    out = decompress(stream)
    return out.device_values, sp.v0, sp.v1
