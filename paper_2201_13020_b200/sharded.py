"""One UFZX stream from a field sharded across GPUs.

Blocks are independent once the bound e is fixed (``prev`` restarts at every block,
``pipeline.py:108-111``; decode state is per block, ``pipeline.py:212-213``), so each rank
compresses a contiguous, block-aligned shard of the field with the same absolute e and the
per-rank pools are byte ranges of the single-stream pools.  Shards hold a multiple of 8 blocks
(map bytes stay whole) and, for block sizes divisible by 4, every shard's codes start on a byte.

Collectives (NCCL over NVLink on GPUs, gloo in the CPU tests): one all-reduce of the shard
range for a relative bound, one all-gather of the per-shard pool sizes.  The payload never
crosses GPUs: every rank writes its own pools at its offsets in the shared output.
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
