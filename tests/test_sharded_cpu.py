"""Host logic of the multi-GPU path on CPU: shard plans, single-stream offsets, and a
world-size-2 gloo run of the size all-gather + range all-reduce + pool assembly.

Per-shard pools come from the oracle (test infrastructure) compressing each block-aligned shard
with the global absolute bound -- by block independence they are byte ranges of the
single-stream pools; the assembled file must equal the reference's stream."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import fields
import oracle
from paper_2201_13020_b200 import sharded


def test_shard_plan_alignment_and_coverage():
    for n, bs, world in [(1, 128, 2), (1000, 128, 2), (25_000_000, 128, 8), (280_953_867, 128, 8),
                         (4096 * 8 + 17, 17, 3), (12345, 8, 4)]:
        plan = sharded.shard_plan(n, bs, world)
        assert len(plan) == world
        assert plan[0][0] == 0 and plan[-1][1] == n
        for (a0, a1), (b0, _) in zip(plan, plan[1:]):
            assert a1 == b0
        for v0, v1 in plan[:-1]:
            if v1 > v0 and v1 < n:
                assert (v1 - v0) % (8 * bs) == 0


def _pools_for(values, bs, e):
    p = oracle.compress_pools(values, bs, e)
    return p, sharded.ShardSizes(int(p["nb"]), int(p["n_nc"]), int(p["m"]), int(p["mid_len"]))


def test_offsets_reassemble_stream_serially():
    rng = np.random.default_rng(4)
    x = fields.smooth_ridges(rng, 8 * 128 * 37 + 11)
    e = oracle.resolve_bound(x, "rel", 1e-3)
    blob = oracle.compress(x, None, 128, "abs", e)
    for world in (1, 2, 3, 5):
        plan = sharded.shard_plan(x.size, 128, world)
        parts = [_pools_for(x[v0:v1], 128, e) if v1 > v0 else (None, sharded.ShardSizes(0, 0, 0, 0))
                 for v0, v1 in plan]
        sizes = [s for _, s in parts]
        out = bytearray(sharded.shard_offsets(sizes, 0, 1).total_len)
        head = sharded.header_bytes((x.size,), 128, e)
        out[: len(head)] = head
        for r, (p, _) in enumerate(parts):
            if p is None:
                continue
            off = sharded.shard_offsets(sizes, r, 1)
            for key, pos in (("map", off.map_off), ("mu", off.mu_off), ("req", off.req_off),
                             ("codes", off.codes_off), ("mid", off.mid_off)):
                b = np.ascontiguousarray(p[key]).view(np.uint8).tobytes()
                out[pos: pos + len(b)] = b
        assert bytes(out) == blob, world


def test_offsets_reject_misaligned_code_pools():
    sizes = [sharded.ShardSizes(8, 8, 17 * 8 - 3, 10), sharded.ShardSizes(8, 8, 17 * 8, 10)]
    with pytest.raises(ValueError):
        sharded.shard_offsets(sizes, 1, 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, path, x, bs, rel, result_q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        v0, v1 = sharded.shard_plan(x.size, bs, world)[rank]
        local = x[v0:v1]
        lo, hi = (float(local.min()), float(local.max())) if local.size else (np.inf, -np.inf)
        gmin, gmax, bad = sharded.global_range(lo, hi, False)
        e = rel * (gmax - gmin)
        if local.size:
            p, size = _pools_for(local, bs, e)
        else:
            p, size = ({k: np.zeros(0, np.uint8) for k in ("map", "mu", "req", "codes", "mid")},
                       sharded.ShardSizes(0, 0, 0, 0))
        sizes = sharded.gather_sizes(size)
        off = sharded.shard_offsets(sizes, rank, 1)
        pools = {"constant_map": p["map"], "mu": p["mu"], "req": p["req"], "codes": p["codes"],
                 "mid": p["mid"]}
        sharded.write_pools(path, off, sharded.header_bytes((x.size,), bs, e), pools, rank)
        dist.barrier()
        if rank == 0:
            result_q.put((e, off.total_len))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_two_ranks_assemble_one_stream(world):
    rng = np.random.default_rng(9)
    x = fields.random_walk(rng, 128 * 8 * 50 + 77, step=0.05)
    bs, rel = 128, 1e-3
    blob = oracle.compress(x, None, bs, "rel", rel)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "stream.ufzx")
        mp.start_processes(_worker, args=(world, port, path, x, bs, rel, q), nprocs=world,
                           join=True, start_method="spawn")
        e, total = q.get(timeout=30)
        with open(path, "rb") as f:
            got = f.read()
    assert total == len(blob)
    assert got == blob
